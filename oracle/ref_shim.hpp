// TEST INFRASTRUCTURE ONLY (oracle/): never linked into the product library.
//
// Pre-include shim that lets the reference headers under /root/reference/proj/include compile
// unmodified.  lmshoot::Vec<T,D> is std::array<T,D> with an `int D` template parameter
// (vec.hpp:12-13); std::array's extent is std::size_t, so the operator templates at
// vec.hpp:18-47 can never deduce D and the expressions q[i] - q[j] at shooting.hpp:132,159,250,255
// do not compile.  Declaring the same component-wise operators over std::array<T, std::size_t N>
// in namespace lmshoot *before* the reference headers are parsed makes ordinary unqualified lookup
// find them at the template definition point.  Arithmetic is the same loop as vec.hpp:18-47.
#pragma once
#include <array>
#include <cstddef>

namespace lmshoot {

template <class T, std::size_t N>
inline std::array<T, N> operator+(const std::array<T, N>& a, const std::array<T, N>& b)
{
  std::array<T, N> r;
  for (std::size_t k = 0; k < N; ++k) r[k] = a[k] + b[k];
  return r;
}

template <class T, std::size_t N>
inline std::array<T, N> operator-(const std::array<T, N>& a, const std::array<T, N>& b)
{
  std::array<T, N> r;
  for (std::size_t k = 0; k < N; ++k) r[k] = a[k] - b[k];
  return r;
}

template <class T, std::size_t N>
inline std::array<T, N> operator*(T s, const std::array<T, N>& a)
{
  std::array<T, N> r;
  for (std::size_t k = 0; k < N; ++k) r[k] = s * a[k];
  return r;
}

template <class T, std::size_t N>
inline std::array<T, N>& operator+=(std::array<T, N>& a, const std::array<T, N>& b)
{
  for (std::size_t k = 0; k < N; ++k) a[k] += b[k];
  return a;
}

}  // namespace lmshoot
