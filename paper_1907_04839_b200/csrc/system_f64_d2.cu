// System<double, 2> and its kernel shapes.
#include "system_impl.cuh"

namespace lms {

template <>
KernelChoice<double> pick_kernel<double, 2, kFwd>(int)
{
  return make_choice<double, 2, kFwd, 2, 2, 3, false, 1, false, false, false, true>("fwd_f64_d2_r2_j2");
}
template <>
KernelChoice<double> pick_kernel<double, 2, kAdj>(int)
{
  return make_choice<double, 2, kAdj, 2, 2, 2, false, 1, false, false, false, true>("adj_f64_d2_r2_j2");
}
template <>
KernelChoice<double> pick_kernel<double, 2, kVel>(int)
{
  return make_choice<double, 2, kVel, 2, 2, 4>("vel_f64_d2_r2_j2");
}

template class System<double, 2>;

}  // namespace lms
