// TEST INFRASTRUCTURE ONLY (oracle/): never linked into the product library.
//
// Contract-equivalent replacement for /root/reference/proj/src/parallel.cpp, which has a
// use-after-return race between Pool::run (parallel.cpp:41-57) and worker_loop (:109-115) and
// segfaults under multi-threaded load.  The contract kept is parallel.hpp:11-20: [0,n) split into
// at most `threads` contiguous chunks, chunk c = [n*c/chunks, n*(c+1)/chunks) (parallel.cpp:145-146),
// blocking, first exception rethrown.  Chunk contents depend only on (n, threads), so results are
// bitwise identical to the reference's single-threaded path for any worker count.
#include <algorithm>
#include <exception>
#include <mutex>
#include <thread>
#include <vector>

#include "lmshoot/parallel.hpp"

namespace lmshoot {

unsigned hardware_threads()
{
  unsigned n = std::thread::hardware_concurrency();
  return n == 0 ? 1u : n;
}

void parallel_for(std::size_t n, unsigned threads,
                  const std::function<void(std::size_t, std::size_t)>& body)
{
  if (n == 0) return;
  const std::size_t want = threads == 0 ? hardware_threads() : threads;
  const std::size_t chunks = std::min<std::size_t>(want, n);
  if (chunks <= 1) {
    body(0, n);
    return;
  }
  std::mutex err_mutex;
  std::exception_ptr first_error;
  auto run_chunk = [&](std::size_t c) {
    const std::size_t begin = n * c / chunks;
    const std::size_t end = n * (c + 1) / chunks;
    if (begin >= end) return;
    try {
      body(begin, end);
    } catch (...) {
      std::lock_guard<std::mutex> lock(err_mutex);
      if (!first_error) first_error = std::current_exception();
    }
  };
  std::vector<std::thread> pool;
  pool.reserve(chunks - 1);
  for (std::size_t c = 1; c < chunks; ++c) pool.emplace_back(run_chunk, c);
  run_chunk(0);
  for (auto& t : pool) t.join();
  if (first_error) std::rethrow_exception(first_error);
}

}  // namespace lmshoot
