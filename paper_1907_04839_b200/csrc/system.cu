// Non-template parts of the engine: the row partition, variant names, the (precision, dim) dispatch
// (shooting.hpp:348-368).
#include "system.cuh"

namespace lms {

namespace {
inline long long round_up(long long v, long long m) { return (v + m - 1) / m * m; }
}  // namespace

RowPartition partition_rows(long long n, int world, int rank)
{
  // Equal, tile-aligned slices so the per-step exchange is one in-place all-gather per plane: the chunk
  // formula of parallel.cpp:145-146 applied to kRowAlign-row blocks, every rank padded to the same count.
  RowPartition p;
  p.slice = std::max<long long>(round_up((n + world - 1) / world, kRowAlign), kRowAlign);
  p.stride = p.slice * world;
  p.row_begin = std::min<long long>(p.slice * rank, n);
  p.row_end = std::min<long long>(p.slice * (rank + 1), n);
  return p;
}

const char* variant_name(int precision, int variant)
{
  // names of the 3-D forward kernels; the adjoint / velocity variants follow the same index
  if (precision == LMS_PRECISION_F32) return pick_kernel<float, 3, kFwd>(variant).name;
  return pick_kernel<double, 3, kFwd>(variant).name;
}

SystemBase* create_system(const lms_config& cfg, int batch_count)
{
  const bool f32 = cfg.precision == LMS_PRECISION_F32;
  if (cfg.dim == 3)
    return f32 ? (SystemBase*)new System<float, 3>(cfg, batch_count) : (SystemBase*)new System<double, 3>(cfg, batch_count);
  return f32 ? (SystemBase*)new System<float, 2>(cfg, batch_count) : (SystemBase*)new System<double, 2>(cfg, batch_count);
}

}  // namespace lms
