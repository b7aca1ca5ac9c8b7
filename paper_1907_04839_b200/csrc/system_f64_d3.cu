// System<double, 3> and its kernel shapes.
#include "system_impl.cuh"

// Thin last row tile (PairArgs::thin_split) in the default fp64 shapes: measured and not adopted -- the extra code lifts
// the adjoint kernel from 180 to 222 registers and N = 20 000 goes from 21.92 to 22.39 ms per gradient for at most 0.9 %
// less row-tile padding (-DLMS_F64_THIN=true builds it for an A/B).
#ifndef LMS_F64_THIN
#define LMS_F64_THIN false
#endif

namespace lms {

template <>
KernelChoice<double> pick_kernel<double, 3, kFwd>(int v)
{
  switch (v) {
    case 1: return make_choice<double, 3, kFwd, 1, 2, 4>("fwd_f64_r1_j2");
    case 5: return make_choice<double, 3, kFwd, 2, 2, 3, false, 2>("fwd_f64_r2_j2_u2");
    default: return make_choice<double, 3, kFwd, 2, 2, 3, false, 2, true, false, false, true, LMS_F64_THIN>("fwd_f64_r2_j2_u2_tma");
  }
}
template <>
KernelChoice<double> pick_kernel<double, 3, kAdj>(int v)
{
  switch (v) {
    case 1: return make_choice<double, 3, kAdj, 1, 2, 3>("adj_f64_r1_j2");
    case 5: return make_choice<double, 3, kAdj, 2, 2, 2, false, 2>("adj_f64_r2_j2_u2");
    default: return make_choice<double, 3, kAdj, 2, 2, 2, false, 2, true, false, false, true, LMS_F64_THIN>("adj_f64_r2_j2_u2_tma");
  }
}
template <>
KernelChoice<double> pick_kernel<double, 3, kVel>(int)
{
  return make_choice<double, 3, kVel, 2, 2, 4>("vel_f64_r2_j2");
}

template class System<double, 3>;

}  // namespace lms
