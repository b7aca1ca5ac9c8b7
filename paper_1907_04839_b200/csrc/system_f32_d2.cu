// System<float, 2> and its kernel shapes.
#include "system_impl.cuh"

namespace lms {

template <>
KernelChoice<float> pick_kernel<float, 2, kFwd>(int v)
{
  if (v == 25) return make_choice<float, 2, kFwd, 4, 4, 3, true, 2, true, false, false, true, true>("fwd_f32x2_d2_r4_j4_b3_u2_tma");
  if (v == 11) return make_choice<float, 2, kFwd, 2, 4, 7, true>("fwd_f32x2_d2_r2_j4");
  return make_choice<float, 2, kFwd, 2, 4, 6, true, 2, true, false, false, true>("fwd_f32x2_d2_r2_j4_b6_u2_tma");
}
template <>
KernelChoice<float> pick_kernel<float, 2, kAdj>(int v)
{
  if (v == 25) return make_choice<float, 2, kAdj, 4, 1, 3, true, 4, false, true, false, true, true>("adj_f32x2_d2_r4_aos_b3_u4");
  return make_choice<float, 2, kAdj, 2, 2, 5, true, 2, false, false, false, true>("adj_f32x2_d2_r2_j2_u2");
}
template <>
KernelChoice<float> pick_kernel<float, 2, kVel>(int)
{
  return make_choice<float, 2, kVel, 4, 2, 4, true>("vel_f32x2_d2_r4_j2");
}

template class System<float, 2>;

}  // namespace lms
