// System<float, 3>: the headline instantiation (BASELINE configs[1-4]) and its kernel shapes.
#include "system_impl.cuh"

// the two-row default shapes also come with a thin-tile instantiation (N = 10 000: 2.268 -> 2.216 ms per gradient);
// -DLMS_R2_THIN=false leaves it out
#ifndef LMS_R2_THIN
#define LMS_R2_THIN true
#endif

namespace lms {

// (R rows per thread, JU columns per shared-memory vector load, min CTAs/SM for __launch_bounds__).
// Variant 0 is the default the library ships with; the rest are kept for on-GPU A/B (bench.py --variant).
//   default   forward R=2, 4 columns per LDS.128, column loop unrolled x2, tiles staged by bulk-async copies (TMA,
//             cp.async.bulk + mbarrier), 80 registers (6 CTAs/SM); adjoint R=2, 2 columns per load, unrolled x2,
//             register-staged tiles, 96 registers (5 CTAs/SM)
//   25        forward R=4, same loop, 168 registers (3 CTAs/SM); adjoint R=4 with column-major tiles (LDS.128);
//             variant 0 maps to it from N = 16 000 on (see pick_kernels)
//   1         scalar-FFMA kernels (the first version);   11   the R=2 shapes, register-staged forward tiles
// Shapes measured in round 1 and dropped from the build (numbers per launch at N = 20 000, one session, ms):
//   forward R=4: j4 0.2584 | j2_u2 0.2508 | j4_u2 0.2500 | j4_u2_tma 0.2468 (kept) | j4_u4 0.2554 | j2_u4 0.2589;
//   adjoint R=4: aos_u4 0.5536 (kept) | aos_u2 0.5660 | j4_tma 0.5558 | j2_u2_tma 0.5633 | j2_tma 0.5661;
//   R=6 / R=8: 0.8 % faster per pair, lost to row-tile quantisation.  Round 2, R=6 again with the current
//   loops (forward u2 + TMA at 246 registers, adjoint column-major u4 at 240, 2 CTAs/SM) and the thin last tile, ms per
//   gradient R=4 / R=6: N = 20 000 7.841 / 7.950, 50 000 47.29 / 47.54, 100 000 188.4 / 188.9 -- no longer ahead.
template <>
KernelChoice<float> pick_kernel<float, 3, kFwd>(int v)
{
  switch (v) {
    case 1: return make_choice<float, 3, kFwd, 4, 4, 3>("fwd_f32_r4_j4");
    case 11: return make_choice<float, 3, kFwd, 2, 4, 7, true>("fwd_f32x2_r2_j4_b7");
    case 25: return make_choice<float, 3, kFwd, 4, 4, 3, true, 2, true, false, false, true, true>("fwd_f32x2_r4_j4_b3_u2_tma");
    default: return make_choice<float, 3, kFwd, 2, 4, 6, true, 2, true, false, true, true, LMS_R2_THIN>("fwd_f32x2_r2_j4_b6_u2_tma");
  }
}
template <>
KernelChoice<float> pick_kernel<float, 3, kAdj>(int v)
{
  switch (v) {
    case 1: return make_choice<float, 3, kAdj, 2, 4, 3>("adj_f32_r2_j4");
    case 25: return make_choice<float, 3, kAdj, 4, 1, 3, true, 4, false, true, false, true, true>("adj_f32x2_r4_aos_b3_u4");
    default: return make_choice<float, 3, kAdj, 2, 2, 5, true, 2, false, false, true, true, LMS_R2_THIN>("adj_f32x2_r2_j2_b5_u2");
  }
}
template <>
KernelChoice<float> pick_kernel<float, 3, kVel>(int v)
{
  if (v == 1) return make_choice<float, 3, kVel, 4, 4, 4>("vel_f32_r4_j4");
  return make_choice<float, 3, kVel, 4, 2, 4, true>("vel_f32x2_r4_j2");
}

template class System<float, 3>;

}  // namespace lms
