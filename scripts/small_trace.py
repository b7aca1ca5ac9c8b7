"""Phase timeline of the persistent small-problem kernel (CTA 0, globaltimer ns), from a trace build:
   LMS_BUILD_TAG=trace LMS_NVCC_EXTRA=-DLMS_SMALL_TRACE python __graft_entry__.py
   LMS_LIB_PATH=paper_1907_04839_b200/liblmshoot_b200_trace.so python scripts/small_trace.py [n ...]"""
import ctypes
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_1907_04839_b200 import HamiltonianSystem, make_template_points, rng_normals  # noqa: E402

T = 10
for n in [int(v) for v in sys.argv[1:]] or [500, 1000, 2000]:
    for prec in ("f32", "f64"):
        q0 = make_template_points(n, 40.0 * float(np.sqrt(n / 1847.0)))
        target = q0 + 0.5 * rng_normals(1, n * 3).reshape(n, 3)
        x0 = np.ascontiguousarray(((target - q0) / T).ravel())
        s = HamiltonianSystem(1.5, n, 3, prec, max_timesteps=T)
        s.bind_registration(q0, target, 5e5, T)
        for _ in range(5):
            s.objective(x0)
        tr = np.zeros(8 * 2 * T, dtype=np.uint64)
        s.lib.lms_debug_read_trace.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t]
        s.lib.lms_debug_read_trace(s.handle, tr.ctypes.data, tr.size)
        tr = tr.reshape(2 * T, 8).astype(np.int64)
        # columns: 0 step start, 1 row operands staged, 2 sweep + lane tree done (warp 0), 3 all warps done, 4 epilogue done, 5 barrier passed
        d = np.diff(tr[:, :6], axis=1)
        names = ["rows staged", "sweep", "wait for warps", "epilogue", "barrier"]
        print(f"n={n} {prec}: device {s.last_eval_device_ms()*1e3:.1f} us; kernel span {(tr[-1,4]-tr[0,0])/1e3:.1f} us")
        for half, rows in (("forward", d[:T]), ("adjoint", d[T:])):
            print(f"   {half:8s} " + "  ".join(f"{nm} {np.median(rows[:, k])/1e3:.2f}" for k, nm in enumerate(names)) +
                  f"   | step {np.median(rows.sum(axis=1))/1e3:.2f} us")
        s.close()
