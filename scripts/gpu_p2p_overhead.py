"""Upper bound on the cost of the row-partition exchanges, measured on ONE GPU: `world` ranks as threads of one
process share the device, so a partitioned evaluation does the same total pair work as an unpartitioned one;
whatever it takes longer is exchange + scheduling overhead.  Transports: peer-push (p2p) and loopback."""
import sys, threading, time
import numpy as np
sys.path.insert(0, ".")
from paper_1907_04839_b200 import HamiltonianSystem, LocalGroup, make_template_points, rng_normals

n, T, prec = int(sys.argv[1]) if len(sys.argv) > 1 else 20000, 10, "f32"
q0 = make_template_points(n, 40.0 * float(np.sqrt(n / 1847.0)))
target = q0 + 0.5 * rng_normals(1, n * 3).reshape(n, 3)
x0 = np.ascontiguousarray(((target - q0) / T).ravel())
plain = HamiltonianSystem(1.5, n, 3, prec, max_timesteps=T)
plain.bind_registration(q0, target, 5e5, T)
for _ in range(3):
    plain.objective(x0)
t0 = time.perf_counter()
for _ in range(10):
    plain.objective(x0)
base = (time.perf_counter() - t0) * 100
print(f"N={n} unpartitioned: {base:.3f} ms wall per evaluation")
plain.close()
for transport in ("p2p", "loopback"):
    for world in (2, 4):
        ranks = [HamiltonianSystem(1.5, n, 3, prec, max_timesteps=T) for _ in range(world)]
        blobs = [None] * world
        meet = threading.Barrier(world)
        group = LocalGroup(world) if transport == "loopback" else None
        times = [0.0] * world

        def run(r):
            s = ranks[r]
            if transport == "p2p":
                blobs[r] = s.p2p_export(r, world)
                meet.wait()
                s.p2p_connect(blobs)
            else:
                s.join_local_group(group, r)
            s.bind_registration(q0, target, 5e5, T)
            meet.wait()
            for _ in range(3):
                s.objective(x0)
            meet.wait()
            t0 = time.perf_counter()
            for _ in range(10):
                s.objective(x0)
            times[r] = (time.perf_counter() - t0) * 100

        th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
        [t.start() for t in th]
        [t.join() for t in th]
        print(f"  {transport:8s} world={world}: {max(times):.3f} ms wall per evaluation ({max(times) / base:.3f}x)")
        for s in ranks:
            s.close()
        if group:
            group.close()
