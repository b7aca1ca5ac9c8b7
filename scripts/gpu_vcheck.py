import sys; sys.path.insert(0, ".")
import numpy as np
from oracle import load_oracle
from paper_1907_04839_b200 import HamiltonianSystem
prec, variant = sys.argv[1], int(sys.argv[2])
o = load_oracle(); rng = np.random.default_rng(0)
for n in (7, 257, 600, 1000, 1100, 2300):
    q = rng.uniform(-7, 7, (n, 3)); p = 0.75 * rng.normal(size=(n, 3)); tg = q + 0.5 * rng.normal(size=(n, 3))
    try:
        s = HamiltonianSystem(1.5, n, 3, prec, max_timesteps=5, variant=variant)
        r = s.compute_gradient(q, p, tg, 10.0, 5)
        l, k, m, g = o.compute_gradient(prec, q, p, tg, 1.5, 10.0, 5)
        err = np.abs(r.grad - g).max() / np.abs(g).max()
        bad = np.argwhere(np.abs(r.grad - g).max(axis=1) > 1e-4 * np.abs(g).max()).ravel()
        print(n, "err", err, "loss", r.loss, l, "bad rows", bad[:10], len(bad))
        s.close()
    except Exception as e:
        print(n, "EXC", repr(e))
