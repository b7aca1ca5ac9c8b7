"""World-size-2 CPU test (gloo) of the row-partitioned evaluation's host logic.

The product runs the partition inside liblmshoot_b200.so over NCCL (csrc/system.cu: enqueue_eval +
all_gather_state).  Here the same schedule -- which slices are exchanged after which step, with the
library's own partition arithmetic (lms_row_partition) and its in-place equal-slice all-gather layout --
is replayed on two CPU processes with the oracle's per-row sums standing in for the kernels, and must
reproduce the unsharded oracle bit for bit (a row's sum does not depend on who owns the row)."""
import os
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SIGMA = 1.5


def _all_gather_inplace(plane, slice_rows, rank, world):
    """ncclAllGather(sendbuff = plane + rank*slice, recvbuff = plane, count = slice): the in-place layout."""
    send = torch.from_numpy(np.ascontiguousarray(plane[rank * slice_rows:(rank + 1) * slice_rows]))
    recv = [torch.empty_like(send) for _ in range(world)]
    dist.all_gather(recv, send)
    for r in range(world):
        plane[r * slice_rows:(r + 1) * slice_rows] = recv[r].numpy()


def _worker(rank, world, port, prec, n, T, lam, q0, p0, target, out_dir):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import load_oracle
        from paper_1907_04839_b200 import row_partition

        oracle = load_oracle()
        t = np.float32 if prec == "f32" else np.float64
        slice_rows, stride, lo, hi = row_partition(n, world, rank)
        rows = np.arange(lo, hi)
        d = q0.shape[1]

        def padded(a):  # planes are zero-padded to `stride` rows (row-major here; the layout is per row)
            buf = np.zeros((stride, d), dtype=t)
            buf[:n] = a.astype(t)
            return buf

        dt = t(1.0 / T)
        traj_q, traj_p = [padded(q0)], [padded(p0)]
        h_part = np.zeros(world)
        for step in range(T):
            q, p = traj_q[-1], traj_p[-1]
            hq, hp = oracle.pair_rows(prec, q[:n], p[:n], rows, SIGMA)
            qn, pn = np.zeros_like(q), np.zeros_like(p)
            qn[lo:hi] = q[lo:hi] + dt * hp.astype(t)
            pn[lo:hi] = p[lo:hi] - dt * hq.astype(t)
            if step == 0:
                hp0 = hp.astype(t)
                h_part[rank] = float((p[lo:hi].astype(np.float64) * hp0.astype(np.float64)).sum())
            _all_gather_inplace(qn, slice_rows, rank, world)  # all_gather_state(snapshot(t + 1))
            _all_gather_inplace(pn, slice_rows, rank, world)
            traj_q.append(qn)
            traj_p.append(pn)
        tg = padded(target)
        mm_part = np.zeros(world)
        mm_part[rank] = float(((traj_q[-1][lo:hi].astype(np.float64) - tg[lo:hi].astype(np.float64)) ** 2).sum())
        for part in (h_part, mm_part):  # all_gather_doubles: every rank sums the partials in rank order
            tt = torch.from_numpy(part.copy())
            gathered = [torch.empty_like(tt) for _ in range(world)]
            dist.all_gather(gathered, tt)
            part[:] = [float(gathered[r][r]) for r in range(world)]
        kinetic = 0.5 * float(sum(h_part))
        mismatch = float(sum(mm_part))
        alpha, beta = np.zeros((stride, d), dtype=t), np.zeros((stride, d), dtype=t)
        alpha[lo:hi] = (t(2) * t(lam)) * (traj_q[-1][lo:hi] - tg[lo:hi])
        _all_gather_inplace(alpha, slice_rows, rank, world)  # all_gather_state(adj_[0]) after the last forward step
        _all_gather_inplace(beta, slice_rows, rank, world)
        for step in range(T - 1, -1, -1):
            da, db = oracle.pair_rows(prec, traj_q[step][:n], traj_p[step][:n], rows, SIGMA, alpha[:n], beta[:n])
            an, bn = np.zeros_like(alpha), np.zeros_like(beta)
            an[lo:hi] = alpha[lo:hi] + dt * da.astype(t)
            bn[lo:hi] = beta[lo:hi] + dt * db.astype(t)
            if step > 0:
                _all_gather_inplace(an, slice_rows, rank, world)
                _all_gather_inplace(bn, slice_rows, rank, world)
            alpha, beta = an, bn
        grad = np.zeros((stride, d))
        grad[lo:hi] = (beta[lo:hi] + hp0).astype(np.float64)
        _all_gather_inplace(grad, slice_rows, rank, world)  # the final gradient all-gather
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), grad=grad[:n], scalars=np.array([kinetic + lam * mismatch,
                 kinetic, mismatch]), final_q=traj_q[-1][:n].astype(np.float64))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_row_partitioned_schedule_world2(tmp_path, oracle, prec):
    n, T, lam, world = 700, 3, 10.0, 2
    rng = np.random.default_rng(5)
    q0 = rng.uniform(-6, 6, (n, 3))
    p0 = 0.75 * rng.normal(size=(n, 3))
    target = q0 + 0.5 * rng.normal(size=(n, 3))
    port = 29500 + (os.getpid() % 2000) + (0 if prec == "f64" else 1)
    mp.spawn(_worker, args=(world, port, prec, n, T, lam, q0, p0, target, str(tmp_path)), nprocs=world, join=True)
    loss, kin, mm, grad = oracle.compute_gradient(prec, q0, p0, target, SIGMA, lam, T)
    final_q = oracle.integrate_forward(prec, q0, p0, SIGMA, T)[0][-1]
    for rank in range(world):
        got = np.load(tmp_path / f"rank{rank}.npz")
        assert np.array_equal(got["grad"], grad)          # every rank ends with the full, identical gradient
        assert np.array_equal(got["final_q"], final_q)
        tol = 1e-12 if prec == "f64" else 1e-6            # H = 1/2 sum p.hp vs the reference's pairwise double sum
        assert got["scalars"][0] == pytest.approx(loss, rel=tol)
        assert got["scalars"][1] == pytest.approx(kin, rel=tol)
        assert got["scalars"][2] == pytest.approx(mm, rel=1e-13)


def test_row_partition_covers_rows_once():
    from paper_1907_04839_b200 import row_partition

    for n in (0, 1, 511, 512, 513, 20000, 200000, 1000003):
        for world in (1, 2, 3, 4, 8):
            parts = [row_partition(n, world, r) for r in range(world)]
            slices = {p[0] for p in parts}
            assert len(slices) == 1 and parts[0][0] % 512 == 0        # equal, tile-aligned slices
            assert all(p[1] == parts[0][0] * world for p in parts)    # one padded plane length everywhere
            assert parts[0][2] == 0 and parts[-1][3] == n
            for a, b in zip(parts, parts[1:]):
                assert a[3] == b[2]                                   # contiguous, no gaps or overlaps
            assert all(p[3] - p[2] <= p[0] for p in parts)
    with pytest.raises(ValueError):
        row_partition(10, 2, 2)
