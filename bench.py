#!/usr/bin/env python
"""bench.py -- the hot path's headline metric on B200 (BASELINE.json).

  metric   pairwise kernel evaluations per second for one fwd+bwd gradient (2*T*N^2 units per gradient,
           the algorithmic count of SURVEY.md §8d), plus ms per L-BFGS iteration in `lbfgs`
  step     one objective evaluation (forward flow + loss + adjoint sweep) = lmshoot::Objective::operator()
  N = 1    BASELINE.json configs[1]: N = 20 000 landmarks, T = 10, fp32 (fp64 reported beside it)
  N > 1    configs[2]: one registration of N = 200 000, T = 20, row-partitioned with a per-step NCCL
           all-gather of (q,p) / (alpha,beta)  (--mode rows, strong scaling), or independent replicas
           of configs[1] (--mode replicas, weak scaling)

`value` times the evaluation with x / grad resident in HBM (CUDA events on the library's stream, summed
over the K steps); `e2e` times the same call through the host-buffer C ABI (lms_objective_eval) with
pinned host x / grad, H2D + D2H inside the timed region.  `--impl reference` times the reference's own
CPU implementation (oracle/_ref, compiled from /root/reference where that exists, else the oracle port).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

SIGMA, LAMBDA = 1.5, 5e5  # shooting.hpp:26-28
FWD_SLOTS, ADJ_SLOTS = 18, 43  # FP32 lane-instructions per pair, SURVEY.md §8d (fp64: 35 / 60)
FWD_SLOTS_F64, ADJ_SLOTS_F64 = 35, 60
# lane-instructions the kernels actually execute per pair, MUFU/exp included (profiles/r2_sass_*.md)
FWD_EXEC, ADJ_EXEC = 18, 40
FWD_EXEC_F64, ADJ_EXEC_F64 = 28, 50
# CPU legs.  `--impl reference` runs the reference's compute_gradient on the SAME configuration our arm prints
# (N = 20 000, T = 10: (2T+2) N^2 = 8.8e9 pair evaluations, ~10 s per gradient on 16 host threads) and caps the number
# of timed steps by wall clock instead of shrinking N; only configs[2] (N = 200 000, T = 20: ~30 min per gradient)
# is sampled, and then `config.n` carries the N actually run.  The in-line `cpu_baseline` of the B200 arm is a
# bounded sample (N = 6000, same generator and density, ~1 s per gradient).
CPU_SAMPLE_N = 6000
REF_ROWS_SAMPLE_N = 20000      # reference arm, rows mode: the sample of the N = 200 000 workload
REF_BUDGET_S = 90.0            # reference arm: wall-clock budget for the timed steps


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--precision", default="f32", choices=["f32", "f64"])
    ap.add_argument("--landmarks", "--n", dest="n", type=int, default=0, help="landmarks (default: 20000 at 1 GPU, 200000 at >1)")
    ap.add_argument("--timesteps", type=int, default=0)
    ap.add_argument("--variant", type=int, default=0)
    ap.add_argument("--mode", default="rows", choices=["rows", "replicas"])
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "p2p"],
                    help="rows mode: per-step NCCL all-gather, or peer stores from the kernel epilogues + stream flags")
    ap.add_argument("--batch", type=int, default=0, help="population mode: B registrations of --n landmarks per GPU")
    ap.add_argument("--no-extras", action="store_true", help="skip fp64, L-BFGS and cpu_baseline legs")
    ap.add_argument("--lbfgs-iters", type=int, default=30)
    ap.add_argument("--fixed-extent", action="store_true",
                    help="template on the fixed 40 mm sphere (synth.hpp:20) instead of constant landmark density")
    ap.add_argument("--launch-check", action="store_true",
                    help="start the ranks exactly as a measurement would, report who showed up, measure nothing")
    return ap.parse_args()


def self_launch(args):
    """`python bench.py --gpus N` outside torchrun: start the N ranks ourselves, the way the driver does
    (python -m torch.distributed.run --nnodes=1 --nproc-per-node N --master-addr 127.0.0.1 ...)."""
    import socket
    import subprocess

    with socket.socket() as sock:
        sock.bind(("127.0.0.1", 0))
        port = sock.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def init_ranks():
    """Rank / device / process group from the torchrun environment.  More ranks than visible GPUs (a one-GPU box
    running a two-rank check) share devices round-robin: the control plane then runs over gloo and the data path over
    the peer-push exchange (CUDA IPC), because NCCL refuses two ranks on one device."""
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    ndev = torch.cuda.device_count() if torch.cuda.is_available() else 0
    device = local_rank % ndev if ndev else -1
    oversub = ndev > 0 and world > ndev
    backend = "nccl" if (ndev and not oversub) else "gloo"
    if ndev:
        torch.cuda.set_device(device)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", device))
        else:
            dist.init_process_group("gloo")
    return world, rank, device, oversub, backend


def launch_check(args):
    import torch.distributed as dist

    world, rank, device, oversub, backend = init_ranks()
    seen = [None] * world
    if world > 1:
        dist.all_gather_object(seen, {"rank": rank, "pid": os.getpid(), "device": device})
        dist.destroy_process_group()
    else:
        seen = [{"rank": rank, "pid": os.getpid(), "device": device}]
    if rank == 0:
        print(json.dumps({"launch_check": True, "n_gpus": world, "requested": args.gpus, "backend": backend,
                          "oversubscribed": oversub, "ranks": seen}), flush=True)


# ---- clocks -----------------------------------------------------------------------------------------
class ClockSampler(threading.Thread):
    """Samples SM clock and throttle reasons during the timed region (nvidia-smi's counters via NVML)."""

    def __init__(self, index):
        super().__init__(daemon=True)
        self.index, self.samples, self.reasons, self.stop_flag = index, [], set(), threading.Event()
        self.max_mhz = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def run(self):
        if self.nv is None:
            return
        nv = self.nv
        names = {
            nv.nvmlClocksThrottleReasonHwSlowdown: "hw_slowdown",
            nv.nvmlClocksThrottleReasonHwThermalSlowdown: "hw_thermal_slowdown",
            nv.nvmlClocksThrottleReasonSwThermalSlowdown: "sw_thermal_slowdown",
            nv.nvmlClocksThrottleReasonSwPowerCap: "sw_power_cap",
        }
        while not self.stop_flag.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                mask = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for bit, name in names.items():
                    if mask & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            self.stop_flag.wait(0.05)

    def result(self):
        self.stop_flag.set()
        if self.is_alive():
            self.join(timeout=1.0)
        s = sorted(self.samples)
        return {"sm_mhz": s[len(s) // 2] if s else None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(s)}


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            return json.load(f), "measured"
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


def measured_traffic(mode, prec):
    """DRAM bytes per launch of the forward / adjoint pair kernel from the committed `ncu --set full` capture
    (profiles/*_traffic.json, written by scripts/summarize_profiles.py); None when no capture is committed."""
    import glob

    best = None
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "*_traffic.json"))):
        with open(path) as f:
            doc = json.load(f)
        for name, val in doc.get("kernels", {}).items():
            if f",{mode}," in name and name.startswith("pair_kernel<" + ("float" if prec == "f32" else "double")):
                best = {"bytes_per_launch": val, "source": doc.get("source")}
    return best


def ffma_peak_lanes():
    """Measured FP32 lane-ops/SM/clk from profiles/ubench (None until a GPU run committed it)."""
    path = os.path.join(ROOT, "profiles", "ubench", "pipes_b200.json")
    if not os.path.exists(path):
        return None
    with open(path) as f:
        res = {r["name"]: r for r in json.load(f)["results"]}
    return res


# ---- the reference arm ------------------------------------------------------------------------------------
def template_label(fixed_extent):
    return ("Fibonacci sphere, fixed 40 mm diameter (synth.hpp:20)" if fixed_extent else
            "Fibonacci sphere, radius 20*sqrt(N/1847) mm (constant landmark density)")


def cpu_workload(n, timesteps, fixed_extent, cpu, oracle):
    """The GPU arm's generator, host-only: Fibonacci sphere, Rng(0) momenta, target = fp64 flow of the template
    (synth.hpp:40-43), x0 = (target - q0)/T (registration.cpp:47-52)."""
    import numpy as np

    golden = np.pi * (3.0 - np.sqrt(5.0))
    i = np.arange(n, dtype=np.float64)
    z = 1.0 - 2.0 * (i + 0.5) / n
    r = np.sqrt(np.maximum(0.0, 1.0 - z * z))
    radius = 20.0 if fixed_extent else 20.0 * np.sqrt(n / 1847.0)
    q0 = np.stack([radius * r * np.cos(golden * i), radius * r * np.sin(golden * i), radius * z], axis=1)
    p_true = (0.75 * oracle.rng_normals(0, n * 3)).reshape(n, 3)
    target = cpu.integrate_forward("f64", q0, p_true, SIGMA, timesteps)[0][-1]
    return q0, target, (target - q0) / timesteps


def cpu_reference_run(n_run, timesteps, precision, steps, warmup, fixed_extent=False, budget_s=None, n_workload=None):
    """Times the reference's compute_gradient (shooting.hpp:277-315) on all host threads.  With a wall-clock budget
    the first gradient is the warm-up and sets how many timed steps fit (at least 2, at most `steps`)."""
    from oracle import load_oracle, load_reference, reference_available

    kind = "reference" if reference_available() else "port"
    cpu = load_reference() if kind == "reference" else load_oracle()
    cores = cpu.hardware_threads()
    q0, target, x0 = cpu_workload(n_run, timesteps, fixed_extent, cpu, load_oracle())

    def one():
        t0 = time.perf_counter()
        cpu.compute_gradient(precision, q0, x0, target, SIGMA, LAMBDA, timesteps)
        return time.perf_counter() - t0

    first = one()
    if budget_s is not None and first * (steps + warmup) > budget_s:
        warmup_run, steps_run = 1, max(2, min(steps, int(budget_s / first)))
    else:
        warmup_run, steps_run = max(warmup, 1), steps
    for _ in range(warmup_run - 1):
        one()
    times = [one() for _ in range(steps_run)]
    sec = sum(times) / len(times)
    units = 2.0 * timesteps * n_run * n_run
    full = n_workload is None or n_workload == n_run
    return {
        "value": units / sec, "sec_per_gradient": sec, "cores": cores, "kind": kind,
        "steps_run": steps_run, "warmup_run": warmup_run, "n_run": n_run,
        "sample": (f"{'the full workload' if full else f'a sample of the N={n_workload} workload'}: compute_gradient at "
                   f"N={n_run}, T={timesteps}, {precision}, blocked_tree/256, {cores} threads, {steps_run} timed "
                   f"gradients after {warmup_run} warm-up; same generator, "
                   f"{'fixed 40 mm sphere' if fixed_extent else 'same landmark density'}; units counted as 2*T*N^2"),
    }


def reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    rows_mode = args.gpus > 1 and args.mode == "rows"  # the workload our own arm measures at this --gpus
    T = args.timesteps or (20 if rows_mode else 10)
    n_workload = args.n or (200000 if rows_mode else 20000)
    # configs[1] runs in full; one N = 200 000, T = 20 gradient is ~30 min of 16 host threads, so configs[2] is
    # sampled at N = 20 000 (same density, same T) and config.n says so
    n_run = min(n_workload, REF_ROWS_SAMPLE_N) if rows_mode else n_workload
    res = cpu_reference_run(n_run, T, args.precision, max(args.steps, 1), max(args.warmup, 0),
                            fixed_extent=args.fixed_extent, budget_s=REF_BUDGET_S, n_workload=n_workload)
    line = {
        "impl": "reference", "metric": "pair_kernel_evals_per_sec_per_gradient", "value": res["value"],
        "unit": "pair-evals/s", "n_gpus": args.gpus, "steps": res["steps_run"], "warmup": res["warmup_run"],
        "steps_requested": args.steps, "warmup_requested": args.warmup,
        "ms_per_step": res["sec_per_gradient"] * 1e3, "higher_is_better": True,
        "scaling": "strong" if rows_mode else "weak",
        "vs_baseline": None, "dtype": args.precision, "data": "synthetic",
        "config": {"workload": (f"single registration N={n_workload}, T={T}, row-partitioned over {args.gpus} GPUs"
                                if rows_mode else
                                f"single registration N={n_workload}, T={T}, one fwd+bwd gradient per step"
                                + (f", {args.gpus} independent replicas" if args.gpus > 1 else "")),
                   "n": n_run, "n_workload": n_workload,
                   "timesteps": T, "sigma": SIGMA, "lambda": LAMBDA, "units_per_step": "2*T*N^2",
                   "template": template_label(args.fixed_extent), "sample": res["sample"]},
        "cpu_baseline": {"value": res["value"], "unit": "pair-evals/s", "cores": res["cores"], "kind": res["kind"],
                         "sample": res["sample"]},
        "e2e": {"value": res["value"], "unit": "pair-evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    if not rows_mode and not args.fixed_extent and not args.no_extras and n_workload <= 20000:
        # the CPU's exp cost depends on the data (glibc expf's underflow path), so the fixed-diameter
        # sphere is timed beside the constant-density one (one warm-up + two gradients)
        fx = cpu_reference_run(n_run, T, args.precision, 2, 1, fixed_extent=True, budget_s=30.0, n_workload=n_workload)
        line["fixed_extent_40mm"] = {"value": fx["value"], "ms_per_step": fx["sec_per_gradient"] * 1e3,
                                     "sample": fx["sample"]}
    print(json.dumps(line), flush=True)


# ---- the B200 arm ------------------------------------------------------------------------------------------
def nccl_log_summary(path_glob):
    """The communicator lines of NCCL's own log (NCCL_DEBUG=INFO, NCCL_DEBUG_SUBSYS=INIT,GRAPH to a file): version,
    ranks, whether the NVLink-SHARP (NVLS) multicast path came up, channel count."""
    import glob
    import re

    lines = []
    for path in sorted(glob.glob(path_glob)):
        try:
            with open(path, errors="replace") as f:
                lines += f.read().splitlines()
        except OSError:
            pass
    if not lines:
        return None
    pick = [ln.strip() for ln in lines if re.search(r"NCCL version|nranks|NVLS|Connected all|comm 0x\w+ rank|Channel \d+/\d+ :", ln)]
    return {"nvls": any("NVLS" in ln and "disabled" not in ln.lower() for ln in lines), "log_lines": len(lines),
            "excerpt": pick[:12]}


def b200_arm(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    if int(os.environ.get("WORLD_SIZE", "1")) > 1 and args.mode == "rows" and args.exchange == "nccl":
        # keep NCCL's communicator log (one file per rank under gpurun_out/, summarised in the JSON line)
        os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT,GRAPH")
        os.environ.setdefault("NCCL_DEBUG_FILE", os.path.join(ROOT, "gpurun_out", "nccl_%h_%p.log"))

    from paper_1907_04839_b200 import HamiltonianSystem, comm_unique_id, make_synthetic_pair

    world, rank, device, oversub, backend = init_ranks()
    distributed = world > 1

    def barrier():
        if distributed:
            dist.barrier()
        torch.cuda.synchronize()

    rows_mode = distributed and args.mode == "rows"
    exchange = "p2p" if (rows_mode and oversub) else args.exchange
    n = args.n or (200000 if rows_mode else 20000)
    T = args.timesteps or (20 if rows_mode else 10)
    prec = args.precision
    K, W = max(args.steps, 1), max(args.warmup, 3)

    # ---- workload (synthetic) ----
    # Template radius grows with sqrt(N/1847) so the landmark density is that of the reference's default
    # problem (synth.hpp:19-20: 1847 points on a 40 mm sphere).  At fixed 40 mm diameter N = 20 000 packs
    # 4 landmarks/mm^2 against sigma = 1.5 mm and the flow turns chaotic (|target - q0| up to 1.2 m, loss
    # 1e16, fp32 and fp64 differ by 0.6 %): not a meaningful evaluation point, so it is timed as an extra
    # (`fixed_extent_40mm`, or the whole run with --fixed-extent).  GPU time is data-independent.
    q0, target, _ = make_synthetic_pair(n, SIGMA, T, seed=0 if rows_mode else rank, device=device,
                                        density_scaled=not args.fixed_extent)
    x0 = np.ascontiguousarray(((target - q0) / T).ravel())

    system = HamiltonianSystem(SIGMA, n, 3, prec, device=device, max_timesteps=T, variant=args.variant)
    if rows_mode and exchange == "p2p":
        blobs = [None] * world
        dist.all_gather_object(blobs, system.p2p_export(rank, world))
        system.p2p_connect(blobs)
    elif rows_mode:
        uid = [comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        system.comm_init(uid[0], rank, world)
    system.bind_registration(q0, target, LAMBDA, T)
    if distributed:
        dist.barrier()  # nobody's first step may store into a peer that is still binding

    d_x = torch.from_numpy(x0).cuda()
    d_grad = torch.empty_like(d_x)
    h_x = torch.from_numpy(x0).pin_memory()
    h_grad = torch.empty_like(h_x).pin_memory()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2

    def flush_l2():
        flush.fill_(1)
        torch.cuda.synchronize()

    def timed_pass(device_buffers):
        """K steps; returns (sum of device-event ms, sum of host wall ms) over the steps."""
        dev_ms = wall_ms = 0.0
        for _ in range(K):
            flush_l2()
            if rows_mode:
                dist.barrier()  # the ranks enter every step together, as one job would
            t0 = time.perf_counter()
            if device_buffers:
                system.objective_ptrs(d_x.data_ptr(), d_grad.data_ptr(), device=True)
            else:
                system.objective_ptrs(h_x.data_ptr(), h_grad.data_ptr(), device=False)
            wall_ms += (time.perf_counter() - t0) * 1e3
            dev_ms += system.last_eval_device_ms()
        return dev_ms, wall_ms

    for _ in range(W):
        system.objective_ptrs(d_x.data_ptr(), d_grad.data_ptr(), device=True)
        system.objective_ptrs(h_x.data_ptr(), h_grad.data_ptr(), device=False)
    launches_per_step = system.last_eval_kernel_launches()

    sampler = ClockSampler(device)
    sampler.start()
    barrier()
    dev_ms, wall_dev = timed_pass(True)
    barrier()
    clocks = sampler.result()
    barrier()
    _, wall_host = timed_pass(False)
    barrier()

    def max_over_ranks(v):
        if not distributed:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cuda" if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    my_dev_ms = dev_ms
    dev_ms = max_over_ranks(dev_ms)
    wall_host = max_over_ranks(wall_host)
    units_per_step = 2.0 * T * float(n) * float(n)
    jobs = 1 if (rows_mode or not distributed) else world  # replicas: every rank runs its own registration
    value = jobs * units_per_step * K / (dev_ms * 1e-3)
    e2e_value = jobs * units_per_step * K / (wall_host * 1e-3)

    line = {
        "metric": "pair_kernel_evals_per_sec_per_gradient", "value": value, "unit": "pair-evals/s",
        "n_gpus": world, "steps": K, "warmup": W, "ms_per_step": dev_ms / K, "higher_is_better": True,
        "scaling": "strong" if rows_mode else "weak", "vs_baseline": None, "dtype": prec, "data": "synthetic",
        "config": {
            "workload": (f"single registration N={n}, T={T}, row-partitioned over {world} GPUs, per-step "
                         + ("NCCL all-gather" if exchange == "nccl" else "peer-push exchange (P2P stores + flags)")
                         if rows_mode else
                         f"single registration N={n}, T={T}, one fwd+bwd gradient per step"
                         + (f", {world} independent replicas" if distributed else "")),
            "n": n, "timesteps": T, "sigma": SIGMA, "lambda": LAMBDA, "units_per_step": "2*T*N^2",
            "template": template_label(args.fixed_extent),
            "l2": "flushed between timed steps (256 MiB write)", "variant": args.variant,
            "kernel_variant": system.lib.lms_system_kernel_names(system.handle).decode(),
        },
        "e2e": {"value": e2e_value, "unit": "pair-evals/s", "h2d_bytes_per_step": int(x0.nbytes),
                "d2h_bytes_per_step": int(x0.nbytes) + 32, "ms_per_step": wall_host / K},
        "gpu_launches": launches_per_step * K * 2,  # both timed passes
        "clocks": clocks,
        "wall_ms_per_step_device_buffers": wall_dev / K,
    }
    if oversub:
        line["config"]["oversubscribed"] = (f"{world} ranks share {torch.cuda.device_count()} GPU(s): a launcher / "
                                            "exchange check, not a scaling measurement")

    # ---- per-launch kernel times of every rank (events around each pair-kernel launch; separate timed pass) ----
    system.set_kernel_timing(True)
    fwd_ms = adj_ms = step_ms = 0.0
    for _ in range(K):
        flush_l2()
        if rows_mode:
            dist.barrier()
        system.objective_ptrs(d_x.data_ptr(), d_grad.data_ptr(), device=True)
        fwd_ms += system.last_kernel_ms("forward")
        adj_ms += system.last_kernel_ms("adjoint")
        step_ms += system.last_eval_device_ms()
    system.set_kernel_timing(False)
    fwd_ms /= K
    adj_ms /= K
    step_ms /= K
    if rows_mode:
        # what is left of a step after its 2T pair-kernel launches: the exchanges (all-gathers or flag waits,
        # including the time spent waiting for the slowest rank) plus the O(N) kernels
        mine = {"rank": rank, "ms_per_step": my_dev_ms / K, "forward_launch_ms": fwd_ms, "adjoint_launch_ms": adj_ms,
                "pair_kernels_ms_per_step": (fwd_ms + adj_ms) * T,
                "exchange_and_wait_ms_per_step": step_ms - (fwd_ms + adj_ms) * T}
        per_rank = [None] * world
        dist.all_gather_object(per_rank, mine)
        line["per_rank"] = per_rank
        if exchange == "nccl" and rank == 0:
            line["nccl"] = nccl_log_summary(os.path.join(ROOT, "gpurun_out", "nccl_*.log"))

    # ---- roofline of the dominant kernel (adjoint pair kernel), from the per-launch events above ----
    if rank == 0:
        peaks, peaks_src = measured_peaks()
        rows_share = 1.0 / world if rows_mode else 1.0
        pairs_per_launch = float(n) * float(n) * rows_share
        f_slots, a_slots = (FWD_SLOTS, ADJ_SLOTS) if prec == "f32" else (FWD_SLOTS_F64, ADJ_SLOTS_F64)
        f_exec, a_exec = (FWD_EXEC, ADJ_EXEC) if prec == "f32" else (FWD_EXEC_F64, ADJ_EXEC_F64)
        lanes = 128 if prec == "f32" else 64
        sm_mhz = float(peaks.get("sm_max_mhz", 1965.0))
        peak_slots = 148 * lanes * sm_mhz * 1e6
        adj_rate = a_slots * pairs_per_launch / (adj_ms * 1e-3)
        fwd_rate = f_slots * pairs_per_launch / (fwd_ms * 1e-3)
        grad_rate = (f_slots + a_slots) * T * pairs_per_launch / ((fwd_ms + adj_ms) * T * 1e-3)
        bytes_per_launch = (3 * 12 + 12) * n * (4 if prec == "f32" else 8)  # read q,p,a,b rows+cols, write a,b
        line["roofline"] = {
            "bound": "fp32_cuda_core" if prec == "f32" else "fp64_cuda_core",
            "kernel": "adjoint pair kernel (adjoint_step + Euler-adjoint epilogue)",
            "achieved": adj_rate / 1e12, "peak": peak_slots / 1e12, "unit": "Tslot/s (FP lane-instructions)",
            "frac": adj_rate / peak_slots,
            "peak_source": f"148 SM x {lanes} lanes x sm_max_mhz {sm_mhz:.0f} MHz ({peaks_src} MEASURED_PEAKS.json)",
            "algorithmic_slots_per_pair": a_slots, "pairs_per_launch": pairs_per_launch,
            "avg_launch_ms": adj_ms,
            # the contract counts 43 / 18 (fp64 60 / 35) slots per pair; the kernels EXECUTE fewer (hand-fused terms,
            # branch-free exp): this is the pipe utilisation by executed lane-instructions (cf. ncu's pipe counters)
            "executed_slots_per_pair": a_exec, "frac_executed": a_exec * pairs_per_launch / (adj_ms * 1e-3) / peak_slots,
            "traffic": (measured_traffic("adj", prec) or {}).get("bytes_per_launch") if n == 20000 and T == 10 else None,
            "traffic_source": (measured_traffic("adj", prec) or {}).get("source"),
            "forward_kernel": {"avg_launch_ms": fwd_ms, "achieved": fwd_rate / 1e12, "frac": fwd_rate / peak_slots,
                               "algorithmic_slots_per_pair": f_slots, "executed_slots_per_pair": f_exec,
                               "frac_executed": f_exec * pairs_per_launch / (fwd_ms * 1e-3) / peak_slots},
            # `frac`: from the separately timed launches of the pass above (events around every launch, no graph);
            # `frac_of_timed_step`: the same slots over the headline step time (one graph launch per gradient)
            "gradient": {"achieved": grad_rate / 1e12, "frac": grad_rate / peak_slots,
                         "slots_per_gradient": (f_slots + a_slots) * T * pairs_per_launch,
                         "frac_of_timed_step": (f_slots + a_slots) * T * pairs_per_launch / (dev_ms / K * 1e-3) / peak_slots},
            "hbm": {"algorithmic_bytes_per_launch": bytes_per_launch,
                    "achieved_gbs": bytes_per_launch / (adj_ms * 1e-3) / 1e9, "peak_gbs": peaks.get("hbm_gbs")},
            "kernel_share_of_step": (fwd_ms + adj_ms) * T / (dev_ms / K),
            # the same launch in flop terms (FMA = 2 flop; 69 flop per adjoint pair, 28 per forward
            # pair) against the all-FMA peak of the pipe: lower than `frac` because only ~60 % of the slots are FMAs
            "flops": {"achieved_tflops": 69 * pairs_per_launch / (adj_ms * 1e-3) / 1e12,
                      "peak_tflops": 2 * peak_slots / 1e12, "flop_per_pair": 69},
        }
        ub = ffma_peak_lanes()
        if ub and prec == "f32" and "ffma" in ub:
            meas = 148 * ub["ffma"]["lane_ops_per_sm_clk"] * ub["ffma"]["sm_mhz"] * 1e6
            line["roofline"]["peak_measured_ffma"] = meas / 1e12
            line["roofline"]["frac_of_measured_ffma"] = adj_rate / meas

    # ---- extras on rank 0 at one GPU: fp64 beside fp32, ms per L-BFGS iteration, CPU baseline ----
    if rank == 0 and not distributed and not args.no_extras:
        def time_steps(sys_, reps):
            for _ in range(2):
                sys_.objective_ptrs(d_x.data_ptr(), d_grad.data_ptr(), device=True)
            ms = 0.0
            for _ in range(reps):
                flush_l2()
                sys_.objective_ptrs(d_x.data_ptr(), d_grad.data_ptr(), device=True)
                ms += sys_.last_eval_device_ms()
            return ms / reps

        if prec == "f32":
            s64 = HamiltonianSystem(SIGMA, n, 3, "f64", device=device, max_timesteps=T, variant=args.variant)
            s64.bind_registration(q0, target, LAMBDA, T)
            ms64 = time_steps(s64, max(3, K // 2))
            slots64 = (FWD_SLOTS_F64 + ADJ_SLOTS_F64) * T * float(n) * float(n)
            exec64 = (FWD_EXEC_F64 + ADJ_EXEC_F64) * T * float(n) * float(n)
            peak64 = 148 * 64 * float(measured_peaks()[0].get("sm_max_mhz", 1965.0)) * 1e6
            line["fp64"] = {"ms_per_step": ms64, "value": units_per_step / (ms64 * 1e-3),
                            "frac_of_fp64_roofline": slots64 / (ms64 * 1e-3) / peak64,
                            "frac_executed": exec64 / (ms64 * 1e-3) / peak64,
                            "note": "contract slots 35/60 per pair; executed DP-pipe ops 28/50 (branch-free exp)"}
            s64.close()
        if not args.fixed_extent:
            # the fixed 40 mm sphere beside the constant-density one (device time is data-independent;
            # the CPU arm's is not)
            fq0, ftarget, _ = make_synthetic_pair(n, SIGMA, T, seed=0, device=device, density_scaled=False)
            sfx = HamiltonianSystem(SIGMA, n, 3, prec, device=device, max_timesteps=T, variant=args.variant)
            sfx.bind_registration(fq0, ftarget, LAMBDA, T)
            keep = d_x.clone()
            d_x.copy_(torch.from_numpy(np.ascontiguousarray(((ftarget - fq0) / T).ravel())))
            msfx = time_steps(sfx, max(3, K // 2))
            d_x.copy_(keep)
            sfx.close()
            line["fixed_extent_40mm"] = {"ms_per_step": msfx, "value": units_per_step / (msfx * 1e-3)}
        # ms per L-BFGS iteration: the whole registration loop through the C ABI (lms_register: host-buffer
        # objective + the library's host L-BFGS driver, no Python inside the loop); every variant is run twice and
        # both runs are reported (the first includes whatever one-time cost is left after binding, which already
        # allocated and warmed the device-resident optimiser's workspace)
        from paper_1907_04839_b200 import ShootingConfig, register_landmarks

        cfg = ShootingConfig(sigma=SIGMA, timesteps=T, lam=LAMBDA, max_iter=args.lbfgs_iters, precision=prec)
        eval_ms = dev_ms / K

        def registration(device_vectors):
            runs = []
            for _ in range(2):
                t0 = time.perf_counter()
                reg = register_landmarks(q0, target, cfg, device=device, system=system, device_vectors=device_vectors,
                                         already_bound=True)
                runs.append((time.perf_counter() - t0) * 1e3)
            # the whole call divided by the accepted iterations: every evaluation of the line searches, the
            # optimiser's vector work and the read-back of q(1) are inside (the re-integration under p0* of
            # registration.cpp:85-93 is skipped when the resident trajectory already is the one of p0*)
            per_iter = [ms / max(reg.iterations, 1) for ms in runs]
            return reg, {"iterations": reg.iterations, "evaluations": reg.evaluations,
                         "ms_per_iteration": per_iter[1], "ms_per_iteration_first_run": per_iter[0],
                         "ms_total": runs[1], "ms_total_first_run": runs[0],
                         "ms_per_iteration_over_ms_per_gradient": per_iter[1] / eval_ms,
                         "final_loss": reg.final_loss, "initial_loss": reg.initial_loss,
                         "avg_dist_before_mm": reg.avg_before, "avg_dist_after_mm": reg.avg_after}

        _, line["lbfgs"] = registration(False)
        _, line["lbfgs_device_vectors"] = registration(True)
        try:
            cpu = cpu_reference_run(CPU_SAMPLE_N, T, prec, 1, 1, fixed_extent=args.fixed_extent, n_workload=n)
            line["cpu_baseline"] = {"value": cpu["value"], "unit": "pair-evals/s", "cores": cpu["cores"],
                                    "kind": cpu["kind"], "sample": cpu["sample"]}
        except Exception as e:  # the oracle is test infrastructure; its absence must not hide the GPU number
            line["cpu_baseline"] = {"value": None, "unit": "pair-evals/s", "cores": 0, "kind": "unavailable",
                                    "sample": repr(e)}
    system.close()
    if rank == 0:
        print(json.dumps(line), flush=True)
    if distributed:
        dist.destroy_process_group()


def batch_arm(args):
    """BASELINE configs[3]: a population of independent registrations (default 128 x N=2000 per GPU, the per-GPU
    share of 1024 problems on 8 GPUs), one batched objective evaluation per step.  No collective: weak scaling."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1907_04839_b200 import BatchedRegistrations, make_template_points, rng_normals, HamiltonianSystem

    world, rank, local_rank, oversub, backend = init_ranks()
    B, n, T = args.batch, args.n or 2000, args.timesteps or 10
    K, W = max(args.steps, 1), max(args.warmup, 3)
    q0 = np.empty((B, n, 3))
    target = np.empty((B, n, 3))
    base = make_template_points(n, 40.0 * float(np.sqrt(n / 1847.0)))
    gen = HamiltonianSystem(SIGMA, n, 3, "f64", device=local_rank, max_timesteps=T)
    for b in range(B):  # seeds 0..1023 across the population
        p_true = (0.75 * rng_normals(rank * B + b, n * 3)).reshape(n, 3)
        q0[b] = base
        target[b] = gen.integrate_forward(base, p_true, T)[0][-1]
    gen.close()
    x0 = (target - q0) / T
    br = BatchedRegistrations(SIGMA, n, B, 3, args.precision, device=local_rank, max_timesteps=T, variant=args.variant)
    br.bind(q0, target, LAMBDA, T)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    h_x = torch.from_numpy(np.ascontiguousarray(x0)).pin_memory()
    h_grad = torch.empty_like(h_x).pin_memory()
    h_scalars = torch.empty(B * 3, dtype=torch.float64).pin_memory()
    for _ in range(W):
        br.evaluate_ptrs(h_x.data_ptr(), h_grad.data_ptr(), h_scalars.data_ptr())
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(local_rank)
    sampler.start()
    dev_ms = wall_ms = 0.0
    for _ in range(K):
        flush.fill_(1)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        br.evaluate_ptrs(h_x.data_ptr(), h_grad.data_ptr(), h_scalars.data_ptr())  # pinned host buffers
        wall_ms += (time.perf_counter() - t0) * 1e3
        dev_ms += br.last_eval_device_ms()
    clocks = sampler.result()
    if world > 1:
        t = torch.tensor([dev_ms, wall_ms], dtype=torch.float64, device="cuda" if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dev_ms, wall_ms = float(t[0]), float(t[1])
    units = 2.0 * T * float(n) * float(n) * B * world
    line = {
        "metric": "pair_kernel_evals_per_sec_per_gradient", "value": units * K / (dev_ms * 1e-3),
        "unit": "pair-evals/s", "n_gpus": world, "steps": K, "warmup": W, "ms_per_step": dev_ms / K,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": args.precision, "data": "synthetic",
        "config": {"workload": f"population: {B} independent registrations of N={n}, T={T} per GPU, one batched "
                               f"fwd+bwd gradient of all problems per step", "n": n, "batch_per_gpu": B, "timesteps": T,
                   "sigma": SIGMA, "lambda": LAMBDA, "l2": "flushed between timed steps (256 MiB write)"},
        "e2e": {"value": units * K / (wall_ms * 1e-3), "unit": "pair-evals/s", "h2d_bytes_per_step": int(x0.nbytes),
                "d2h_bytes_per_step": int(x0.nbytes) + 32 * B, "ms_per_step": wall_ms / K},
        "gpu_launches": (2 * T + 2) * K,
        "clocks": clocks,
        "registrations_per_sec_per_gradient": B * world * K / (dev_ms * 1e-3),
    }
    # whole batched gradient against the CUDA-core pipe (the per-kernel split is the single-problem arm's business):
    # contract slots per pair, forward + adjoint = 61 (fp64: 95), SURVEY.md section 8(d)
    peaks, peaks_src = measured_peaks()
    sm_mhz = float(peaks.get("sm_max_mhz", 1965.0))
    lanes = 128 if args.precision == "f32" else 64
    slots = (61.0 if args.precision == "f32" else 95.0) * T * float(n) * float(n) * B
    peak = 148 * lanes * sm_mhz * 1e6 / 1e12
    achieved = slots / (dev_ms / K * 1e-3) / 1e12
    line["roofline"] = {"bound": "fp32_cuda_core" if args.precision == "f32" else "fp64_cuda_core",
                        "kernel": "whole batched gradient (T forward + T adjoint pair-kernel launches over all problems)",
                        "achieved": achieved, "peak": peak, "unit": "Tslot/s (FP lane-instructions)",
                        "frac": achieved / peak, "traffic": None,
                        "peak_source": f"148 SM x {lanes} lanes x sm_max_mhz {sm_mhz:.0f} MHz ({peaks_src} MEASURED_PEAKS.json)"}
    br.close()
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse_args()
    if args.impl == "reference":
        reference_arm(args)  # host cores only: rank 0 runs it, under torchrun the other ranks exit at once
        return 0
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_launch(args)
    if args.launch_check:
        launch_check(args)
    elif args.batch > 0:
        batch_arm(args)
    else:
        b200_arm(args)
    return 0


if __name__ == "__main__":
    sys.exit(main())
