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
# CPU arm: the reference's compute_gradient on a sample of the workload at the same landmark density; N = 6000 is
# (2T+2) * 3.6e7 pair evaluations = about 1 s per gradient on 16 host threads, 15-20 core-seconds of CPU work
CPU_SAMPLE_N = 6000


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
    return ap.parse_args()


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
def cpu_reference_run(n_sample, timesteps, precision, steps, warmup):
    """Times the reference's compute_gradient (shooting.hpp:277-315) on all host threads."""
    import numpy as np

    from oracle import load_oracle, load_reference, reference_available

    kind = "reference" if reference_available() else "port"
    cpu = load_reference() if kind == "reference" else load_oracle()
    cores = cpu.hardware_threads()
    oracle = load_oracle()
    # same generator as the GPU arm, host-only: Fibonacci sphere at the same point density, Rng(0) momenta,
    # target = fp64 flow of the template (synth.hpp:40-43)
    golden = np.pi * (3.0 - np.sqrt(5.0))
    i = np.arange(n_sample, dtype=np.float64)
    z = 1.0 - 2.0 * (i + 0.5) / n_sample
    r = np.sqrt(np.maximum(0.0, 1.0 - z * z))
    radius = 20.0 * np.sqrt(n_sample / 1847.0)  # constant landmark density (synth.hpp:19-20)
    q0 = np.stack([radius * r * np.cos(golden * i), radius * r * np.sin(golden * i), radius * z], axis=1)
    p_true = (0.75 * oracle.rng_normals(0, n_sample * 3)).reshape(n_sample, 3)
    target = cpu.integrate_forward("f64", q0, p_true, SIGMA, timesteps)[0][-1]
    x0 = (target - q0) / timesteps
    times = []
    for s in range(warmup + steps):
        t0 = time.perf_counter()
        cpu.compute_gradient(precision, q0, x0, target, SIGMA, LAMBDA, timesteps)
        dt = time.perf_counter() - t0
        if s >= warmup:
            times.append(dt)
    sec = sum(times) / len(times)
    units = 2.0 * timesteps * n_sample * n_sample
    return {
        "value": units / sec, "sec_per_gradient": sec, "cores": cores, "kind": kind,
        "sample": f"full compute_gradient on N={n_sample} (same generator and density as the N=20000 workload), "
                  f"T={timesteps}, {precision}, blocked_tree/256, {cores} threads; units counted as 2*T*N^2",
        "n_sample": n_sample,
    }


def reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    rows_mode = args.gpus > 1 and args.mode == "rows"  # the workload our own arm measures at this --gpus
    T = args.timesteps or (20 if rows_mode else 10)
    n = 200000 if rows_mode else 20000
    n_sample = args.n or CPU_SAMPLE_N
    res = cpu_reference_run(n_sample, T, args.precision, max(args.steps, 1), max(args.warmup, 0))
    line = {
        "impl": "reference", "metric": "pair_kernel_evals_per_sec_per_gradient", "value": res["value"],
        "unit": "pair-evals/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": res["sec_per_gradient"] * 1e3, "higher_is_better": True,
        "scaling": "strong" if rows_mode else "weak",
        "vs_baseline": None, "dtype": args.precision, "data": "synthetic",
        # our arm's workload; every step times the reference on a bounded sample of it (same generator, same
        # landmark density, same T, sigma, lambda), throughput counted in the same unit
        "config": {"workload": (f"single registration N={n}, T={T}, row-partitioned over {args.gpus} GPUs, per-step "
                                + ("NCCL all-gather" if args.exchange == "nccl" else "peer-push exchange (P2P stores + flags)")
                                if rows_mode else
                                f"single registration N={n}, T={T}, one fwd+bwd gradient per step"
                                + (f", {args.gpus} independent replicas" if args.gpus > 1 else "")), "n": n,
                   "timesteps": T, "sigma": SIGMA, "lambda": LAMBDA, "units_per_step": "2*T*N^2",
                   "template": "Fibonacci sphere, radius 20*sqrt(N/1847) mm (constant landmark density)",
                   "sample": res["sample"], "n_sample": n_sample},
        "cpu_baseline": {"value": res["value"], "unit": "pair-evals/s", "cores": res["cores"], "kind": res["kind"],
                         "sample": res["sample"]},
        "e2e": {"value": res["value"], "unit": "pair-evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


# ---- the B200 arm ------------------------------------------------------------------------------------------
def b200_arm(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1907_04839_b200 import HamiltonianSystem, comm_unique_id, make_synthetic_pair

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local_rank)
    distributed = world > 1
    if distributed:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))

    def barrier():
        if distributed:
            dist.barrier()
        torch.cuda.synchronize()

    rows_mode = distributed and args.mode == "rows"
    n = args.n or (200000 if rows_mode else 20000)
    T = args.timesteps or (20 if rows_mode else 10)
    prec = args.precision
    K, W = max(args.steps, 1), max(args.warmup, 3)

    # ---- workload (synthetic) ----
    # Template radius grows with sqrt(N/1847) so the landmark density is that of the reference's default
    # problem (synth.hpp:19-20: 1847 points on a 40 mm sphere).  At fixed 40 mm diameter N = 20 000 packs
    # 4 landmarks/mm^2 against sigma = 1.5 mm and the flow turns chaotic (|target - q0| up to 1.2 m, loss
    # 1e16, fp32 and fp64 differ by 0.6 %): not a meaningful evaluation point.  GPU time is data-independent.
    q0, target, _ = make_synthetic_pair(n, SIGMA, T, seed=0 if rows_mode else rank, device=local_rank,
                                        density_scaled=True)
    x0 = np.ascontiguousarray(((target - q0) / T).ravel())

    system = HamiltonianSystem(SIGMA, n, 3, prec, device=local_rank, max_timesteps=T, variant=args.variant)
    if rows_mode and args.exchange == "p2p":
        blobs = [None] * world
        dist.all_gather_object(blobs, system.p2p_export(rank, world))
        system.p2p_connect(blobs)
    elif rows_mode:
        uid = [comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        system.comm_init(uid[0], rank, world)
    system.bind_registration(q0, target, LAMBDA, T)

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

    sampler = ClockSampler(local_rank)
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
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

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
                         + ("NCCL all-gather" if args.exchange == "nccl" else "peer-push exchange (P2P stores + flags)")
                         if rows_mode else
                         f"single registration N={n}, T={T}, one fwd+bwd gradient per step"
                         + (f", {world} independent replicas" if distributed else "")),
            "n": n, "timesteps": T, "sigma": SIGMA, "lambda": LAMBDA, "units_per_step": "2*T*N^2",
            "template": "Fibonacci sphere, radius 20*sqrt(N/1847) mm (constant landmark density)",
            "l2": "flushed between timed steps (256 MiB write)", "variant": args.variant,
            "kernel_variant": system.lib.lms_system_kernel_names(system.handle).decode(),
        },
        "e2e": {"value": e2e_value, "unit": "pair-evals/s", "h2d_bytes_per_step": int(x0.nbytes),
                "d2h_bytes_per_step": int(x0.nbytes) + 32, "ms_per_step": wall_host / K},
        "gpu_launches": launches_per_step * K * 2,  # both timed passes
        "clocks": clocks,
        "wall_ms_per_step_device_buffers": wall_dev / K,
    }

    # ---- roofline of the dominant kernel (adjoint pair kernel), measured live with per-launch events ----
    if rank == 0:
        peaks, peaks_src = measured_peaks()
        system.set_kernel_timing(True)
        fwd_ms = adj_ms = 0.0
        for _ in range(K):
            flush_l2()
            system.objective_ptrs(d_x.data_ptr(), d_grad.data_ptr(), device=True)
            fwd_ms += system.last_kernel_ms("forward")
            adj_ms += system.last_kernel_ms("adjoint")
        system.set_kernel_timing(False)
        fwd_ms /= K
        adj_ms /= K
        rows_share = 1.0 / world if rows_mode else 1.0
        pairs_per_launch = float(n) * float(n) * rows_share
        f_slots, a_slots = (FWD_SLOTS, ADJ_SLOTS) if prec == "f32" else (FWD_SLOTS_F64, ADJ_SLOTS_F64)
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
            "traffic": (measured_traffic("adj", prec) or {}).get("bytes_per_launch") if n == 20000 and T == 10 else None,
            "traffic_source": (measured_traffic("adj", prec) or {}).get("source"),
            "forward_kernel": {"avg_launch_ms": fwd_ms, "achieved": fwd_rate / 1e12, "frac": fwd_rate / peak_slots,
                               "algorithmic_slots_per_pair": f_slots},
            "gradient": {"achieved": grad_rate / 1e12, "frac": grad_rate / peak_slots,
                         "slots_per_gradient": (f_slots + a_slots) * T * pairs_per_launch},
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
        if prec == "f32":
            s64 = HamiltonianSystem(SIGMA, n, 3, "f64", device=local_rank, max_timesteps=T, variant=args.variant)
            s64.bind_registration(q0, target, LAMBDA, T)
            for _ in range(2):
                s64.objective_ptrs(d_x.data_ptr(), d_grad.data_ptr(), device=True)
            ms64 = 0.0
            reps = max(3, K // 2)
            for _ in range(reps):
                flush_l2()
                s64.objective_ptrs(d_x.data_ptr(), d_grad.data_ptr(), device=True)
                ms64 += s64.last_eval_device_ms()
            ms64 /= reps
            slots64 = (FWD_SLOTS_F64 + ADJ_SLOTS_F64) * T * float(n) * float(n)
            line["fp64"] = {"ms_per_step": ms64, "value": units_per_step / (ms64 * 1e-3),
                            "frac_of_fp64_roofline": slots64 / (ms64 * 1e-3) / (148 * 64 * 1965e6)}
            s64.close()
        # ms per L-BFGS iteration: the whole registration loop through the C ABI (lms_register: host-buffer
        # objective + the library's host L-BFGS driver, no Python inside the loop)
        from paper_1907_04839_b200 import ShootingConfig, register_landmarks

        cfg = ShootingConfig(sigma=SIGMA, timesteps=T, lam=LAMBDA, max_iter=args.lbfgs_iters, precision=prec)
        t0 = time.perf_counter()
        reg = register_landmarks(q0, target, cfg, device=local_rank, system=system, already_bound=True)
        lb_ms = (time.perf_counter() - t0) * 1e3
        final_eval_ms = wall_host / K  # lms_register ends with one extra evaluation to leave q(1) resident
        line["lbfgs"] = {"iterations": reg.iterations, "evaluations": reg.evaluations,
                         "ms_per_iteration": (lb_ms - final_eval_ms) / max(reg.iterations, 1),
                         "ms_total": lb_ms, "final_loss": reg.final_loss, "initial_loss": reg.initial_loss,
                         "avg_dist_before_mm": reg.avg_before, "avg_dist_after_mm": reg.avg_after}
        # the same loop with the optimiser's vectors resident in HBM (lms_register_device)
        t0 = time.perf_counter()
        regd = register_landmarks(q0, target, cfg, device=local_rank, system=system, device_vectors=True,
                                  already_bound=True)
        lbd_ms = (time.perf_counter() - t0) * 1e3
        line["lbfgs_device_vectors"] = {"iterations": regd.iterations, "evaluations": regd.evaluations,
                                        "ms_per_iteration": (lbd_ms - dev_ms / K) / max(regd.iterations, 1),
                                        "ms_total": lbd_ms, "final_loss": regd.final_loss}
        try:
            cpu = cpu_reference_run(CPU_SAMPLE_N, T, prec, 1, 1)
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

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local_rank)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
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
    dev_ms = wall_ms = 0.0
    for _ in range(K):
        flush.fill_(1)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        br.evaluate_ptrs(h_x.data_ptr(), h_grad.data_ptr(), h_scalars.data_ptr())  # pinned host buffers
        wall_ms += (time.perf_counter() - t0) * 1e3
        dev_ms += br.last_eval_device_ms()
    if world > 1:
        t = torch.tensor([dev_ms, wall_ms], dtype=torch.float64, device="cuda")
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
        "registrations_per_sec_per_gradient": B * world * K / (dev_ms * 1e-3),
    }
    br.close()
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse_args()
    if args.impl == "reference":
        reference_arm(args)
    elif args.batch > 0:
        batch_arm(args)
    else:
        b200_arm(args)


if __name__ == "__main__":
    main()
