"""bench.py's host-side plumbing (no GPU): the self-launcher really starts N ranks, and the reference arm times
the configuration it prints."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(*flags, env=None, timeout=300):
    e = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        e.pop(k, None)
    e.update(env or {})
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *flags], capture_output=True, text=True,
                         timeout=timeout, env=e, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout  # rank 0 prints ONE JSON line, the other ranks nothing
    return json.loads(lines[0])


def test_gpus_flag_starts_that_many_ranks_by_itself():
    """`python bench.py --gpus 2` with no torchrun environment must launch two ranks (it used to run one rank and
    print n_gpus: 1)."""
    doc = run_bench("--gpus", "2", "--launch-check")
    assert doc["launch_check"] and doc["n_gpus"] == 2 and doc["requested"] == 2
    ranks = doc["ranks"]
    assert sorted(r["rank"] for r in ranks) == [0, 1]
    assert len({r["pid"] for r in ranks}) == 2  # two processes, one per rank


def test_launch_check_inside_an_existing_torchrun_environment_does_not_nest():
    doc = run_bench("--gpus", "1", "--launch-check")
    assert doc["n_gpus"] == 1 and len(doc["ranks"]) == 1


def test_reference_arm_times_the_configuration_it_prints():
    """The reference arm's `config.n` is the N it ran (round 1 printed 20000 while timing 6000)."""
    doc = run_bench("--impl", "reference", "--landmarks", "300", "--timesteps", "3", "--steps", "2", "--warmup", "1",
                    "--no-extras")
    assert doc["impl"] == "reference" and doc["config"]["n"] == 300 and doc["config"]["n_workload"] == 300
    assert doc["config"]["timesteps"] == 3 and doc["steps"] == 2 and doc["warmup"] == 1
    assert "N=300" in doc["cpu_baseline"]["sample"] and doc["cpu_baseline"]["kind"] in ("reference", "port")
    assert doc["value"] > 0 and doc["e2e"]["value"] == doc["value"]
    # units are 2*T*N^2 per step
    assert abs(doc["value"] * doc["ms_per_step"] * 1e-3 - 2 * 3 * 300 * 300) < 1e-3 * 2 * 3 * 300 * 300


def test_reference_arm_samples_only_the_row_partitioned_workload_and_says_so():
    doc = run_bench("--impl", "reference", "--gpus", "2", "--landmarks", "400", "--timesteps", "2", "--steps", "1",
                    "--warmup", "0")
    assert doc["n_gpus"] == 2 and doc["scaling"] == "strong"
    assert doc["config"]["n"] == 400 and doc["config"]["n_workload"] == 400  # below the sample size: run in full
