"""bench.py's launch contract on CPU: `--gpus N` really drives N ranks.

* Outside torchrun, `--gpus N` re-launches the script under torch.distributed.run with N
  ranks; the plumbing dry run (gloo, host memcpy in place of the load) proves every rank
  started with WORLD_SIZE = N, picked its own partition of the config chosen for N, and that
  rank 0 printed ONE line with n_gpus = N.
* Without enough GPUs the real run fails loudly (nonzero exit) instead of measuring one GPU.
* `--config auto` maps N to the BASELINE config (N = 8: LLaMA-2-70B TP8, the north star).
* The reference arm (the oracle) runs mode (i) on one partition and mode (ii) -- one process
  per partition -- on a sharded config, with the host description and median / min.
"""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BENCH = os.path.join(ROOT, "bench.py")


def _env():
    env = dict(os.environ)
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT", "SLLM_BENCH_SAME_GPU"):
        env.pop(k, None)
    env["CUDA_VISIBLE_DEVICES"] = ""
    return env


def _run(args, timeout=300):
    out = subprocess.run([sys.executable, BENCH, *args], capture_output=True, text=True, timeout=timeout,
                         env=_env(), cwd=ROOT)
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    return out, lines


def test_config_for_gpu_count():
    sys.path.insert(0, ROOT)
    import bench
    a = bench.parse([])
    assert [bench.resolve_config(a, n) for n in (1, 2, 4, 8)] == \
        ["opt-6.7b", "llama2-13b-tp2", "llama2-70b-tp4", "llama2-70b-tp8"]
    assert bench.resolve_config(bench.parse(["--fanout", "bcast"]), 8) == "opt-30b"
    assert bench.resolve_config(bench.parse(["--config", "toy"]), 8) == "toy"
    # rank -> partition: sharded configs one partition per rank, replicated partition 0
    assert [bench.choose_partitions(a, r, 8, 8, False) for r in range(8)] == [[r] for r in range(8)]
    assert bench.choose_partitions(a, 3, 4, 2, False) == [1]
    assert bench.choose_partitions(a, 3, 4, 1, True) == [0]


@pytest.mark.parametrize("n", [2, 4])
def test_self_launch_spawns_n_ranks(n):
    out, lines = _run(["--plumbing", "--gpus", str(n), "--steps", "2", "--warmup", "1"])
    assert out.returncode == 0, out.stderr[-3000:]
    assert len(lines) == 1, out.stdout          # rank 0 alone prints
    line = lines[0]
    assert line["n_gpus"] == n and line["plumbing"] is True
    ranks = line["ranks"]
    assert sorted(r["rank"] for r in ranks) == list(range(n))
    assert all(r["world_size_env"] == n for r in ranks)
    assert len({r["pid"] for r in ranks}) == n  # one process per rank
    assert line["config"]["workload"] == {2: "llama2-13b-tp2", 4: "llama2-70b-tp4"}[n]
    assert sorted(r["partitions"][0] for r in ranks) == list(range(n))


def test_gpus_n_without_gpus_fails_loudly():
    out, lines = _run(["--gpus", "2", "--steps", "1", "--warmup", "1"], timeout=120)
    assert out.returncode != 0 and not lines
    assert "needs 2 visible GPUs, found 0" in out.stderr


def test_single_gpu_run_without_gpu_fails_loudly():
    out, lines = _run(["--steps", "1", "--warmup", "1"], timeout=120)
    assert out.returncode != 0 and not lines
    assert "no CUDA GPU visible" in out.stderr


def test_reference_arm_mode_i_toy():
    out, lines = _run(["--impl", "reference", "--config", "toy", "--steps", "3", "--warmup", "1"])
    assert out.returncode == 0, out.stderr[-3000:]
    (line,) = lines
    cpu = line["cpu_baseline"]
    assert line["impl"] == "reference" and line["n_gpus"] == 1 and cpu["cores"] == 1 and cpu["kind"] == "oracle"
    assert cpu["reps"] == 3 and cpu["min_s"] <= cpu["median_s"]
    assert set(cpu["host"]) == {"cpu_model", "os_cpu_count", "affinity_cores"}
    assert line["step_s"]["n"] == 3 and line["e2e"]["h2d_bytes_per_step"] == 0
    assert "13569860 payload bytes" in cpu["sample"]      # the whole toy (budget > partition)


def test_reference_arm_mode_ii_sharded():
    """Sharded config at N = 2: rank 0 alone times the oracle with one process per partition."""
    if len(os.sched_getaffinity(0)) < 2:
        pytest.skip("needs 2 cores")
    out, lines = _run(["--impl", "reference", "--gpus", "2", "--config", "llama2-13b-tp2", "--steps", "2",
                       "--warmup", "0", "--cpu-sample-gib", "0.01"], timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    (line,) = lines
    assert line["n_gpus"] == 2 and line["cpu_baseline"]["cores"] == 2
    assert line["cpu_baseline"]["mode"].startswith("(ii)") and line["sampled_partitions"] == [0, 1]
