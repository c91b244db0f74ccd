"""bench.py's launch contract on CPU (gloo): `--gpus N` without torchrun
re-launches N ranks, the C3 batch is sharded so that the ranks cover the
65536 matrices exactly once, and a WORLD_SIZE that disagrees with --gpus is
refused."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env_extra=None):
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    env.update(env_extra or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], env=env,
                          capture_output=True, text=True, timeout=300, cwd=ROOT)


def _plan(res):
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert res.returncode == 0 and len(lines) == 1, (res.returncode, res.stdout, res.stderr[-3000:])
    return json.loads(lines[0])


@pytest.mark.parametrize("gpus", [1, 2, 3])
def test_gpus_flag_launches_ranks_and_shards_c3(gpus):
    plan = _plan(_run(["--gpus", str(gpus), "--plan-only"]))
    assert plan["n_gpus"] == gpus and plan["global_batch"] == 65536
    ranks = sorted(plan["ranks"], key=lambda r: r["rank"])
    assert [r["rank"] for r in ranks] == list(range(gpus))
    # contiguous, disjoint, covering [0, 65536); seeds follow the global index
    edges = [r["shard"] for r in ranks]
    assert edges[0][0] == 0 and edges[-1][1] == 65536
    assert all(a[1] == b[0] for a, b in zip(edges, edges[1:]))
    assert max(e[1] - e[0] for e in edges) - min(e[1] - e[0] for e in edges) <= 1
    assert all(r["seed0"] == 42 + r["shard"][0] for r in ranks)


def test_world_size_must_match_gpus():
    res = _run(["--gpus", "2", "--plan-only"], {"WORLD_SIZE": "1", "RANK": "0", "LOCAL_RANK": "0"})
    assert res.returncode != 0 and "WORLD_SIZE" in (res.stderr + res.stdout)


def test_shard_rule_matches_the_package():
    sys.path.insert(0, ROOT)
    import bench
    from paper_1204_3052_b200 import distributed as D

    for total in (1, 5, 65536, 65537):
        for world in (1, 2, 3, 8):
            for r in range(world):
                assert bench.shard_range(total, r, world) == D.shard_range(total, r, world)


def test_roofline_counts_the_k3h_launch_over_the_step():
    """A C3 step is one K3H launch (all the flops) + the K3B fixup pass (no
    work on an empty list): the roofline's rate is the step's flops over the
    step time, so a step at the measured 3.7 ms stays below the datapath peak
    (round 2 divided by 2 launches and reported frac 1.59)."""
    import bench

    w = bench.WORKLOADS["c3"]
    fl = bench.flops(w)
    peaks = {"bf16_tflops": 1641.9, "bf16_tflops_sustained": 1383.8}
    r = bench.roofline_of(w, True, fl, 3.7, 2, fl / 3.7e-3 / 1e12, 1, peaks, 759.0)
    assert abs(r["achieved"] - fl / 3.7e-3 / 1e12) < 1e-6
    assert r["algorithmic_flops_per_launch"] == fl
    assert 0.5 < r["frac"] < 1.0
    assert r["kernel"] == "k3h_batched_power"
    w5 = bench.WORKLOADS["c5"]
    f5 = bench.flops(w5)
    # K1PH (fp16 datapath / 3) on one GPU and row-sharded over 2
    r5 = bench.roofline_of(w5, False, f5, 24.0, 23, f5 / 24e-3 / 1e12, 1, peaks, 759.0)
    assert r5["kernel"] == "k1ph_gemm_f16x2" and 0.5 < r5["frac"] < 1.0
    r5s = bench.roofline_of(w5, False, f5, 13.0, 21, f5 / 13e-3 / 1e12, 2, peaks, 759.0)
    assert r5s["kernel"] == "k1ph_gemm_f16x2" and 0.5 < r5s["frac"] < 1.0
    # a 3xTF32 size (n_pad 1152, inside K1C's range): cuBLAS TF32 / 3
    w2 = bench.WORKLOADS["c2"]
    r2 = bench.roofline_of(w2, False, bench.flops(w2), 0.1, 2, bench.flops(w2) / 0.1e-3 / 1e12, 1,
                           peaks, 759.0)
    assert r2["kernel"] == "k1c_chain_3xtf32"
