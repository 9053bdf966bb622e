"""bench.py's JSON line contract, checked on the CPU through the reference
arm (--impl reference runs the CPU port; no GPU needed)."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("method", ["local-gd", "local-ch"])
def test_reference_arm_json_line(method):
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--shape", "cora",
           "--eps", "1e-6", "--seeds", "16", "--steps", "2", "--warmup", "1", "--method", method]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["value"] > 0 and line["unit"] == "solves/s"
    assert line["steps"] == 2 and line["warmup"] == 1 and line["higher_is_better"] is True
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    assert "workload" in line["config"] and "model" not in line["config"]
    # the timed reference path never loads the product library
    probe = ("import runpy, sys; sys.argv = %r; runpy.run_path(%r, run_name='__main__'); "
             "print('LIBGDIFF', any('libgdiff' in l for l in open('/proc/self/maps')))"
             % (cmd[1:], cmd[1]))
    out2 = subprocess.run([sys.executable, "-c", probe], capture_output=True, text=True,
                          timeout=600, cwd=ROOT)
    assert out2.returncode == 0, out2.stderr[-2000:]
    assert "LIBGDIFF False" in out2.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("method", ["local-gd", "local-ch", "local-sor", "local-hk"])
def test_gpu_arm_json_line(method):
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--shape", "arxiv", "--eps", "1e-5",
           "--seeds", "64", "--steps", "2", "--warmup", "3", "--method", method,
           "--cpu-seconds", "1", "--tau", "1"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    r = line["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 1
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert line["gpu_launches"] > 0 and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] > 0 and line["e2e"]["d2h_bytes_per_step"] > 0
    assert "sm_mhz" in line["clocks"] and "reasons" in line["clocks"]
    cb = line["cpu_baseline"]
    assert cb["parity_sweeps_ops_identical"] is True
    assert cb["x_l1_rel_max"] <= cb["x_l1_rel_tolerance"] == 1e-9
    assert cb["topk_identical_up_to_ties"] >= 1
    assert line["exec_form"] and line["slots_used"] >= 1
    amb = line["ambiguous_seeds"]
    assert amb["flagged_per_step"] >= 0
    if method in ("local-gd", "local-ch"):
        assert amb["exact_resolve"]["changed_by_exact_resolve"] <= amb["exact_resolve"]["flagged"]
    if method == "local-gd":  # the global GD reference point beside the batched line
        gg = line["global_gd_reference"]
        assert gg["solves_per_s"] > 0 and gg["seeds"] == 2 and all(s >= 1 for s in gg["sweeps"])
    # the reference arm: same config dict, and it never loads the product library
    ref = subprocess.run(cmd + ["--impl", "reference"], capture_output=True, text=True,
                         timeout=900, cwd=ROOT)
    assert ref.returncode == 0, ref.stderr[-2000:]
    rline = json.loads(ref.stdout.strip().splitlines()[-1])
    assert rline["config"] == line["config"]
    assert rline["impl"] == "reference" and rline["metric"] == line["metric"]


@pytest.mark.gpu
def test_gpu_arm_torchrun_two_ranks():
    """The multi-rank code path of bench.py (torchrun, seed sharding, max-over-ranks
    timing, the per-step result gather) with 2 ranks; on a one-GPU box both ranks
    share cuda:0 and the collectives go through gloo (GDIFF_BENCH_BACKEND) -- a
    code-path check, not a scaling number."""
    import socket

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(ROOT, "bench.py"), "--gpus", "2", "--shape", "cora", "--eps", "1e-6",
           "--seeds", "16", "--steps", "2", "--warmup", "3"]
    env = dict(os.environ, GDIFF_BENCH_BACKEND="gloo")
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.strip().splitlines() if l.startswith("{")]
    assert len(lines) == 1  # rank 0 only
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["scaling"] == "weak"
    assert line["with_gather"]["value"] > 0 and line["e2e"]["value"] > 0
