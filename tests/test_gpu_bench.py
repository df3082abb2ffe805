"""bench.py end to end on the GPU box: the default single-GPU line has every contract key,
and the multi-rank code paths (neuron sharding, time split with the fused handoff) run
under torchrun with every rank on cuda:0 (--debug-single-gpu: gloo group; numbers are not
bench values)."""
import json
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, nproc=1, port=29531):
    if nproc == 1:
        cmd = [sys.executable, "bench.py", *args]
    else:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
               "--master-addr", "127.0.0.1", f"--master-port={port}", "bench.py", *args]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_sweep_records_clean_and_dirty_flush_and_floor():
    """bench.py --sweep (BASELINE configs[1]'s T sweep): per T, the isolated launches after a
    clean flush, the dirty-memset repeat, the empty-launch floor and the back-to-back figure;
    the clean-flush launch is never slower than the floor alone."""
    d = _run(["--sweep", "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--no-e2e"])
    sw = d["sweep"]
    assert [s["T"] for s in sw] == [8, 32, 128, 512]
    for s in sw:
        for k in ("fwd_ms", "bwd_ms", "neuron_steps_per_s", "fwd_GBps", "bwd_GBps", "floor_ms",
                  "dirty_flush", "stream"):
            assert k in s, k
        assert 0 < s["floor_ms"] < s["fwd_ms"] and s["floor_ms"] < s["bwd_ms"]
        assert s["dirty_flush"]["fwd_ms"] > 0 and s["stream"]["neuron_steps_per_s"] > 0


def test_default_line_contract_keys():
    d = _run(["--steps", "5", "--warmup", "3", "--T", "64", "--cpu-seconds", "1", "--e2e-steps", "1"])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e",
              "gpu_launches", "clocks"):
        assert k in d, k
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and r["achieved"] > 0 and r["peak"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] == 1
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["gpu_launches"] == 10


@pytest.mark.parametrize("workload,extra", [("cfg1", ["--T", "32"]), ("cfg3", ["--T", "64"]),
                                            ("cfg3", ["--T", "64", "--transport", "handoff"]),
                                            ("cfg3", ["--T", "64", "--transport", "handoff-nccl"])])
def test_multirank_paths_under_torchrun(workload, extra):
    d = _run(["--gpus", "2", "--workload", workload, "--steps", "2", "--warmup", "3", "--no-e2e",
              "--debug-single-gpu", *extra], nproc=2, port=29532 if workload == "cfg1" else 29533)
    assert d["n_gpus"] == 2
    assert d["scaling"] == ("weak" if workload == "cfg1" else "strong")
    ts = d["tsplit"]
    assert ts["k"] == 2 and ts["Tk_ms"] > 0 and ts["T1_ms"] > 0 and ts["mu_measured"] > 0
    if "handoff-nccl" in extra:   # two NCCL "hosts" on one GPU are no LSA team: refused, IPC peers used
        assert "load/store peer" in ts["window_refused"]


def test_gpus_flag_self_launches_ranks():
    """`python bench.py --gpus 2` outside torchrun starts 2 ranks itself; at N > 1 the line
    carries the cfg3 time-split sub-record (T(k), T(1) of this run, mu_measured) beside the
    weak neuron-shard value.  (--debug-single-gpu: both ranks on cuda:0; NCCL over loopback.)"""
    d = _run(["--gpus", "2", "--steps", "2", "--warmup", "3", "--T", "32", "--no-e2e", "--debug-single-gpu",
              "--tsplit-steps", "2"])
    assert d["n_gpus"] == 2 and d["scaling"] == "weak"
    ts = d["tsplit"]
    assert ts["k"] == 2 and ts["transport"] == "nccl" and ts["mu_measured"] > 0
    assert ts["chunks"] >= 1 and 0 < ts["pipeline_efficiency"] <= 1


def test_affine_and_inference_legs():
    d = _run(["--steps", "3", "--warmup", "3", "--T", "32", "--no-e2e", "--no-cpu-baseline", "--affine",
              "--inference"])
    a, inf = d["affine"], d["inference"]
    assert a["fused_ms"] > 0 and a["fused_residual_ms"] > 0 and a["speedup_fused_vs_unfused"] > 1
    assert inf["forward_only_ms"] > 0 and inf["bn_folded_plan_neuron_steps_per_s"] > 0
