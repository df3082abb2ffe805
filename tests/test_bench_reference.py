"""bench.py --impl reference (CPU only, no GPU needed): the reference arm of this tier is the
fp64 oracle timed on the host cores; one JSON line with the contract keys, rank 0 only under
a multi-rank launch."""
import json
import os
import subprocess
import sys

from conftest import ROOT


def _lines(out):
    return [l for l in out.splitlines() if l.startswith("{")]


def test_reference_arm_single_process():
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "3"],
                         cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = _lines(out.stdout)
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "neuron-steps/s"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    for k in ("metric", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling", "config"):
        assert k in d


def test_reference_arm_other_ranks_exit_quietly():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2")
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "3"],
                         cwd=ROOT, capture_output=True, text=True, timeout=600, env=env)
    assert out.returncode == 0 and not _lines(out.stdout)


def test_gpus_flag_relaunches_under_torchrun(monkeypatch):
    """`python bench.py --gpus N` (N > 1) without torchrun re-executes itself as N ranks of
    torch.distributed.run on 127.0.0.1, forwarding every argument (the driver's N-GPU runs)."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    seen = {}

    def fake_call(cmd, env=None):
        seen["cmd"], seen["env"] = cmd, env
        return 0

    import subprocess as sp
    monkeypatch.setattr(sp, "call", fake_call)
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "7", "--warmup", "3"])
    args = bench.parse()
    assert bench.relaunch_under_torchrun(args) == 0
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"] and "--nproc-per-node=4" in cmd
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1"
    assert cmd[-6:] == ["--gpus", "4", "--steps", "7", "--warmup", "3"]
    assert seen["env"]["NCCL_DEBUG"] == "INFO"
    # under torchrun, a --gpus that disagrees with WORLD_SIZE is refused
    monkeypatch.setenv("WORLD_SIZE", "2")
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4"])
    import pytest
    with pytest.raises(SystemExit):
        bench.main()


def test_serial_pytorch_baseline_matches_oracle():
    """Fig. 5's "Serial (PyTorch)" baseline that bench.py --sweep --serial times computes the same
    layer as the method: spikes and dL/dX against the fp64 oracle (CPU, paper parameters)."""
    import torch
    sys.path.insert(0, ROOT)
    import bench
    import paper_2408_00280_b200 as snn
    import snn_synth
    from parity import oracle_check
    p = snn.LIFParams.paper()
    T, N = 24, 700
    X = snn_synth.normal_tensor(1234, T, N)
    G = snn_synth.normal_tensor(4321, T, N)
    S, gX = bench.torch_serial_lif(X, G, p)
    rep = oracle_check(p, X, G, S.to(torch.uint8), gX)
    assert rep.ok, str(rep)
    assert 0.05 < S.float().mean() < 0.95   # non-degenerate firing


def test_algorithmic_bytes_count_the_stored_checkpoints():
    """bench.py's algorithmic bytes: fp32 io, u8 spikes, RECOMPUTE moves
    X in + S out (+ checkpoints) forward and gS, X in + gX out (+ checkpoints) backward; the
    V[-1] checkpoint is never stored (r2c), so T <= 16 moves exactly 5 + 12 bytes."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    assert b.bytes_per_neuron_step(4, "u8", "recompute", 16) == (5.0, 12.0)
    assert b.bytes_per_neuron_step(4, "u8", "recompute", 8) == (5.0, 12.0)
    f, w = b.bytes_per_neuron_step(4, "u8", "recompute", 512)       # 31 stored rows of 4 B each
    assert abs(f - (5 + 4 * 31 / 512)) < 1e-12 and abs(w - (12 + 4 * 31 / 512)) < 1e-12
    assert b.bytes_per_neuron_step(2, "io", "recompute", 16) == (4.0, 6.0)   # cfg2 with bf16 spikes
    assert b.bytes_per_neuron_step(4, "bits", "h", 64) == (4 + 1 / 8 + 4, 12.0)
    assert b.ckpt_bytes(33, ck0=True) == 4.0 * 3 / 33
