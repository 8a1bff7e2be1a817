"""bench.py contract on the CPU: the reference arm (the oracle as it stands, a bounded
sample of the workload) prints one JSON line with the keys the driver reads."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "C2",
                        "--steps", "1", "--warmup", "0", "--ref-blocks", "8"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["value"] > 0 and d["unit"] == "TFLOP/s" and d["dtype"] == "f64"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


def test_nominal_flops_closed_form():
    """F = sum_c 2 r_c (r_c - 1) over all columns = 2 m (m+1)(m-1)/3 for an all-1x1 pencil."""
    sys.path.insert(0, ROOT)
    import bench
    m = 1000
    blocks = [(j, 1) for j in range(m)]
    assert bench.nominal_flops(blocks) == 2.0 * m * (m + 1) * (m - 1) / 3.0
    # the update kernels' algorithmic work is F minus the in-tile (diagonal solve) part
    f_upd, per, M = bench.update_flops(blocks, m, 128)
    assert M == 8 and len(per) == M - 1 and 0 < f_upd < bench.nominal_flops(blocks)


def test_gpus_n_outside_torchrun_starts_ranks(monkeypatch):
    """--gpus N > 1 without torchrun's environment re-launches bench.py through torchrun with
    N ranks (one per GPU) and the same flags (the driver's `bench.py --gpus 8`)."""
    sys.path.insert(0, ROOT)
    import bench
    calls = []
    monkeypatch.setattr(bench.subprocess, "call", lambda cmd: calls.append(cmd) or 0)
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "2"])
    try:
        bench.main()
    except SystemExit as e:
        assert e.code == 0
    assert len(calls) == 1
    cmd = calls[0]
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert cmd[cmd.index("--nproc-per-node") + 1] == "4"
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1"
    assert cmd[-4:] == ["--gpus", "4", "--steps", "2"] and cmd[-5].endswith("bench.py")
