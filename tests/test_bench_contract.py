"""bench.py's JSON-line contract, checked on the reference arm (the fp64 oracle on
the host cores; no GPU needed): one line, the keys the driver reads, the metric
and unit of BASELINE.json, and a cpu_baseline / e2e block describing the run."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    res = subprocess.run(
        [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
         "--warmup", "0", "--cpu-qblocks", "8", "--config", "wan13b_480p"],
        capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [l for l in res.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    with open(os.path.join(ROOT, "BASELINE.json")) as f:
        base = json.load(f)
    assert d["impl"] == "reference"
    assert d["metric"] == base["metric"]
    for key in ("value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["value"] > 0 and d["higher_is_better"] is True
    assert d["config"]["workload"] == "wan13b_480p"
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


def _bench():
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_gpus_n_relaunches_under_torchrun():
    """`bench.py --gpus N` outside torchrun becomes one process per GPU: the driver's
    own torch.distributed.run form, 127.0.0.1 rendezvous, the arguments passed on."""
    b = _bench()
    argv = ["--gpus", "4", "--steps", "7", "--dist-backend", "gloo"]
    cmd = b.torchrun_cmd(argv, 4, 29555)
    assert cmd[:3] == [sys.executable, "-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--nnodes=1" in cmd
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1"
    assert "--master-port=29555" in cmd
    assert cmd[-len(argv) - 1].endswith("bench.py") and cmd[-len(argv):] == argv
    a = b.parse(argv)
    assert a.gpus == 4 and a.dist_backend == "gloo" and a.steps == 7


def test_gpus_must_match_world_size(monkeypatch):
    b = _bench()
    monkeypatch.setenv("WORLD_SIZE", "2")
    import pytest
    with pytest.raises(SystemExit):
        b.main(["--gpus", "4"])


def test_reference_arm_world2_rank1_exits_without_work(monkeypatch):
    """Under torchrun (N > 1) the reference arm runs on rank 0 only; the other ranks
    exit 0 without work."""
    b = _bench()
    monkeypatch.setenv("WORLD_SIZE", "2")
    monkeypatch.setenv("RANK", "1")
    assert b.main(["--gpus", "2", "--impl", "reference"]) == 0


def test_cta_pair_needs_bq256_and_parses():
    """--cta-pair (the tcgen05 cta_group::2 kernel) is a Bq = 256 variant: without
    --bq 256 bench.py refuses before touching a GPU; with it the flags parse."""
    b = _bench()
    import pytest
    with pytest.raises(SystemExit):
        b.main(["--cta-pair"])
    a = b.parse(["--bq", "256", "--cta-pair"])
    assert a.bq == 256 and a.cta_pair
