"""bench.py's reference arm (the oracle on bounded samples, CPU only) keeps the
JSON-line contract, at one process and under torchrun with two ranks (rank 0
alone prints; the other exits 0 without work).  -m "not gpu"."""
import json
import os
import socket
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
        "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"}


def _lines(out):
    return [json.loads(l) for l in out.splitlines() if l.startswith("{")]


def test_reference_arm_single_process():
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--workload", "C3s", "--steps", "1",
                          "--warmup", "0", "--ref-seconds", "1"], cwd=ROOT, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    (line,) = _lines(out.stdout)
    assert KEYS <= set(line), KEYS - set(line)
    assert line["impl"] == "reference" and line["value"] > 0 and line["config"]["workload"] == "C3s"
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] == 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0


def test_reference_arm_under_torchrun_two_ranks():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--impl", "reference",
           "--workload", "C3s", "--steps", "1", "--warmup", "0", "--ref-seconds", "1", "--gpus", "2"]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = _lines(out.stdout)
    assert len(lines) == 1 and lines[0]["impl"] == "reference"


def test_gpus_flag_relaunches_under_torchrun():
    """--gpus 2 outside torchrun re-launches bench.py with two ranks (one per GPU);
    the reference arm's line then reports n_gpus = 2 and only rank 0 prints."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--workload", "C3s", "--steps", "1",
                          "--warmup", "0", "--ref-seconds", "1", "--gpus", "2"], cwd=ROOT, capture_output=True,
                         text=True, timeout=900, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = _lines(out.stdout)
    assert len(lines) == 1 and lines[0]["n_gpus"] == 2 and lines[0]["impl"] == "reference"


def test_gpus_flag_must_match_world_size():
    """Under a launcher, --gpus disagreeing with WORLD_SIZE fails loudly (exit 2)
    instead of silently measuring another configuration."""
    env = dict(os.environ, WORLD_SIZE="3", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--steps", "1", "--warmup", "0"], cwd=ROOT,
                         capture_output=True, text=True, timeout=300, env=env)
    assert out.returncode == 2 and "WORLD_SIZE" in out.stderr


def test_cpu_baseline_sample_is_bounded_and_comparable():
    """cpu_baseline: oracle tier 5 (the method itself, sequential) solving a
    same-recipe cube in full; its numerator is the metric's (live edges +
    phantoms per cycle); it reports the host's core count and CPU model."""
    sys.path.insert(0, ROOT)
    import bench
    c = bench.cpu_sample("C3", 2.0)
    assert c["kind"] == "oracle" and c["cores"] == 1 and c["value"] > 0 and c["host_nproc"] >= 1
    assert c["seconds"] < 30 and "tier 5" in c["sample"]


def test_alg_bytes_is_survey_formula():
    """roofline.achieved uses SURVEY §8(d)'s 'alg' numerator."""
    sys.path.insert(0, ROOT)
    import bench
    from types import SimpleNamespace as R
    r = R(edge_updates=10, arrivals=3, triggered=2, phantoms_created=5, relabels=7, lanes_started=1)
    assert bench.alg_bytes(r, 3) == 2 * 10 + 13 * 3 + (6 * 8 + 22) * 2 + 8 * 5 + 2 * 7
