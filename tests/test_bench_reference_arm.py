"""bench.py's reference arm runs on CPU only (the unmodified reference
engine from baseline/_ref, else the oracle port, on every host core) and
prints the contract's JSON line; checked here so the CPU suite catches a
broken arm before a GPU round does.  Also the --gpus N self-launch."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_prints_contract_line():
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--steps", "2", "--warmup", "0"], capture_output=True, text=True,
                         env=env, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    assert line["unit"] == "MFLUPS" and line["value"] > 0
    assert line["warmup"] >= 3  # the contract's minimum
    cb = line["cpu_baseline"]
    want = "reference" if os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "slbm")) else "port"
    assert cb["kind"] == want and cb["cores"] >= 1 and cb["value"] == line["value"]
    assert cb["single_core"]["cores"] == 1 and cb["single_core"]["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]


def test_gpus_flag_self_launches_ranks():
    """`bench.py --gpus 2` without torchrun becomes two ranks (rank 0 prints
    one line with n_gpus 2); a WORLD_SIZE that contradicts --gpus is refused."""
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--gpus", "2", "--steps", "2", "--warmup", "0"], capture_output=True,
                         text=True, env=env, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    assert json.loads(lines[0])["n_gpus"] == 2
    env.update(WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    bad = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--gpus", "2", "--steps", "2"], capture_output=True, text=True, env=env,
                         timeout=300, cwd=ROOT)
    assert bad.returncode != 0 and "WORLD_SIZE" in bad.stderr
