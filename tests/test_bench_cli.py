"""bench.py's driver contract on a host without a GPU (CPU suite): the reference arm prints
one JSON line timing the unmodified reference on the host cores, and a multi-GPU request
without the devices fails loudly instead of silently measuring fewer GPUs."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout):
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, env=env,
                          capture_output=True, text=True, timeout=timeout)


def test_gpus_without_devices_fails_loudly():
    r = _run(["--gpus", "2", "--steps", "1", "--warmup", "1"], 300)
    assert r.returncode != 0
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert "error" in line and "--gpus 2" in line["error"]


def test_reference_arm_json_line():
    if not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libcortex_ref.so")):
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    r = _run(["--impl", "reference", "--steps", "1", "--warmup", "0"], 600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "compressions/s" and line["value"] > 0
    assert line["higher_is_better"] is True and line["metric"].startswith("synapse compressions/s")
    cb = line["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] >= 1 and cb["value"] == line["value"]
    assert line["e2e"] == {"value": line["value"], "unit": line["unit"], "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}
    assert line["decode"]["decode_N1000"]["value"] > 0
