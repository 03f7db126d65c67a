"""bench.py's reference arm (CPU): `--impl reference` prints ONE JSON line with the
contract's keys, on the same metric / unit / config dict as the GPU arm would emit for
that config, and it does so without mapping libamgcu.so into the process (its inputs come
from oracle/build/libconfiggen.so).  Runs the reference build when oracle/_ref is present,
else the own-code restatement -- a tiny size, a fraction of a second."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

PROBE = r"""
import json, runpy, sys, io, contextlib
sys.argv = ["bench.py", "--impl", "reference", "--config", "1", "--size", "48", "--steps", "1", "--warmup", "0",
            "--cpu-budget", "3"]
buf = io.StringIO()
with contextlib.redirect_stdout(buf):
    try:
        runpy.run_path("bench.py", run_name="__main__")
    except SystemExit:
        pass
maps = open("/proc/self/maps").read()
print(json.dumps({"line": buf.getvalue().strip().splitlines()[-1], "amgcu_loaded": "libamgcu.so" in maps,
                  "oracle_loaded": "oracle/" in maps}))
"""


def test_reference_arm_line_and_isolation():
    r = subprocess.run([sys.executable, "-c", PROBE], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    probe = json.loads(r.stdout.strip().splitlines()[-1])
    assert not probe["amgcu_loaded"], "the reference arm must not load the product library"
    assert probe["oracle_loaded"]
    line = json.loads(probe["line"])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["unit"] == "s" and line["higher_is_better"] is False
    assert line["vs_baseline"] is None and line["dtype"] == "f64"
    assert line["config"]["config"] == 1 and line["config"]["size"] == 48 and "workload" in line["config"]
    assert line["cpu_baseline"]["kind"] in ("reference", "port") and line["cpu_baseline"]["cores"] == 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    assert line["value"] > 0 and abs(line["ms_per_step"] - 1e3 * line["value"]) < 1e-6
