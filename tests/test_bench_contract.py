"""bench.py output contract (CPU): stdout carries exactly the JSON line even
when native code writes to fd 1 (NCCL's version banner at communicator init)."""
import json
import subprocess
import sys

from helpers import ROOT

SCRIPT = r'''
import os, sys
sys.path.insert(0, sys.argv[1])
import bench
bench._stdout_to_stderr()
os.write(1, b"NCCL version 0.0.0 (native banner)\n")
print("python-level chatter")
bench.emit({"metric": "m", "value": 1.5})
'''


def test_stdout_is_only_the_json_line():
    r = subprocess.run([sys.executable, "-c", SCRIPT, ROOT], capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = r.stdout.splitlines()
    assert len(lines) == 1 and json.loads(lines[0]) == {"metric": "m", "value": 1.5}
    assert "NCCL version" in r.stderr and "python-level chatter" in r.stderr
