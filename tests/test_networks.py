"""The generated median-selection / sorting networks of K2 (csrc/selnet.cuh, sortnet.cuh) are reproduced by the
committed generator and verified by the 0-1 principle (exhaustive for k <= 16) and random inputs (k <= 32)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_networks_regenerate_and_verify():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "gen_networks.py"), "--check"],
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "identical to the generator's: True" in out.stdout
