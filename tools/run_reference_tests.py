"""Run the REFERENCE's own test suite (baseline/_ref/tests, installed by
tools/install_reference.sh) against the B200 drop-in, on a GPU box:

    python tools/run_reference_tests.py [pytest args]

``import fftlattice`` resolves to paper_2303_02317_b200 (tools/ref_shim.py);
writes a per-test pass / fail list to gpurun_out/reference_suite.txt.
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tests = os.path.join(ROOT, "baseline", "_ref", "tests")
if not os.path.isdir(tests):
    sys.exit("baseline/_ref/tests missing: run tools/install_reference.sh")
env = dict(os.environ, PYTHONPATH=os.path.join(ROOT, "tools") + os.pathsep + ROOT)
cmd = [sys.executable, "-m", "pytest", tests, "-p", "ref_shim", "-p", "no:cacheprovider", "-rA", "-q",
       "--rootdir", tests, *sys.argv[1:]]
sys.exit(subprocess.call(cmd, env=env, cwd=tests))
