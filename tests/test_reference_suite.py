"""The reference package's own test-suite against the drop-in package.

tests/ref_suite/fetch.py copies /root/reference/pkg/tests/*.py into the git-ignored
tests/ref_suite/_ref/ (the copies travel to the GPU box; they are not committed), and
tests/ref_suite/shim aliases `maxwelldd` to paper_1711_03789_b200.  The files then run
unchanged on the device path.  What cannot pass is listed below with its reason; anything
else that fails is a drop-in regression.

  test_analysis.py        not collected: `analysis` (dense theory diagnostics) is out of scope
  test_oracles.py         collected: pure numpy helpers of the reference's tests
"""

import os
import re
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
REF = os.path.join(HERE, "ref_suite", "_ref")
SHIM = os.path.join(HERE, "ref_suite", "shim")

# test id (file::name) -> why the drop-in does not pass it
EXPECTED_FAILURES = {
    # the CLI's theory-diagnostic subcommands wrap `analysis`, which is out of scope:
    # they exit with status 2 and say so (cli.py)
    "test_experiments.py::TestCli::test_coercivity": "cli `coercivity` needs analysis.py (out of scope)",
    "test_experiments.py::TestCli::test_fov_identity": "cli `fov` needs analysis.py (out of scope)",
    "test_experiments.py::TestCli::test_abs_error": "cli `abs-error` needs analysis.py (out of scope)",
}


def test_reference_suite_on_the_device_path(gpu):
    if not os.path.isdir(REF) or not any(f.startswith("test_") for f in os.listdir(REF)):
        pytest.skip("tests/ref_suite/_ref not populated (python tests/ref_suite/fetch.py in the build container)")
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([SHIM, REF, os.path.dirname(HERE)]))
    cmd = [sys.executable, "-m", "pytest", REF, "-q", "-p", "no:cacheprovider", "--ignore",
           os.path.join(REF, "test_analysis.py"), "-rfEs", "--tb=line", "-c", os.devnull, "--rootdir", REF,
           "--confcutdir", REF]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=3000)
    out = r.stdout + r.stderr
    log = os.path.join(os.path.dirname(HERE), "gpurun_out", "ref_suite.log")
    try:
        os.makedirs(os.path.dirname(log), exist_ok=True)
        with open(log, "w") as f:
            f.write(out)
    except OSError:
        pass
    failed = set(re.findall(r"^(?:FAILED|ERROR) (\S+)", out, flags=re.M))
    failed = {f.split("_ref/")[-1] for f in failed}
    unexpected = sorted(f for f in failed if f not in EXPECTED_FAILURES)
    m = re.search(r"(\d+) passed", out)
    passed = int(m.group(1)) if m else 0
    print(out[-1500:])
    assert passed >= 140, out[-3000:]
    assert not unexpected, f"{len(unexpected)} reference tests fail on the drop-in: {unexpected[:20]}"
