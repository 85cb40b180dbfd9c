"""The small-case GPU suite under the -DQJ2_CHECK debug build (-m gpu).

compute-sanitizer is not available on this pool; its substitute is a build of
the library with device-side checks of every index computed from the arguments
(QJ2_DCHECK in csrc/: tile and vector bounds against Np, walker/trial/tile
indices, shared-memory layouts against the launch's dynamic size, the sweep's k
and partner slots, the SPO gather rows).  A failing check traps the kernel.
This test runs the parity suites' small cases in a subprocess that loads
libqmcj2_check.so (QJ2_LIB) and requires them to pass unchanged.
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SMALL = ["tests/test_gpu_parity.py", "tests/test_gpu_accept.py", "tests/test_gpu_sweep.py", "tests/test_gpu_j1.py",
         "tests/test_gpu_spo.py", "tests/test_gpu_randomized.py"]
# the bench-size cases are the release build's (they take minutes of oracle time, not more coverage of indices)
EXCLUDE = ("full_size or C3_ or C4_ or C5_ or N64S or nio64 or S1V or deterministic or "
           "multi_trial_full or sweep_batch_full or accept_C3")


def test_small_suite_under_device_checks():
    sys.path.insert(0, ROOT)
    from paper_1708_02645_b200 import _build
    lib = _build.build_check()
    env = dict(os.environ, QJ2_LIB=lib)
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider", "-m", "gpu",
                        "-k", f"not ({EXCLUDE})", *SMALL], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=3000)
    tail = r.stdout[-3000:] + r.stderr[-2000:]
    assert r.returncode == 0, tail
    assert "QJ2_CHECK failed" not in r.stdout + r.stderr, tail
    print(tail[-400:])
