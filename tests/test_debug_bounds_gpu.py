"""Memory-safety evidence without compute-sanitizer (closed on this GPU pool):
the debug-bounds build (`-DFLLF_DEBUG_BOUNDS`) checks every global store of
the pyramid kernels against the range the host declared for the launch and
traps on a miss.  The parity suites run against that build here, and a
self-test proves the check fires."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DBG = os.path.join(ROOT, "paper_2206_04681_b200", "lib", "variants", "libfllf_dbg.so")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dbg_lib():
    csrc = os.path.join(ROOT, "paper_2206_04681_b200", "csrc")
    newest = max(os.path.getmtime(os.path.join(csrc, n)) for n in os.listdir(csrc))
    if not os.path.exists(DBG) or os.path.getmtime(DBG) < newest:
        subprocess.run([sys.executable, "-m", "paper_2206_04681_b200.build", "--variant", "dbg",
                        "-DFLLF_DEBUG_BOUNDS"], cwd=ROOT, check=True, stdout=subprocess.DEVNULL)
    assert os.path.exists(DBG)
    return DBG


def _pytest(args, env):
    return subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", *args],
                          cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)


def test_parity_suites_under_bounds_checks(dbg_lib):
    env = dict(os.environ, FLLF_LIB=dbg_lib)
    # the random sweep reaches every kernel variant (SCALAR / COEFFS / MAPS, batches,
    # padded pitches, 2..6 levels) in ~10 s; the full-size suites were run once
    # under the checks as well
    r = _pytest(["tests/test_parity_random_gpu.py", "tests/test_bands_gpu.py", "-m", "gpu"], env)
    print(r.stdout[-2000:], r.stderr[-2000:])
    assert r.returncode == 0


def test_bounds_check_fires(dbg_lib):
    code = ("import torch; from paper_2206_04681_b200 import fllf as F; "
            "x = torch.rand(64, 64, device='cuda') * 255; o = torch.empty_like(x); "
            "p = F.Plan(64, 64, 3, 4); p.filter(x, o); torch.cuda.synchronize()")
    env = dict(os.environ, FLLF_LIB=dbg_lib, FLLF_DEBUG_BOUNDS_SELFTEST="1")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode != 0 and "fllf bounds" in (r.stdout + r.stderr)
