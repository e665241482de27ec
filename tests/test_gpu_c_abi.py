"""The boundary used from plain C (examples/c_abi_demo.c, no Python or torch on the call
path): FK, model pack and the proxy collision check on the planar 2-link arm, against
hand-computed values (PAPER.md:183 with Eq. 4; the same sums as test_oracle_kernel)."""
import os
import subprocess

import pytest

from gpu_helpers import require_gpu

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_plain_c_program():
    require_gpu()
    exe = os.path.join(ROOT, "build", "c_abi_demo")
    os.makedirs(os.path.dirname(exe), exist_ok=True)
    cuda = "/usr/local/cuda"
    subprocess.check_call(["gcc", "-O2", "-I" + os.path.join(ROOT, "include"), "-I" + cuda + "/include",
                           os.path.join(ROOT, "examples", "c_abi_demo.c"),
                           "-L" + os.path.join(ROOT, "paper_1910_06451_b200"), "-lfastron_b200",
                           "-L" + cuda + "/lib64", "-lcudart",
                           "-Wl,-rpath," + os.path.join(ROOT, "paper_1910_06451_b200"), "-o", exe])
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    lines = out.stdout.strip().splitlines()
    got = [(float(a), int(b)) for a, b in (ln.split() for ln in lines[:3])]
    # Gaussian, gamma = ln 2: supports (pi,0) alpha 2 and (0,0) alpha -1
    ref = [2 * (2 ** -4 + 2 ** -16) / 2 - 1,            # query (0, 0)
           2 - (2 ** -4 + 2 ** -16) / 2,                 # query (pi, 0)
           2 * 0.25 - (0.25 + 2 ** -10) / 2]             # query (pi/2, pi/2)
    for (s, lab), f in zip(got, ref):
        assert abs(s - f) <= max(1e-4 * abs(f), 1e-5)
        assert lab == (1 if f > 0 else -1)
    assert "sm_100a" in lines[3]
