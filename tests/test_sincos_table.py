"""CPU checks of K1's sin/cos table (paper_1910_06451_b200/csrc/fk_device.cuh,
`kFkSinCos`): it is what tools/gen_sincos_table.py generates, each entry is within one
fp64 ulp of sin / cos(k pi / 64), and the multiples of pi / 2 are exact."""
import os
import re
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "paper_1910_06451_b200", "csrc", "fk_device.cuh")


def _table():
    text = open(HDR).read()
    body = text[text.index("kFkSinCos[128] = {"):]
    body = body[:body.index("};")]
    pairs = re.findall(r"\{(-?0x[0-9a-fp.+-]+), (-?0x[0-9a-fp.+-]+)\}", body)
    return np.array([(float.fromhex(s), float.fromhex(c)) for s, c in pairs])


def test_table_matches_generator():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "gen_sincos_table.py")], capture_output=True,
                         text=True, check=True).stdout.splitlines()[1:]
    gen = np.array([(float.fromhex(a), float.fromhex(b))
                    for a, b in re.findall(r"\{(-?0x[0-9a-fp.+-]+), (-?0x[0-9a-fp.+-]+)\}", "\n".join(out))])
    tab = _table()
    assert tab.shape == (128, 2)
    assert np.array_equal(tab, gen)


def test_table_values():
    tab = _table()
    x = np.arange(128) * (np.pi / 64)
    ref = np.stack([np.sin(x), np.cos(x)], axis=1)
    # np.pi / 64 * k carries up to ~k ulp(pi) of argument error: compare with a bound that
    # covers it plus one ulp of the value
    tol = np.spacing(np.abs(ref)) + 128 * np.spacing(np.pi) / 64 * np.arange(128)[:, None]
    assert np.all(np.abs(tab - ref) <= tol)
    assert np.allclose(tab[:, 0] ** 2 + tab[:, 1] ** 2, 1.0, rtol=0, atol=4e-16)
    for k, (s, c) in {0: (0.0, 1.0), 32: (1.0, 0.0), 64: (0.0, -1.0), 96: (-1.0, 0.0)}.items():
        assert tab[k, 0] == s and tab[k, 1] == c
    # symmetry of the exact values: sin(k pi/64) = cos((32 - k) pi/64) for k = 0..32
    assert np.array_equal(tab[:33, 0], tab[32::-1, 1])
