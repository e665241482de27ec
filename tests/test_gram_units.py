"""Host check of K3's work-unit enumeration (gram.cu units_before / unit_coords, restated
here): for every T and block count the units cover each upper-triangle tile (bi <= bj)
exactly once, which is what makes the streamed Gram write every entry of K."""
import math

import pytest


def units_before(b, T):
    q, r = divmod(b, T)
    return T * q * (q + 1) // 2 + r * (q + 1)


def unit_coords(u, nb, T):
    b = int((math.sqrt(T * T + 8.0 * T * u) - T) * 0.5)
    b = max(0, min(nb - 1, b))
    while b > 0 and units_before(b, T) > u:
        b -= 1
    while b + 1 < nb and units_before(b + 1, T) <= u:
        b += 1
    return b, (u - units_before(b, T)) * T


@pytest.mark.parametrize("T", [1, 2, 3, 4, 7])
@pytest.mark.parametrize("nb", [1, 2, 5, 40, 157, 1000])
def test_units_cover_upper_triangle_once(T, nb):
    tiles = []
    for u in range(units_before(nb, T)):
        bj, bi_first = unit_coords(u, nb, T)
        assert 0 <= bi_first <= bj < nb
        tiles += [(bi, bj) for bi in range(bi_first, min(bj, bi_first + T - 1) + 1)]
    assert len(tiles) == nb * (nb + 1) // 2
    assert set(tiles) == {(i, j) for j in range(nb) for i in range(j + 1)}


def test_units_sum_closed_form():
    # units_before(b) = sum_{k=1..b} ceil(k / T)
    for T in (1, 3, 4):
        for b in range(60):
            assert units_before(b, T) == sum(-(-k // T) for k in range(1, b + 1))
