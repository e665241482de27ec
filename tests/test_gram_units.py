"""Host check of K3's work-unit enumeration (gram.cu g2_units_before / g2_unit, restated
here). Column blocks are W = 128 * QT wide; with NBf = n // W full blocks and R = n - W NBf
remainder columns (E = ceil(R / 64) remainder row tiles), full block b takes the row tiles of
[0, W (b + 1)) plus the E remainder tiles, and the remainder block takes its own E diagonal
tiles; one unit = one (block, row tile). For every width and n the units must cover each
such pair exactly once, and the direct + mirror stores they imply must write every entry of
K exactly once (the diagonal square of a block: direct stores only)."""
import math

import pytest


def units_before(b, hb, E):
    return hb * b * (b + 1) + E * b


def unit(u, nbf, hb, E):
    A, B = float(hb), float(hb + E)
    b = int((-B + math.sqrt(B * B + 4.0 * A * u)) / (2.0 * A))
    b = max(0, min(nbf, b))
    while b > 0 and units_before(b, hb, E) > u:
        b -= 1
    while b < nbf and units_before(b + 1, hb, E) <= u:
        b += 1
    k = u - units_before(b, hb, E)
    tpb, tf = 2 * hb, nbf * 2 * hb
    tile = tf + k if b == nbf else (k if k < tpb * (b + 1) else tf + (k - tpb * (b + 1)))
    return b, tile


def n_units(n, qt, uh=64):
    W = 128 * qt
    nbf, R = n // W, n % W
    E = -(-R // uh)
    hb = W // uh // 2
    return units_before(nbf, hb, E) + (E if R else 0), nbf, E, hb


@pytest.mark.parametrize("uh", [32, 64])
@pytest.mark.parametrize("qt", [1, 2, 3])
@pytest.mark.parametrize("n", [1, 63, 64, 127, 383, 384, 385, 1000, 5000, 20000, 100_003])
def test_units_cover_needed_row_tiles_once(qt, n, uh):
    W = 128 * qt
    total, nbf, E, hb = n_units(n, qt, uh)
    seen = {}
    for u in range(total):
        b, t = unit(u, nbf, hb, E)
        seen[(b, t)] = seen.get((b, t), 0) + 1
    tf = nbf * 2 * hb
    want = {(b, t) for b in range(nbf) for t in range(2 * hb * (b + 1))}
    want |= {(b, t) for b in range(nbf + (1 if n % W else 0)) for t in range(tf, tf + E)}
    assert set(seen) == want and all(c == 1 for c in seen.values()), (n, qt)


@pytest.mark.parametrize("uh", [32, 64])
@pytest.mark.parametrize("qt,n", [(1, 300), (3, 1000), (3, 385), (1, 129), (3, 770), (2, 700), (2, 256)])
def test_entries_written_once(qt, n, uh):
    W = 128 * qt
    total, nbf, E, hb = n_units(n, qt, uh)
    cnt = [[0] * n for _ in range(n)]
    for u in range(total):
        b, t = unit(u, nbf, hb, E)
        j0 = b * W
        cols = range(j0, min(n, j0 + W))
        r0 = uh * t
        mirror = r0 < j0 or r0 >= j0 + W
        for r in range(r0, min(n, r0 + uh)):
            for c in cols:
                cnt[r][c] += 1
                if mirror:
                    cnt[c][r] += 1
    assert all(v == 1 for row in cnt for v in row), (qt, n)
