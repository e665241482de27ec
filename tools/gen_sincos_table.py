"""Generate the FK kernel's sin/cos table (k pi / 64, k = 0..127) as fp64 hex literals.

Values are computed in x87 long double (64-bit mantissa: sinl/cosl of k * pi_l / 64 with
pi_l = 4 atanl(1)) and rounded once to double. Also prints the two-part Cody-Waite split
of pi / 64 (hi with its low 21 mantissa bits clear, so k * hi is exact for |k| < 2^20).
Output is pasted into paper_1910_06451_b200/csrc/fk_device.cuh (CUDA path only; the
oracle uses std::sin / std::cos)."""
import numpy as np

L = np.longdouble
pi_l = L(4) * np.arctan(L(1))
assert np.finfo(L).nmant >= 63, "needs x87 long double"
step = pi_l / L(64)
rows = []
for k in range(128):
    x = L(k) * step
    s, c = float(np.sin(x)), float(np.cos(x))
    if k % 32 == 0:  # multiples of pi/2: the exact values (pi_l carries ~1e-20 error)
        s, c = [(0.0, 1.0), (1.0, 0.0), (0.0, -1.0), (-1.0, 0.0)][k // 32]
    rows.append((s, c))
hi = float(step)
hi = np.frombuffer(np.array([hi]).tobytes(), dtype=np.uint64)[0] & ~np.uint64((1 << 21) - 1)
hi = float(np.frombuffer(np.array([hi], dtype=np.uint64).tobytes(), dtype=np.float64)[0])
lo = float(step - L(hi))
print(f"// pi/64 = hi + lo: hi = {hi.hex()}, lo = {lo.hex()}; 64/pi = {float(L(64) / pi_l).hex()}")
for k, (s, c) in enumerate(rows):
    print(f"    {{{s.hex()}, {c.hex()}}},  // k = {k}")
