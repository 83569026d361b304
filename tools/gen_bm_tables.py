"""Generate the Box-Muller cosine table (common.cuh kBmCosTab): cos / sin of k pi/32, k = 0..32, and the
two-part Cody-Waite constant C1 + C2 = pi/32 (C1 with 44 significant bits so k C1 is exact for k <= 64),
correctly rounded from 60-digit decimal arithmetic."""
from decimal import Decimal, getcontext
import struct

getcontext().prec = 60


def pi():
    # Machin: pi = 16 atan(1/5) - 4 atan(1/239)
    def atan_inv(x):
        x = Decimal(x)
        s, t, k, x2 = Decimal(0), 1 / x, 0, x * x
        while True:
            term = t / (2 * k + 1)
            if abs(term) < Decimal(10) ** -58:
                break
            s += -term if k % 2 else term
            t /= x2
            k += 1
        return s
    return 16 * atan_inv(5) - 4 * atan_inv(239)


def sincos(a):
    s, c, term, k = Decimal(0), Decimal(0), Decimal(1), 0
    while abs(term) > Decimal(10) ** -58:
        if k % 4 == 0: c += term
        elif k % 4 == 1: s += term
        elif k % 4 == 2: c -= term
        else: s -= term
        k += 1
        term = term * a / k
    return s, c


def hexd(x: float) -> str:
    return float(x).hex()


P = pi() / 32
c1 = float(P)
m, e = __import__("math").frexp(c1)
c1 = __import__("math").ldexp(round(m * 2 ** 44) / 2 ** 44, e)
c2 = float(P - Decimal(c1))
rows = []
for k in range(33):
    s, c = sincos(P * k)
    s, c = (Decimal(0) if abs(s) < Decimal(10) ** -40 else s), (Decimal(0) if abs(c) < Decimal(10) ** -40 else c)
    rows.append(f"    {{{hexd(float(c))}, {hexd(float(s))}}},  // k = {k}")
if len(__import__("sys").argv) == 1:
    print(f"// C1 = {hexd(c1)}, C2 = {hexd(c2)}")
    print("\n".join(rows))


def log_table():
    """Box-Muller log table (common.cuh kBmLogTab): for j = 48..96, inv_j = 64/j rounded to double and
    -ln(inv_j) (the exact logarithm of the stored reciprocal) as a hi + lo pair; ln 2 as hi (44 bits) +
    lo."""
    rows = []
    for j in range(48, 97):
        inv = float(Decimal(64) / Decimal(j))
        L = -Decimal(inv).ln()
        hi = float(L)
        lo = float(L - Decimal(hi))
        rows.append(f"    {{{hexd(inv)}, {hexd(hi)}, {hexd(lo)}, 0.0}},  // j = {j}")
    ln2 = Decimal(2).ln()
    m, e = __import__("math").frexp(float(ln2))
    l2hi = __import__("math").ldexp(round(m * 2 ** 44) / 2 ** 44, e)
    l2lo = float(ln2 - Decimal(l2hi))
    return f"// LN2_HI = {hexd(l2hi)}, LN2_LO = {hexd(l2lo)}", rows


if __name__ == "__main__" and len(__import__("sys").argv) > 1 and __import__("sys").argv[1] == "log":
    h, r = log_table()
    print(h)
    print("\n".join(r))
