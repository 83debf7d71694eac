"""tests/tools/gelu_taylor_coeffs.py -- offline generator (run once; output is
pasted into paper_2210_10246_b200/csrc/gelu_fwd_slow.h).

Taylor coefficients of g(x) = x * Phi(x) (proj/include/tempo/math.hpp:26-28)
around the GELU minimum x*, g'(x*) = 0, computed with mpmath at 50 digits.
g^(k)(x) = phi(x) * P_k(x), P_2 = 2 - x^2, P_{k+1} = P_k' - x P_k.
The device evaluates sum_k a_k h^k in fp64 for |x - x*| < 1/64, where the
in-place GELU backward is ill-conditioned (h(y) ~ sqrt(y - y_min)) and the
forward value must therefore round exactly like the reference's double.
"""
import mpmath as mp

mp.mp.dps = 50
DEG = 12


def main():
    phi = lambda x: mp.exp(-x * x / 2) / mp.sqrt(2 * mp.pi)
    Phi = lambda x: mp.ncdf(x)
    xs = mp.findroot(lambda x: Phi(x) + x * phi(x), -0.75)
    c0 = float(xs)  # expansion point: the double nearest x*
    c = mp.mpf(c0)
    coeffs = [c * Phi(c), Phi(c) + c * phi(c)]
    P = [mp.mpf(2), mp.mpf(0), mp.mpf(-1)]  # 2 - x^2, ascending powers
    fact = mp.mpf(2)
    for k in range(2, DEG + 1):
        val = sum(pc * c ** i for i, pc in enumerate(P))
        coeffs.append(phi(c) * val / mp.factorial(k))
        dP = [i * P[i] for i in range(1, len(P))] + [mp.mpf(0), mp.mpf(0)]
        xP = [mp.mpf(0)] + P
        P = [(dP[i] if i < len(dP) else 0) - (xP[i] if i < len(xP) else 0) for i in range(len(xP))]
    print("// x* =", mp.nstr(xs, 25), " c0 =", repr(c0))
    for k, a in enumerate(coeffs):
        print("    %s,  // a_%d" % (repr(float(a)), k))
    # accuracy of the truncated double series over |h| <= 1/32
    worst = 0
    for i in range(-400, 401):
        h = mp.mpf(i) / 400 / 32
        x = c + h
        exact = x * Phi(x)
        s = sum(mp.mpf(float(a)) * h ** k for k, a in enumerate(coeffs))
        worst = max(worst, abs(s / exact - 1))
    print("// max rel error of the double-coefficient series on |h|<=1/32:", mp.nstr(worst, 5))


if __name__ == "__main__":
    main()
