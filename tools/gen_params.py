"""Generate the parameter files under params/ (data shared by the oracle and the library).

Primes are found by a downward search from 2^bits in steps of 2N (so q = 1 mod 2N, NTT-friendly),
exactly as SURVEY.md §8c-C0 / Appendix A.8 describe.  Only sympy.isprime is used.
The paper fixes only N, depth, Delta=2^40 with 40-bit body primes and 64-bit
words; everything else here is the build's reading.
"""
import json, os, sys
from sympy import isprime

def search(bits, step, count, below=None):
    top = below if below is not None else (1 << bits)
    x = top - (top % step) + 1
    if x >= top:
        x -= step
    out = []
    while len(out) < count:
        if isprime(x):
            out.append(x)
        x -= step
    return out

def make(name, N, n_body, alpha, note, K=None):
    """K special primes (default alpha).  For P16 the digits are alpha = 8 limbs of at most
    60 + 7*40 = 340 bits, so K = 6 sixty-bit special primes (360 bits) already give P > Q_j
    (reading R-K6); K = 8 (480 bits) would only add key-switching work."""
    step = 2 * N
    q0 = search(60, step, 1)[0]
    body = search(40, step, n_body)
    sp = search(60, step, K or alpha, below=q0)
    return {"name": name, "N": N, "q": [q0] + body, "p": sp, "alpha": alpha,
            "log2_scale": 40, "note": note}


def k_of_level(q, p, alpha, mu=16):
    """DESIGN.md reading R-KL: at level L the key switch extends by the first K(L) special primes, the smallest K
    with P_K = p_0 ... p_{K-1} >= 2^mu max_j Q_j(L) (Q_j(L) = the product of digit j's live limbs), mu = 16 bits of
    margin (exact integer comparison)."""
    out = []
    for L in range(1, len(q) + 1):
        D = 1
        for j in range(-(-L // alpha)):
            pr = 1
            for i in range(j * alpha, min((j + 1) * alpha, L)):
                pr *= q[i]
            D = max(D, pr)
        P, K = 1, 0
        while K < len(p):
            P *= p[K]
            K += 1
            if P >= D << mu:
                break
        out.append(K)
    return out


if __name__ == "__main__":
    here = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "params")
    p16 = make("P16", 65536, 23, 8, "configs 2-5: N=2^16, q0 60-bit + 23x40-bit, alpha=8, 6x60-bit special primes (SURVEY 8c-C0 with K=6, DESIGN R-K6)", K=6)
    p16["K_of_level"] = k_of_level(p16["q"], p16["p"], 8)
    p13 = make("P13", 8192, 7, 2, "test set: N=2^13, 8 limbs, alpha=2 (insecure; parity tests with dnum>1 and partial digits)")
    p13a8 = dict(p13, name="P13A8", alpha=8, p=[x for x in search(60, 2 * 8192, 8, below=p13["q"][0]) if x not in p13["p"]][:6],
                 note="test set: P13's body primes with alpha = 8 and six 60-bit special primes (exercises K(L) at N = 2^13)")
    p13a8["K_of_level"] = k_of_level(p13a8["q"], p13a8["p"], 8)
    p5 = make("P5", 32, 5, 2, "tiny set: N=32 for the pure-Python big-int cross-model (insecure)")
    p5a6 = dict(p5, name="P5A6", alpha=6, p=[x for x in search(60, 64, 7, below=p5["q"][0]) if x not in p5["p"]][:5],
                note="tiny set: P5's body primes with alpha = 6 and five 60-bit special primes (cross-model pins of K(L))")
    p5a6["K_of_level"] = k_of_level(p5a6["q"], p5a6["p"], 6)
    sets = [
        p16,
        make("P12", 4096, 2, 1, "config 1: N=2^12, 3 limbs, alpha=1 (insecure toy, functional only)"),
        p13,
        p13a8,
        p5,
        p5a6,
    ]
    for s in sets:
        with open(os.path.join(here, s["name"].lower() + ".json"), "w") as f:
            json.dump(s, f, indent=1)
        print(s["name"], s["q"][:3], "...", s["p"][:2])
