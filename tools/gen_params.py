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

if __name__ == "__main__":
    here = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "params")
    sets = [
        make("P16", 65536, 23, 8, "configs 2-5: N=2^16, q0 60-bit + 23x40-bit, alpha=8, 6x60-bit special primes (SURVEY 8c-C0 with K=6, DESIGN R-K6)", K=6),
        make("P12", 4096, 2, 1, "config 1: N=2^12, 3 limbs, alpha=1 (insecure toy, functional only)"),
        make("P13", 8192, 7, 2, "test set: N=2^13, 8 limbs, alpha=2 (insecure; parity tests with dnum>1 and partial digits)"),
        make("P5", 32, 5, 2, "tiny set: N=32 for the pure-Python big-int cross-model (insecure)"),
    ]
    for s in sets:
        with open(os.path.join(here, s["name"].lower() + ".json"), "w") as f:
            json.dump(s, f, indent=1)
        print(s["name"], s["q"][:3], "...", s["p"][:2])
