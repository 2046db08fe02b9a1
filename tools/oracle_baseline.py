"""Time the oracle (as it stands) on COMPLETE units of the benchmark workloads, single-thread and on every core.

  config1   BASELINE configs[0] in full: P12 (N = 2^12, 3 limbs), the 64x64 single-ciphertext projection
            (m = 32, N1 = N2 = 8): keys, encryption, 7 hoisted baby rotations, 64-term MAC, 7 giant rotations,
            conj, rescale.
  qkv_block one complete BERT-base QKV output block at P16 (N = 2^16, L = 8): the full baby-step bank (2 inputs x
            31 hoisted rotations), the 8 giant units of block 0 (8 x 64 plaintext MAC terms, 7 giant rotations),
            ModDown, conj, merged ModDown + rescale.  Keys and plaintext encodings are made before the timer.

Usage: python tools/oracle_baseline.py [--threads N] [--which config1,qkv_block] -> one JSON line.
Without --threads it re-runs itself with OMP_NUM_THREADS=1 and =nproc and prints both.
"""
import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def config1():
    import synth
    from oracle import ckks as O
    from oracle import kernels as K
    P = O.Params("P12")
    plan = K.ProjPlan(P.n, 32, 64, 64, N1=8)
    rots = [q * 32 for q in range(1, 8)] + [p * 8 * 32 for p in range(1, 8)]
    t0 = time.time()
    keys = O.Keys(P, synth.SEED_KEYS, galois=[O.galois_rot(P, r) for r in rots] + [O.galois_conj(P)])
    X = synth.fixed_point_uniform((32, 64), synth.seed_data(1))
    W = synth.uniform((64, 64), synth.seed_data(1) + 100, -0.125, 0.125)
    xs = [O.encrypt_sk(P, keys, O.encode(P, z, 2.0 ** 40, 3), synth.seed_enc(u)) for u, z in enumerate(K.proj_inputs(X, plan))]
    pts = {(b, p, u, q): O.encode(P, K.proj_weight_slots(W, plan, b, p, u, q), float(P.q[2]), 3)
           for b in range(1) for p in range(8) for u in range(1) for q in range(8)}
    t1 = time.time()
    ys = K.projection(K.Ev(P, keys, 32), plan, xs, lambda *a: pts[a])
    t2 = time.time()
    return {"setup_s": round(t1 - t0, 3), "kernel_s": round(t2 - t1, 3), "outputs": len(ys)}


def qkv_block():
    import numpy as np
    import synth
    from oracle import ckks as O
    from oracle import kernels as K
    P = O.Params("P16")
    M, D, L = 128, 768, 8
    plan = K.ProjPlan(P.n, M, D, 11 * 256)
    g = [O.galois_rot(P, q * M) for q in range(1, plan.N1)] + [O.galois_rot(P, p * plan.N1 * M) for p in range(1, plan.N2)]
    t0 = time.time()
    keys = O.Keys(P, synth.SEED_KEYS, galois=g + [O.galois_conj(P)], max_level=L)
    X = synth.fixed_point_uniform((M, D), synth.seed_data(3))
    W = synth.bert_weight((D, 11 * 256), synth.seed_data(3))
    xs = [O.encrypt_sk(P, keys, O.encode(P, z, 2.0 ** 40, L), synth.seed_enc(u)) for u, z in enumerate(K.proj_inputs(X, plan))]
    pts = {}
    for p in range(plan.N2):
        for u in range(plan.U):
            for q in range(plan.N1):
                pts[(0, p, u, q)] = O.encode(P, K.proj_weight_slots(W, plan, 0, p, u, q), float(P.q[L - 1]), L)
    t1 = time.time()
    ev = K.Ev(P, keys, M)
    y0 = K.projection_finalize(ev, plan, K.projection_partial(ev, plan, xs, lambda *a: pts[a], 0, plan.N2)[0])
    t2 = time.time()
    assert y0.L == L - 1 and np.asarray(y0.c).shape[0] == 2
    return {"setup_s": round(t1 - t0, 3), "kernel_s": round(t2 - t1, 3), "ledger": dict(ev.ledger)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--which", default="config1,qkv_block")
    a = ap.parse_args()
    if a.threads:
        out = {w: globals()[w]() for w in a.which.split(",")}
        out["threads"] = a.threads
        print(json.dumps(out), flush=True)
        return
    res = {"nproc": os.cpu_count(), "cpu": open("/proc/cpuinfo").read().split("model name")[1].split("\n")[0].strip(": ")}
    for th in (1, os.cpu_count()):
        env = dict(os.environ, OMP_NUM_THREADS=str(th))
        p = subprocess.run([sys.executable, __file__, "--threads", str(th), "--which", a.which], env=env, capture_output=True, text=True)
        res["threads_%d" % th] = json.loads(p.stdout.strip().splitlines()[-1]) if p.returncode == 0 else p.stderr[-400:]
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
