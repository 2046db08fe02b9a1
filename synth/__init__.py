"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the method (no encoding, no packing, no CKKS): it only draws
plain float64 matrices with the shapes and value distributions of the paper's workloads
 and names the seeds.  Both sides (oracle/ and the CUDA library)
receive the same arrays from here; neither imports the other.
"""
import numpy as np

# Seeds (SURVEY.md 8d "Configs -> inputs").
SEED_KEYS = 0x5EED
def seed_data(cfg):
    return 0xDA7A + int(cfg)
def seed_enc(ct_id):
    return 0xE1C + int(ct_id)
def seed_mask(ct_id):
    return 0x3A5C + int(ct_id)

F_BITS = 13  # fixed-point fractional bits of the MPC side


def rng(seed):
    return np.random.Generator(np.random.PCG64(int(seed)))


def fixed_point_uniform(shape, seed, lo=-1.0, hi=1.0, f_bits=F_BITS):
    """Activations: U[lo,hi] rounded to the F=13 fixed-point grid the MPC side produces."""
    x = rng(seed).uniform(lo, hi, size=shape)
    return np.round(x * (1 << f_bits)) / (1 << f_bits)


def bert_weight(shape, seed, std=0.02, clip=0.04):
    """Weights: N(0, 0.02^2) (BERT init convention), clipped at +-0.04."""
    return np.clip(rng(seed).normal(0.0, std, size=shape), -clip, clip)


def uniform(shape, seed, lo=-1.0, hi=1.0):
    return rng(seed).uniform(lo, hi, size=shape)


def complex_slots(n, seed, amp=1.0):
    g = rng(seed)
    return amp * (g.uniform(-1, 1, n) + 1j * g.uniform(-1, 1, n))


def attention_probs(H, m, seed, power=5):
    """Post-softmax-like attention P: rows of U[0,1]^power normalised to sum 1 (MBMax-like, non-negative)."""
    a = rng(seed).uniform(0.0, 1.0, size=(H, m, m)) ** power
    return a / a.sum(axis=-1, keepdims=True)


# Workload shapes (BASELINE.json configs).
BERT_BASE = dict(m=128, d=768, H=12, d_h=64, d_ff=3072)
GPT2_SMALL = dict(m=256, d=768, H=12, d_h=64, d_ff=3072)
