"""EncFormer (arXiv 2604.09975) CKKS linear hot path on B200: libencf (C ABI, sm_100a CUDA) + binding.

Import `paper_2604_09975_b200.encf` for the binding; it raises if libencf.so is not built (no CPU
fallback).
"""
