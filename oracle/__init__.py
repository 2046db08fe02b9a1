"""CPU oracle for the EncFormer CKKS hot path.  TEST INFRASTRUCTURE ONLY (see ckks.py header)."""
