"""Every alternative kernel path of libencf equals the oracle too (not only the defaults the other GPU tests run).

The switches are read once per process (static initialisers in csrc/), so each variant runs a subset of the parity
tests in a fresh interpreter with its environment:
  ENCF_BCONV_TC=0      CUDA-core base conversion instead of tcgen05 .kind::i8
  ENCF_KS_TMA=0        register-load inner products / masked shifts instead of cp.async.bulk staging
  ENCF_KS_TMA_T=256    the 256-thread TMA inner-product kernel
  ENCF_PSI_TILE=1024   1024-coefficient masked-shift tiles
  ENCF_ROTSUM_TMA=1    the cp.async.bulk ring routing sum
  ENCF_MAC_VARIANT=reg / tma1 / tma3   plaintext-MAC variants
  ENCF_NTT_FUSED=1     the fused persistent two-phase NTT
  ENCF_NTT_INT_ONLY=1  every limb on the integer NTT path (no FP64 path; includes the value kernel's 128-point
                       window transforms)
  ENCF_BCAST_DIRECT=1  the value kernel's direct sliding-window MAC instead of the 128-point window convolution
  ENCF_PROJ_GROUP=0    projection giant steps as separate ext rotations + lifts + block sums (not one grouped launch)
  ENCF_MAC_FP=0        plaintext MAC on the integer pipe only (no FP64-pipe warps)
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUBSET = ("projection_config1 or rotations_conj_bit_exact or tensor_relin or score_and_export or value_bit_exact "
          "or keyswitch_P16 or unit_split")

VARIANTS = [
    {"ENCF_BCONV_TC": "0"},
    {"ENCF_KS_TMA": "0"},
    {"ENCF_KS_TMA_T": "256", "ENCF_PSI_TILE": "1024", "ENCF_ROTSUM_TMA": "1"},
    {"ENCF_MAC_VARIANT": "reg"},
    {"ENCF_MAC_VARIANT": "tma1", "ENCF_MAC_FP": "0"},
    {"ENCF_MAC_VARIANT": "tma3"},
    {"ENCF_NTT_FUSED": "1"},
    {"ENCF_NTT_INT_ONLY": "1"},
    {"ENCF_BCAST_DIRECT": "1", "ENCF_PROJ_GROUP": "0"},
]


@pytest.mark.parametrize("env", VARIANTS, ids=lambda e: ",".join("%s=%s" % kv for kv in e.items()))
def test_variant_parity(env):
    full = dict(os.environ)
    full.update(env)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        os.path.join(ROOT, "tests", "test_gpu_parity.py"), "-k", SUBSET],
                       cwd=ROOT, env=full, capture_output=True, text=True, timeout=1500)
    tail = (r.stdout + r.stderr)[-3000:]
    assert r.returncode == 0, tail
    assert " passed" in r.stdout and "failed" not in r.stdout, tail
