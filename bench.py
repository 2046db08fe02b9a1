#!/usr/bin/env python
"""bench.py -- BERT-base layer CKKS linear path of EncFormer (arXiv 2604.09975) at N = 2^16 on B200.

One "step" = one pass of the whole hot path over one BERT-base layer
(m = 128 tokens, d = 768, H = 12, d_ff = 3072) of synthetic encrypted activations:
  QKV projection (X 128x768 -> Q, K (pi_S, G8-padded) and V, L = 8 -> 7)
  -> score kernel (64 folded-diagonal S_t) -> minimal export stream (K_min(S) = 3) -> C2M export
  -> value kernel (P_fd from the MPC softmax, 3 head blocks) -> decomplexify O -> out-projection
  -> C2M export of the LN1 boundary -> FF1 (768 -> 3072) -> C2M export (GELU boundary)
  -> FF2 (3072 -> 768) -> C2M export (LN2 boundary).
Inputs that arrive from the MPC side (P_fd, the FF1 and FF2 activations) are fresh encryptions made
before the timed region (their MPC producers are out of scope).  Weights are random BERT-init,
encoded once (model state, resident in HBM).

Contract: python bench.py --gpus N --steps K --warmup W [--impl reference] [--workload layer|qkv|ks]
prints ONE JSON line on rank 0.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

M, D, H, DH, DFF = 128, 768, 12, 64, 3072
PROF_KERNELS = ["diag_mac", "ks_inner", "ks_psi", "ks_rotsum", "ks_rma", "ntt", "bcast_mac", "add_kernel", "add_i_batch_kernel", "automorph_kernel", "bconv_batch_kernel", "bconv_kernel",
                "export_mask_kernel", "gather_copy_kernel", "masked_sum_kernel", "mod_reduce_kernel",
                "moddown_finish_batch_kernel", "moddown_finish_kernel", "mul_i_kernel", "mul_kernel",
                "rescale_finish_batch_kernel", "rescale_prep_batch_kernel", "sum_csr_kernel", "tensor_csr_kernel",
                "tensor_acc_kernel", "rescale_prep_kernel", "rescale_finish_kernel"]
L_QKV, L_V_P, L_FF = 8, 5, 3
C_QK, BETA = 192, 16
# layer shapes: BERT-base and the NEXT-row second workload BERT-large; C_qk = 192 used
# segments of 256 = 16 channels x 12 heads (base) / 12 channels x 16 heads (large), all phases 0 (G8)
MODELS = {"layer": dict(name="bert-base-layer", d=768, H=12, dff=3072),
          "qkv": dict(name="bert-base-qkv", d=768, H=12, dff=3072),
          "bert-large-layer": dict(name="bert-large-layer", d=1024, H=16, dff=4096)}
NTT_TRAFFIC = 1.873e6  # ncu dram__bytes (read + write) per limb transform (fwd cols+rows, 384-limb batch)
NTT_TRAFFIC_SRC = "profiles/r02s4_ncu_top_kernels.md (ncu --set full, 384-limb forward batch: (348.4 + 371.0) MB / 384)"
DIAG_MAC_TRAFFIC_SRC = ("profiles/r02s4_ncu_top_kernels.md (ncu --set full of the QKV launches: narrow 21142.9 + 647.0 MB) and "
                        "profiles/r02_ncu_top_kernels.md (128-bit 3020.9 + 93.2 MB)")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="layer", choices=["layer", "qkv", "ks", "gpt2-linear", "bert-large-layer"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-pipeline", action="store_true", help="e2e: copies serialised with each step (one graph)")
    ap.add_argument("--no-cpu-baseline", action="store_true", help="skip the oracle timing (A/B kernel experiments only)")
    ap.add_argument("--replicas", action="store_true",
                    help="N > 1: one independent layer per GPU (weak scaling) instead of ONE layer sharded over the N GPUs")
    ap.add_argument("--ablation", default=None, choices=[None, "wo-scp"],
                    help="wo-scp: insert the Halevi-Shoup RMA repack at the three FHE->FHE edges (App. G; Table 11 ablation)")
    return ap.parse_args()


# ------------------------------------------------------------------------------------ clocks
class Clocks:
    """SM clock / throttle-reason sampling DURING the timed region (B200_PROFILING.md clocks line): NVML every 50 ms,
    nvidia-smi -lms 200 when NVML is unavailable."""

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self.proc = None
        self.nvml = False

    def _nvml_loop(self):
        import pynvml as nv
        h = nv.nvmlDeviceGetHandleByIndex(self.index)
        bits = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap]
        while not self.stop:
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.rows.append([str(self.index), str(sm), str(mx), "", hex(rs)] +
                                 ["Active" if rs & b else "Not Active" for b in bits])
            except Exception:
                pass
            time.sleep(0.05)

    def __enter__(self):
        # NVML in a thread, every 50 ms (the nvidia-smi -lms loop takes ~1 s to start and may miss a ~1 s region)
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.stop = False
            self.t = threading.Thread(target=self._nvml_loop, daemon=True)
            self.t.start()
            self.nvml = True
            self.start = 0
            return self
        except Exception:
            self.nvml = False
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + q, "--format=csv,noheader,nounits",
                                          "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi needs ~1 s to start sampling: wait for its first row so that the (~1 s) timed region is sampled,
            # and keep only the rows taken from here on
            t0 = time.time()
            while not self.rows and time.time() - t0 < 10 and self.proc.poll() is None:
                time.sleep(0.02)
        except Exception:
            self.proc = None
        self.start = len(self.rows)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if getattr(self, "nvml", False):
            self.stop = True
            self.t.join(timeout=1)
            return
        if self.proc:
            t0 = time.time()
            while len(self.rows) <= self.start and time.time() - t0 < 0.5:   # at least one row inside the region
                time.sleep(0.01)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = self.rows[getattr(self, "start", 0):]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        self.rows = rows
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 5 + i and r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ------------------------------------------------------------------------------------ distributed plumbing
def dist_init(args):
    import torch
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return ws, rank, local


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x, ws):
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ------------------------------------------------------------------------------------ the layer
class Layer:
    """BERT-base layer state on one GPU: context, keys, plans, encoded weights, synthetic inputs."""

    ablation = None

    def __init__(self, device, workload, seed_off=0, ablation=None):
        import torch
        import synth
        from paper_2604_09975_b200 import encf as E
        from paper_2604_09975_b200 import packing as PK
        self.E, self.PK, self.torch = E, PK, torch
        self.workload = workload
        ctx = self.ctx = E.Context("P16", device)
        n = ctx.n
        self.sc = 2.0 ** 40
        t0 = time.time()
        if workload == "gpt2-linear":
            return self._init_gpt2(device, seed_off, t0)
        mdl = MODELS[workload]
        D, H, DFF = mdl["d"], mdl["H"], mdl["dff"]
        self.d, self.H, self.dff = D, H, DFF
        self.full = workload != "qkv"
        nblk = 2 * -(-(H * DH) // C_QK) + -(-D // 256)
        self.qkv = E.ProjPlan(ctx, M, D, nblk * 256)
        galois = set(self.qkv.galois())
        if self.full:
            self.attn = E.AttnPlan(ctx, M, H, DH, C_qk=C_QK, beta=BETA)
            self.oproj = E.ProjPlan(ctx, M, D, D)
            self.ff1 = E.ProjPlan(ctx, M, D, DFF)
            self.ff2 = E.ProjPlan(ctx, M, DFF, D)
            for pl in (self.oproj, self.ff1, self.ff2):
                galois |= set(pl.galois())
            galois |= set(self.attn.galois())
        galois.add(ctx.galois_conj())
        self.ablation = ablation
        if ablation == "wo-scp":
            galois |= {ctx.galois_rot(1 << k) for k in range(M.bit_length() - 1)}
        self.keys = ctx.keygen(synth.SEED_KEYS, galois=sorted(galois), relin=True, max_level=L_QKV)
        self.n_keys = len(galois) + 1
        # weights (BERT init, clipped), pre-permuted (pi_S + G8 padding for Q/K, head-major V)
        WQ, WK, WV = (synth.bert_weight((D, D), synth.seed_data(3) + i) for i in range(3))
        Wqkv, nqk, nv = PK.qkv_weight(WQ, WK, WV, H, DH, 256, C_QK)
        self.nqk = nqk
        self.w_qkv = self.qkv.encode_weights(Wqkv, L_QKV)
        self.wsc_qkv = float(ctx.q[L_QKV - 1])
        if self.full:
            self.w_o = self.oproj.encode_weights(synth.bert_weight((D, D), synth.seed_data(5) + 3), L_V_P - 2)
            self.w_1 = self.ff1.encode_weights(synth.bert_weight((D, DFF), synth.seed_data(5) + 4), L_FF)
            self.w_2 = self.ff2.encode_weights(synth.bert_weight((DFF, D), synth.seed_data(5) + 5), L_FF)
        torch.cuda.synchronize()
        self.setup_s = time.time() - t0
        # synthetic client inputs (encrypted before the timed region)
        X = synth.fixed_point_uniform((M, D), synth.seed_data(3) + seed_off)
        self.host_inputs = {"x": [self._enc(z, L_QKV, 10 + i) for i, z in enumerate(PK.complexified_inputs(X, M, 256, n))]}
        if self.full:
            P = synth.attention_probs(H, M, synth.seed_data(4) + seed_off)
            # P_fd (the M2C import of the softmax output) at Delta * 2^7 (DESIGN.md R-PSCALE)
            self.host_inputs["p"] = [self._enc(z, L_V_P, 20 + i, scale=self.sc * 2.0 ** 7)
                                     for i, z in enumerate(PK.folded_diag_blocks(P, M, self.attn.H_blk, self.attn.seg_stride, n))]
            X1 = synth.fixed_point_uniform((M, D), synth.seed_data(5) + seed_off)
            self.host_inputs["f1"] = [self._enc(z, L_FF, 30 + i) for i, z in enumerate(PK.complexified_inputs(X1, M, 256, n))]
            X2 = synth.fixed_point_uniform((M, DFF), synth.seed_data(6) + seed_off, 0.0, 1.0)
            self.host_inputs["f2"] = [self._enc(z, L_FF, 40 + i) for i, z in enumerate(PK.complexified_inputs(X2, M, 256, n))]
        self.dev_inputs = {k: [self._to_dev(h) for h in v] for k, v in self.host_inputs.items()}
        self.h2d_bytes = sum(h[0].nbytes for v in self.host_inputs.values() for h in v)
        self.Lconv = ctx.l_conv()
        self.mask_seed = synth.seed_mask(0)

    def _init_gpt2(self, device, seed_off, t0):
        """Config 5 (BASELINE configs[4]): GPT-2 small linear path, m = 256 tokens (N_seg = 128, C = 128):
        QKV 768 -> 2304 (U = 3, B_out = 18) at L = 8; out-projection on the (decomplexified) attention output
        O at L = 5 (U = 3); FF1 768 -> 3072 and FF2 3072 -> 768 at L = 3; complexify + C2M export of the LN1
        (3), GELU (12) and LN2 (3) boundary tensors at L_conv (SURVEY 8d cfg 5; attention itself is the
        optional part of cfg 5 and is not in this step).  Inputs arriving from the MPC side (O, FF1/FF2
        activations) are fresh encryptions made before the timed region."""
        import synth
        E, PK, ctx, torch = self.E, self.PK, self.ctx, self.torch
        m, d, dff, n = 256, 768, 3072, ctx.n
        C = n // m
        self.m = m
        self.qkv = E.ProjPlan(ctx, m, d, 3 * d)
        self.oproj = E.ProjPlan(ctx, m, d, d)
        self.ff1 = E.ProjPlan(ctx, m, d, dff)
        self.ff2 = E.ProjPlan(ctx, m, dff, d)
        galois = set()
        for pl in (self.qkv, self.oproj, self.ff1, self.ff2):
            galois |= set(pl.galois())
        galois.add(ctx.galois_conj())
        self.keys = ctx.keygen(synth.SEED_KEYS, galois=sorted(galois), relin=True, max_level=L_QKV)
        self.n_keys = len(galois) + 1
        Wqkv = np.concatenate([synth.bert_weight((d, d), synth.seed_data(5) + i) for i in range(3)], axis=1)
        self.w_qkv = self.qkv.encode_weights(Wqkv, L_QKV)
        self.wsc_qkv = float(ctx.q[L_QKV - 1])
        self.w_o = self.oproj.encode_weights(synth.bert_weight((d, d), synth.seed_data(5) + 13), 5)
        self.w_1 = self.ff1.encode_weights(synth.bert_weight((d, dff), synth.seed_data(5) + 14), L_FF)
        self.w_2 = self.ff2.encode_weights(synth.bert_weight((dff, d), synth.seed_data(5) + 15), L_FF)
        torch.cuda.synchronize()
        self.setup_s = time.time() - t0
        X = synth.fixed_point_uniform((m, d), synth.seed_data(5) + seed_off)
        Oa = synth.fixed_point_uniform((m, d), synth.seed_data(5) + 100 + seed_off)
        X1 = synth.fixed_point_uniform((m, d), synth.seed_data(5) + 200 + seed_off)
        X2 = synth.fixed_point_uniform((m, dff), synth.seed_data(5) + 300 + seed_off, 0.0, 1.0)
        self.host_inputs = {"x": [self._enc(z, L_QKV, 10 + i) for i, z in enumerate(PK.complexified_inputs(X, m, C, n))],
                            "o": [self._enc(z, 5, 50 + i) for i, z in enumerate(PK.complexified_inputs(Oa, m, C, n))],
                            "f1": [self._enc(z, L_FF, 60 + i) for i, z in enumerate(PK.complexified_inputs(X1, m, C, n))],
                            "f2": [self._enc(z, L_FF, 70 + i) for i, z in enumerate(PK.complexified_inputs(X2, m, C, n))]}
        self.dev_inputs = {k: [self._to_dev(h) for h in v] for k, v in self.host_inputs.items()}
        self.h2d_bytes = sum(h[0].nbytes for v in self.host_inputs.values() for h in v)
        self.Lconv = ctx.l_conv()
        self.mask_seed = synth.seed_mask(0)

    def _enc(self, z, L, seed, scale=None):
        """Client-side encryption; returns (pinned host words, scale)."""
        ct = self.ctx.encrypt(self.keys, self.ctx.encode(z, scale or self.sc, L), seed)
        return (ct.data.cpu().pin_memory(), ct.n_comp, ct.n_limbs, ct.scale)

    def _to_dev(self, h):
        words, nc, nl, sc = h
        return self.E.Ciphertext(words.to(self.ctx.device), nc, nl, sc, 1)

    def upload(self):
        return {k: [self.E.Ciphertext(h[0].to(self.ctx.device, non_blocking=True), h[1], h[2], h[3], 1) for h in v]
                for k, v in self.host_inputs.items()}

    MASK_EPOCH = 1 << 32

    def _export(self, cts, sid):
        """C2M export: ciphertext i of boundary `sid` draws its mask from stream (epoch 2^32 + sid + i) with the
        (seed, base) read from a DEVICE buffer that every step advances by one epoch (also inside the replayed CUDA
        graph), so no one-time pad is ever reused across inferences."""
        if not cts:
            return []
        if getattr(self, "mask_state", None) is None:
            self.mask_state = {}
        if sid not in self.mask_state:
            self.mask_state[sid] = self.torch.tensor([self.mask_seed, sid], dtype=self.torch.int64, device=self.ctx.device)
        return self.ctx.export_c2m_many(cts, self.Lconv, self.mask_state[sid], 0)

    def _advance_masks(self):
        for t in (getattr(self, "mask_state", None) or {}).values():
            t[1:].add_(self.MASK_EPOCH)

    def _complex_pairs(self, ys):
        h = len(ys) // 2
        out = self.ctx.complexify_many(ys[0:2 * h:2], ys[1:2 * h:2]) if h else []
        if len(ys) % 2:
            out.append(ys[-1])
        return out

    def _mark(self, name):
        if self.marks is not None:
            e = self.torch.cuda.Event(enable_timing=True)
            e.record(self.torch.cuda.current_stream())
            self.marks.append((name, e))

    marks = None

    def step(self, inp):
        """One pass of the hot path.  Returns the exported (masked ct, server share) list."""
        ctx, keys = self.ctx, self.keys
        self._mark("start")
        y = self.qkv.matmul(keys, inp["x"], self.w_qkv, self.wsc_qkv)
        self._mark("qkv")
        if self.workload == "gpt2-linear":
            ex = [(c.data, None) for c in y]          # Q, K, V stay encrypted for the (optional) attention
            yo = self.oproj.matmul(keys, inp["o"], self.w_o, float(ctx.q[4]))
            ex += self._export(self._complex_pairs(yo), 100)
            self._mark("out_proj")
            g1 = self.ff1.matmul(keys, inp["f1"], self.w_1, float(ctx.q[L_FF - 1]))
            ex += self._export(self._complex_pairs(g1), 200)
            self._mark("ff1")
            g2 = self.ff2.matmul(keys, inp["f2"], self.w_2, float(ctx.q[L_FF - 1]))
            ex += self._export(self._complex_pairs(g2), 300)
            self._mark("ff2")
            self._advance_masks()
            return ex
        if self.workload == "qkv":
            return [(c.data, None) for c in y]
        nqk = self.nqk
        Q, K, V = y[:nqk], y[nqk:2 * nqk], y[2 * nqk:]
        if self.ablation == "wo-scp":       # edges (1) QKV -> score and (2) QKV -> value (App. G), cost only
            ctx.repack_rma(keys, Q + K + V, M)
        S = self.attn.score(keys, Q, K)
        self._mark("score")
        ex = self._export(self.attn.export_stream(keys, S), 0)
        self._mark("score_export")
        O = self.attn.value(keys, inp["p"], V)
        if self.ablation == "wo-scp":       # edge (3) value -> out-projection
            ctx.repack_rma(keys, O, M)
        self._mark("value")
        Ore = ctx.decomplexify(keys, O)    # decomplexify the value output (G11): Re o = (o + conj o) / 2, batched
        xo = self._complex_pairs(Ore)
        yo = self.oproj.matmul(keys, xo, self.w_o, float(ctx.q[xo[0].n_limbs - 1]))
        ex += self._export(self._complex_pairs(yo), 100)
        self._mark("out_proj")
        g1 = self.ff1.matmul(keys, inp["f1"], self.w_1, float(ctx.q[L_FF - 1]))
        ex += self._export(self._complex_pairs(g1), 200)
        self._mark("ff1")
        g2 = self.ff2.matmul(keys, inp["f2"], self.w_2, float(ctx.q[L_FF - 1]))
        ex += self._export(self._complex_pairs(g2), 300)
        self._mark("ff2")
        self._advance_masks()                # next inference: fresh C2M masks (device-side, captured in the graph)
        return ex

    def download(self, outs):
        host = [(m.data.cpu(), s.cpu() if s is not None else None) for m, s in outs]
        return sum(a.numel() * 8 + (b.numel() * 8 if b is not None else 0) for a, b in host)


def run_ours(args):
    import torch
    if args.workload == "ks":
        return run_ks(args)
    ws, rank, local = dist_init(args)
    torch.cuda.set_device(local)
    if ws > 1 and args.workload in ("layer", "bert-large-layer") and not args.replicas:
        return run_sharded(args, ws, rank, local)
    layer = Layer(local, args.workload, seed_off=rank, ablation=args.ablation)
    ctx = layer.ctx
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        layer.step(layer.dev_inputs)
    torch.cuda.synchronize()
    # untimed pass with every kernel instrumented: per-kernel breakdown of one step
    ctx.profile("*")
    layer.step(layer.dev_inputs)
    torch.cuda.synchronize()
    breakdown = {k: ctx.profile_read(k) for k in PROF_KERNELS}
    ctx.profile(None)
    layer.marks = []
    layer.step(layer.dev_inputs)
    torch.cuda.synchronize()
    phase_ms = {layer.marks[i][0]: round(layer.marks[i - 1][1].elapsed_time(layer.marks[i][1]), 3) for i in range(1, len(layer.marks))}
    layer.marks = None
    # the step is captured ONCE into a CUDA graph (host enqueue of ~3000 launches would otherwise cost as much
    # as the device time); the graph carries CUDA-event nodes around every NTT / diag_mac launch (live roofline)
    from paper_2604_09975_b200.graphs import GraphedStep
    ctx.stats_reset()
    ctx.profile("ntt,diag_mac")
    h0 = time.time()
    gstep = GraphedStep(layer.step, layer.dev_inputs)
    capture_s = time.time() - h0
    ctx.profile(None)
    stats = ctx.stats()                 # counts of ONE step (the captured one)
    for _ in range(2):
        gstep()
    torch.cuda.synchronize()
    prof = {"diag_mac": [0.0, 0, 0], "ntt": [0.0, 0, 0]}
    barrier(ws)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ncu_region = bool(os.environ.get("ENCF_NCU_REGION"))   # ncu --profile-from-start off: launch list of the timed steps
    with Clocks(local) as clk:
        if ncu_region:
            torch.cuda.profiler.start()
        ev0.record(stream)
        h0 = time.time()
        for _ in range(args.steps):
            gstep()
            for k in prof:              # this replay's event nodes (waits for the replay to finish)
                a = ctx.profile_read(k, keep=True)
                for i in range(3):
                    prof[k][i] += a[i]
        host_enqueue_ms = (time.time() - h0) * 1e3 / args.steps
        ev1.record(stream)
        torch.cuda.synchronize()
        if ncu_region:
            torch.cuda.profiler.stop()
    barrier(ws)
    ms_total = ev0.elapsed_time(ev1)
    ms_total = max_over_ranks(ms_total, ws)
    ms_step = ms_total / args.steps
    stats = {k: v * args.steps for k, v in stats.items()}
    ctx.profile_read("ntt")
    ctx.profile_read("diag_mac")
    # e2e through the public API: per step, H2D of the step's encrypted inputs from pinned memory into the
    # graph's static inputs, the step, D2H of every exported (masked ciphertext, server share) to pinned memory
    e2e = None
    if not args.no_e2e:
        # two graphs on two static input sets (PipelinedStep): step i+1's H2D and step i's D2H run on side streams
        # under step i's device work; every copy of every step stays inside the timed region
        from paper_2604_09975_b200.graphs import PipelinedStep
        inputs_b = {k: [layer.E.Ciphertext(c.data.clone(), c.n_comp, c.n_limbs, c.scale, c.ntt) for c in v]
                    for k, v in layer.dev_inputs.items()}
        pipe = PipelinedStep(layer.step, gstep, inputs_b) if not args.no_pipeline else None
        def pinned_outs(g):
            return [(torch.empty(m.data.shape, dtype=m.data.dtype, pin_memory=True),
                     torch.empty(sh.shape, dtype=sh.dtype, pin_memory=True) if sh is not None else None) for m, sh in g.outputs]
        outs_h = [pinned_outs(gstep), pinned_outs(pipe.g[1]) if pipe else None]   # per input set
        d2h = sum(a.numel() * 8 + (b.numel() * 8 if b is not None else 0) for a, b in outs_h[0])
        host_in = {k: [h[0] for h in v] for k, v in layer.host_inputs.items()}
        if pipe:   # warm-up: the first replay of graph B uploads it to the device (not part of a step)
            pipe.run(host_in, outs_h, 2)
        torch.cuda.synchronize()
        barrier(ws)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with Clocks(local) as clk_e2e:
            e0.record(stream)
            if pipe:
                pipe.run(host_in, outs_h, args.steps)
            else:
                for _ in range(args.steps):
                    outs = gstep(host_in)
                    for (m, sh), (hm, hs) in zip(outs, outs_h[0]):
                        hm.copy_(m.data, non_blocking=True)
                        if sh is not None:
                            hs.copy_(sh, non_blocking=True)
            e1.record(stream)
            torch.cuda.synchronize()
        e_ms = max_over_ranks(e0.elapsed_time(e1), ws) / args.steps
        e2e = {"value": round(e_ms / ws, 3), "unit": "ms/layer", "h2d_bytes_per_step": layer.h2d_bytes, "d2h_bytes_per_step": d2h,
               "path": ("PipelinedStep: two CUDA graphs on two input sets; H2D(pinned) of step i+1 and D2H(pinned) of step i "
                        "on side streams under step i" if pipe else "GraphedStep: H2D(pinned) -> graph replay -> D2H(pinned), per step"),
               "clocks": clk_e2e.summary()}
    if rank != 0:
        return
    import json as _j
    peaks = _j.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    hbm = peaks.get("hbm_gbs", 6650.0)
    mac_ms, mac_n, mac_b = prof["diag_mac"]
    ntt_ms, ntt_n, ntt_bytes = prof["ntt"]
    achieved = (mac_b / mac_n) / ((mac_ms / mac_n) * 1e-3) / 1e9 if mac_n else 0.0
    # dominant kernel by time: the NTT, bound by arithmetic pipes.  Algorithmic work =
    # butterflies (N/2 log2 N per limb transform).  Peak for the step's own limb mix, from SASS op counts per
    # butterfly and the measured unit rates (tools/micro/pipes.cu, profiles/r01_pipes_micro.txt):
    #   FP64 path (q < 2^41): 8 DFMA/DMUL/DADD per butterfly at 64 lanes/clk/SM  -> 8 butterflies/clk/SM
    #   integer path (60-bit q): 6.4 half-rate IMAD.WIDE/HI + 10.3 full-rate IMAD-family -> 2.77 butterflies/clk/SM
    limb_ntts = ntt_bytes / (65536 * 8 * 4)                  # the library counts 4 limb-polys of traffic per limb transform
    bpl = (65536 // 2) * 16
    bfly = limb_ntts * bpl
    ntt_achieved = bfly / (ntt_ms * 1e-3) / 1e9 if ntt_ms else 0.0
    sm_mhz = peaks.get("sm_max_mhz", 1965.0)
    n_fp = stats["limb_ntt_fp64"] / args.steps
    n_all = stats["limb_ntt"] / args.steps
    rate_fp, rate_int = 148 * 8.0 * sm_mhz * 1e6, 148 * 2.77 * sm_mhz * 1e6          # butterflies / s
    t_peak = bpl * (n_fp / rate_fp + (n_all - n_fp) / rate_int)
    ntt_peak = bpl * n_all / t_peak / 1e9 if n_all else 1.0
    ntt_peak_hw = 148 * (63.0 / 10.0) * sm_mhz * 1e6 / 1e9     # 10 IMAD-class ops per butterfly
    ks_total = stats["keyswitch"] / args.steps
    line = {
        "metric": "BERT-base layer CKKS linear latency (ms) & key-switches/s at N=2^16; HBM roofline %",
        "value": round(ms_step / ws, 3),
        "unit": "ms/layer",
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_step, 3),
        "higher_is_better": False,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "u64",
        "data": "synthetic (seeded; BERT-init random weights; encrypted U[-1,1] F=13 activations)",
        "config": {"workload": {"layer": "bert-base-layer", "qkv": "bert-base-qkv", "gpt2-linear": "gpt2-small-linear-path",
                                "bert-large-layer": "bert-large-layer"}[args.workload],
                   "N": 65536, "m": getattr(layer, "m", M), "d": getattr(layer, "d", D), "H": getattr(layer, "H", H),
                   "d_ff": getattr(layer, "dff", DFF),
                   "levels": {"qkv": L_QKV, "p_fd": L_V_P, "out_proj": 5 if args.workload == "gpt2-linear" else L_V_P - 2,
                              "ff": L_FF, "conv": layer.Lconv},
                   "params": "P16 (q0 60b + 23x40b, K=6 x 60b special, alpha=8)",
                   "parallelism": "replicas: one independent layer per GPU" if ws > 1 else "1 GPU",
                   "ablation": args.ablation,
                   "l2": "no flush: per-step working set (~%d GB of plaintext diagonals) >> 126 MB L2" % round(
                       (layer.w_qkv.numel() + sum(getattr(layer, w).numel() for w in ("w_o", "w_1", "w_2") if hasattr(layer, w))) * 8 / 1e9)},
        "key_switches_per_s": round(ks_total / (ms_step * 1e-3), 1),
        "key_switches_per_step": ks_total,
        "gpu_launches": int(stats["kernel_launches"]),
        "kernel_time_ms_per_step": {k: round(v[0], 3) for k, v in sorted(breakdown.items(), key=lambda kv: -kv[1][0]) if v[1]},
        "kernel_time_sum_ms_per_step": round(sum(v[0] for v in breakdown.values()), 3),
        "kernel_calls_per_step": {k: v[1] for k, v in breakdown.items() if v[1]},
        "phase_ms": phase_ms,
        "limb_ntt_per_step": stats["limb_ntt"] // args.steps,
        "host_enqueue_ms_per_step": round(host_enqueue_ms, 3),
        "execution": "CUDA graph of the whole step (captured once in %.2f s), replayed per step" % capture_s,
        "roofline": {"bound": "alu", "kernel": "ntt (ntt_cols_r + ntt_rows_r)", "achieved": round(ntt_achieved, 1),
                     "peak": round(ntt_peak_hw, 1), "unit": "Gbutterfly/s", "frac": round(ntt_achieved / ntt_peak_hw, 4),
                     "peak_source": "SURVEY 8(d) ALU model: a 64-bit Shoup butterfly = 10 IMAD-class ops at the MEASURED 63 "
                                    "IMAD lanes/clk/SM (profiles/r01_pipes_micro.txt) x 148 SMs x sm_max_mhz -- independent of the "
                                    "kernel's own instruction mix",
                     "peak_kernel_op_mix": round(ntt_peak, 1), "frac_kernel_op_mix": round(ntt_achieved / ntt_peak, 4),
                     "us_per_limb_transform": round(ntt_ms / args.steps * 1e3 / n_all, 4) if n_all else None,
                     "traffic": NTT_TRAFFIC, "traffic_source": NTT_TRAFFIC_SRC, "share_of_step": round(ntt_ms / args.steps / ms_step, 3),
                     "limb_transforms_per_step": {"fp64_path": n_fp, "int_path": n_all - n_fp},
                     "hbm_floor_frac": round((limb_ntts * 4 * 65536 * 8 / (ntt_ms * 1e-3) / 1e9) / hbm, 4) if ntt_ms else None,
                     "note": "dominant kernel by device time; achieved = NTT butterflies (N/2 log2 N per limb) / CUDA-event time of "
                             "every transform in the timed steps (graph event nodes); peak = the step's limb mix at the pipe bound: "
                             "FP64-path limbs 8 butterflies/clk/SM (8 fp64-pipe ops each), integer-path limbs 2.77/clk/SM "
                             "(fmaheavy-bound), x 148 SMs x sm_max_mhz (DESIGN.md ALU roofline); hbm_floor_frac = the 4 limb-poly "
                             "passes per transform against the measured HBM peak; traffic = ncu dram bytes per limb transform "
                             "(profiles/r02_ncu_top_kernels.md)"},
        "roofline_hbm": {"bound": "hbm", "kernel": "diag_mac", "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
                         "frac": round(achieved / hbm, 4), "traffic": 24.9e9 if args.workload in ("layer", "qkv") else None,
                         "traffic_source": DIAG_MAC_TRAFFIC_SRC,
                         "note": "the HBM-bound plaintext-diagonal MAC: algorithmic bytes per launch (plaintext stream + bank + "
                                 "accumulators) / CUDA-event duration; peak = MEASURED_PEAKS.json hbm_gbs (burst copy); traffic = "
                                 "ncu dram read+write bytes of the QKV launches (24.8 GB algorithmic; profiles/r02_ncu_top_kernels.md)"},
        "clocks": clk.summary(),
        "e2e": e2e,
        "setup_s": round(layer.setup_s, 1),
    }
    if args.workload in ("layer", "bert-large-layer"):
        parts = layer_model_bytes(ctx.N, ctx.K, ctx.alpha, None,
                                  [("qkv", layer.qkv, L_QKV), ("out_proj", layer.oproj, L_V_P - 2), ("ff1", layer.ff1, L_FF),
                                   ("ff2", layer.ff2, L_FF)], layer.attn, {"score": L_QKV - 1, "p": L_V_P, "v": L_QKV - 1})
        tot = sum(parts.values())
        kb = stats["alg_bytes"] / args.steps
        line["roofline_layer"] = {
            "bound": "hbm", "achieved": round(tot / (ms_step * 1e-3) / 1e9, 1), "peak": hbm, "unit": "GB/s",
            "frac": round(tot / (ms_step * 1e-3) / 1e9 / hbm, 4), "alg_bytes_per_layer": int(tot),
            "alg_bytes_by_part": {k: int(v) for k, v in parts.items()},
            "at_peak_ms": round(tot / (hbm * 1e9) * 1e3, 3),
            "kernel_counted_bytes_per_layer": int(kb), "kernel_counted_frac": round(kb / (ms_step * 1e-3) / 1e9 / hbm, 4),
            "note": "the metric's 'HBM roofline %': SURVEY 8(d) algorithmic bytes of the whole layer (plaintext diagonals, keys, "
                    "ciphertexts the METHOD must move) / measured ms per layer vs MEASURED_PEAKS hbm_gbs; kernel_counted = the "
                    "library's own per-launch algorithmic-byte counters (encf_stats alg_bytes: includes the NTT passes)"}
        try:
            line["ks_config2"] = ks_config2(ctx, 0x5EED, hbm)
        except Exception as e:       # the microbench is an extra key; never lose the main line
            line["ks_config2"] = {"error": str(e)[:200]}
    line["cpu_baseline"] = None if args.no_cpu_baseline else cpu_baseline(layer, stats, args.steps)
    print(json.dumps(line), flush=True)


def run_sharded(args, ws, rank, local):
    """ONE BERT layer sharded over the ws GPUs (paper_2604_09975_b200/layer.py): projection (b, p) units
    with weight-stream shards + an extended-basis uint64 NCCL all-reduce, score t-ranges + all-gather, value
    (block, t) partials + all-reduce, owner finalisation + all-gathers.  value = per-layer latency (max over
    ranks), strong scaling (the layer is fixed as N grows).  The step, collectives included, is captured into a
    CUDA graph when NCCL allows it (else replayed eagerly, said in the JSON)."""
    import torch
    from paper_2604_09975_b200 import layer as LY
    spec = LY.BERT_BASE if args.workload == "layer" else LY.BERT_LARGE
    t0 = time.time()
    layer = LY.ShardedLayer(spec, local, LY.Comm(None))
    setup_s = time.time() - t0
    stream = torch.cuda.current_stream()
    for _ in range(max(args.warmup, 1)):
        layer.step(layer.dev_inputs)
    torch.cuda.synchronize()
    ctx = layer.ctx
    ctx.stats_reset()
    mode = "cuda-graph"
    try:
        from paper_2604_09975_b200.graphs import GraphedStep
        gstep = GraphedStep(layer.step, layer.dev_inputs)
        run = gstep
    except Exception as e:          # NCCL capture unavailable: eager replay
        mode = "eager (graph capture failed: %s)" % str(e)[:120]
        torch.cuda.synchronize()

        def run(host=None):
            if host is not None:
                for k, hs in host.items():
                    for dst, h in zip(layer.dev_inputs[k], hs):
                        dst.data.copy_(h, non_blocking=True)
            return layer.step(layer.dev_inputs)
    stats = ctx.stats()
    for _ in range(2):
        run()
    torch.cuda.synchronize()
    barrier(ws)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            outs = run()
        ev1.record(stream)
        torch.cuda.synchronize()
    barrier(ws)
    ms_step = max_over_ranks(ev0.elapsed_time(ev1), ws) / args.steps
    e2e = None
    if not args.no_e2e:
        outs_h = [(torch.empty(m.data.shape, dtype=m.data.dtype, pin_memory=True), torch.empty(s.shape, dtype=s.dtype, pin_memory=True))
                  for _, _, (m, s) in outs]
        d2h = sum(a.numel() * 8 + b.numel() * 8 for a, b in outs_h)
        d2h = int(max_over_ranks(float(d2h), ws))
        torch.cuda.synchronize()
        barrier(ws)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            o = run({k: [h[0] for h in v] for k, v in layer.host_inputs.items()})
            for (_, _, (m, s)), (hm, hs) in zip(o, outs_h):
                hm.copy_(m.data, non_blocking=True)
                hs.copy_(s, non_blocking=True)
        e1.record(stream)
        torch.cuda.synchronize()
        e2e = {"value": round(max_over_ranks(e0.elapsed_time(e1), ws) / args.steps, 3), "unit": "ms/layer",
               "h2d_bytes_per_step": layer.h2d_bytes, "d2h_bytes_per_step": d2h,
               "path": "per rank: H2D(pinned) of the replicated client inputs -> sharded step -> D2H of this rank's exports; max over ranks"}
    if rank != 0:
        return
    line = {
        "metric": "BERT-base layer CKKS linear latency (ms) & key-switches/s at N=2^16; HBM roofline %",
        "value": round(ms_step, 3), "unit": "ms/layer", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms_step, 3), "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
        "dtype": "u64", "data": "synthetic (seeded; BERT-init random weights; encrypted U[-1,1] F=13 activations)",
        "config": {"workload": spec.name, "N": 65536, "m": spec.m, "d": spec.d, "H": spec.H, "d_ff": spec.dff,
                   "parallelism": "one layer sharded over %d GPUs: projection (b,p) units (weight shards), score t-ranges, "
                                  "value (block,t) units; NCCL uint64 all-reduce of partials + all-gather of outputs" % ws,
                   "execution": mode, "l2": "no flush: plaintext stream per rank >> 126 MB L2"},
        "key_switches_per_step_rank0": stats["keyswitch"], "gpu_launches": int(stats["kernel_launches"]),
        "clocks": clk.summary(), "e2e": e2e, "setup_s": round(setup_s, 1),
    }
    print(json.dumps(line), flush=True)


def run_ks(args):
    """Config 2 (BASELINE configs[1]): the key-switch / rotation microbench of P16 at L = 24 (dnum = 3).
    One ciphertext encrypting U[-1,1] slots; hoisted rotations by {1..N1-1}*128 slots for N1 = 32 and 16
    (one ModUp per batch), the single-KS rotation, conj and relin.  value = hoisted key switches / s
    (N1 = 32 batch, whole job over ranks); roofline = algorithmic bytes of the hoisted batch
    ((N1-1)(key(L) + ct(L)) + ct(L)) / device time vs the measured HBM peak."""
    import torch
    import synth
    from paper_2604_09975_b200 import encf as E
    ws, rank, local = dist_init(args)
    torch.cuda.set_device(local)
    ctx = E.Context("P16", local)
    L, m = 24, M
    K = ctx.K(L)
    steps32 = [k * m for k in range(1, 32)]
    galois = sorted({ctx.galois_rot(s) for s in steps32} | {ctx.galois_conj()})
    t0 = time.time()
    keys = ctx.keygen(synth.SEED_KEYS, galois=galois, relin=True, max_level=L)
    torch.cuda.synchronize()
    setup_s = time.time() - t0
    z = synth.uniform(ctx.n, synth.seed_data(2) + rank) + 1j * synth.uniform(ctx.n, synth.seed_data(2) + 1000 + rank)
    ct = ctx.encrypt(keys, ctx.encode(z, 2.0 ** 40, L), synth.seed_enc(0))
    ct3 = ctx.tensor(ct, ct)
    # correctness spot check (decrypt + decode on the GPU): left rotation by 128 slots, conj
    r = ctx.rotate_hoisted(keys, ct, steps32[:2])
    dec = ctx.decode(ctx.decrypt(keys, r[0]))
    err_rot = float(np.abs(dec - np.roll(z, -m)).max())
    decc = ctx.decode(ctx.decrypt(keys, ctx.conjugate(keys, ct)))
    err_conj = float(np.abs(decc - np.conj(z)).max())
    assert err_rot < 1e-5 and err_conj < 1e-5, (err_rot, err_conj)
    ops = {
        "hoisted_n1_32": (lambda: ctx.rotate_hoisted(keys, ct, steps32), 31),
        "hoisted_n1_16": (lambda: ctx.rotate_hoisted(keys, ct, steps32[:15]), 15),
        "rotate_single": (lambda: ctx.rotate(keys, ct, m), 1),
        "conj": (lambda: ctx.conjugate(keys, ct), 1),
        "relin": (lambda: ctx.relinearize(keys, ct3), 1),
    }
    stream = torch.cuda.current_stream()
    reps = max(args.steps, 1)
    res = {}
    with Clocks(local) as clk:
        for name, (fn, nks) in ops.items():
            for _ in range(args.warmup):
                fn()
            barrier(ws)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ctx.stats_reset()
            a.record(stream)
            for _ in range(reps):
                fn()
            b.record(stream)
            torch.cuda.synchronize()
            st = ctx.stats()
            ms = max_over_ranks(a.elapsed_time(b), ws) / reps
            res[name] = {"ms": round(ms, 4), "ks": nks, "ks_per_s": round(ws * nks / (ms * 1e-3), 1),
                         "launches": st["kernel_launches"] // reps, "limb_ntt": st["limb_ntt"] // reps}
    if rank != 0:
        return
    limb = ctx.N * 8
    dnum = -(-L // ctx.alpha)
    key_b = dnum * 2 * (L + K) * limb
    ct_b = 2 * L * limb
    hb = 31 * (key_b + ct_b) + ct_b
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    hbm = peaks.get("hbm_gbs", 6650.0)
    h = res["hoisted_n1_32"]
    achieved = hb / (h["ms"] * 1e-3) / 1e9
    line = {
        "metric": "BERT-base layer CKKS linear latency (ms) & key-switches/s at N=2^16; HBM roofline %",
        "value": round(ws * 31 / (h["ms"] * 1e-3), 1), "unit": "key-switches/s (hoisted, L=24, dnum=3)",
        "n_gpus": ws, "steps": reps, "warmup": args.warmup, "ms_per_step": h["ms"], "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic (U[-1,1] complex slots, seeded)",
        "config": {"workload": "ckks-keyswitch-microbench", "N": ctx.N, "L": L, "dnum": dnum, "alpha": ctx.alpha, "K": K,
                   "rotations": "hoisted {1..31}*128 (N1=32) and {1..15}*128 (N1=16); single rot 128; conj; relin",
                   "parallelism": "replicas" if ws > 1 else "1 GPU",
                   "l2": "no flush: 31 distinct %.1f MB keys per batch (%.1f GB) >> 126 MB L2" % (key_b / 1e6, 31 * key_b / 1e9)},
        "ops": res,
        "check": {"rot128_max_abs_err": err_rot, "conj_max_abs_err": err_conj},
        "roofline": {"bound": "hbm", "kernel": "hoisted rotation batch (N1=32)", "achieved": round(achieved, 1), "peak": hbm,
                     "unit": "GB/s", "frac": round(achieved / hbm, 4), "traffic": None,
                     "note": "algorithmic bytes 31 x (key %.1f MB + ct %.1f MB) + ct in, per batch / device time" % (key_b / 1e6, ct_b / 1e6)},
        "clocks": clk.summary(), "e2e": None, "gpu_launches": h["launches"], "setup_s": round(setup_s, 1),
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------ algorithmic bytes
def layer_model_bytes(N, K, alpha, spec, pplans, attn, L_lv):
    """Algorithmic HBM bytes of one layer from SURVEY §8(d)'s per-unit formulas (what the METHOD must move; the
    dense work it avoids and the implementation's own extra passes are not counted).  limb = N 8 B;
    ct(L) = 2 L limb, pt(L) = L limb, key(L) = dnum(L) 2 (L + K(L)) limb (K(L): the level's special primes, R-KL).
      projection: B_out U C pt(L) + 2 U N1 ct(L) + U (N1-1)(key + ct) + B_out N2 ct + B_out N2 (key + 2 ct) + B_out (ct(L) + ct(L-1))
      hoisted rotation: key(L) + ct(L) (+ ct(L) once per input); single KS: key(L) + 2 ct(L); relin: key + 5 L limb
      tensor: 2 ct(L) per operand pair + 3 L limb out; masked plaintexts pt(L) per distinct mask; export: 2 ct(Lc) + pt(Lc).
    pplans: [(plan, L)], attn: AttnPlan, L_lv: {"score": L of Q/K, "p": L of P_fd, "v": L of V, "conv": L_conv}."""
    limb = N * 8
    dnum = lambda L: -(-L // alpha)                       # noqa: E731
    ct = lambda L: 2 * L * limb                            # noqa: E731
    pt = lambda L: L * limb                                # noqa: E731
    key = lambda L: dnum(L) * 2 * (L + K(L)) * limb        # noqa: E731
    hoist = lambda n, L: n * (key(L) + ct(L)) + ct(L)      # noqa: E731
    parts = {}
    for name, pl, L in pplans:
        Bo, U, C, N1, N2 = pl.B_out, pl.U, pl.C, pl.N1, pl.N2
        parts[name] = (Bo * N2 * U * N1 * pt(L) + 2 * U * N1 * ct(L) + U * ((N1 - 1) * (key(L) + ct(L)) + ct(L))
                       + Bo * N2 * ct(L) + Bo * N2 * (key(L) + 2 * ct(L)) + Bo * (ct(L) + ct(L - 1)))
    m, B, beta, g = attn.m, attn.B, attn.beta, attn.g
    half = m // 2
    Ls = L_lv["score"]
    k_route = -(-attn.C // attn.H)
    sc = B * hoist(2 * (beta - 1), Ls) + B * hoist(2 * g, Ls)                  # Q / K Psi banks (2 rotations per shift)
    sc += half * (B * 2 * ct(Ls - 1) + 3 * (Ls - 1) * limb)                    # lazy tensor sums
    sc += half * (key(Ls - 1) + 5 * (Ls - 1) * limb)                           # one relin per t
    sc += half * hoist(k_route - 1, Ls - 2) + half * hoist(2, Ls - 2)          # routing sum + align Psi^s
    sc += half * (key(Ls - 3) + 2 * ct(Ls - 3))                                # export-stream offset rotations
    parts["score"] = sc
    Lv, Lp = L_lv["v"], L_lv["p"]
    BV, dh = attn.B_V, attn.d_h
    va = BV * hoist(2, Lv) + BV * hoist(2 * (half - 1), Lv - 1)                # uu + U bank (Psi^t)
    va += BV * hoist(dh - 1 + half - 1, Lp)                                    # Phi bank of P_fd
    va += BV * ((dh + half - 1) * ct(Lp) + dh * pt(Lp) + half * ct(Lp))        # b_t: read the bank + n_u once, write b_t
    va += BV * (half * 2 * ct(Lp - 1) + 3 * (Lp - 1) * limb + key(Lp - 1) + 5 * (Lp - 1) * limb)   # tensor + relin
    parts["value"] = va
    return parts


def ks_config2(ctx, keys_seed, hbm, reps=3):
    """Config 2 key-switches/s inside the default bench (BASELINE configs[1]): P16 at L = 24 (dnum = 3), one
    hoisted batch of 31 rotations {1..31} x 128 slots (N1 = 32).  Returns the extra keys for the JSON line."""
    import torch
    import synth
    L = 24
    steps = [k * M for k in range(1, 32)]
    keys = ctx.keygen(keys_seed, galois=sorted({ctx.galois_rot(s) for s in steps}), max_level=L)
    z = synth.uniform(ctx.n, synth.seed_data(2)) + 1j * synth.uniform(ctx.n, synth.seed_data(2) + 1000)
    ct = ctx.encrypt(keys, ctx.encode(z, 2.0 ** 40, L), synth.seed_enc(0))
    ctx.rotate_hoisted(keys, ct, steps)
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(reps):
        ctx.rotate_hoisted(keys, ct, steps)
    b.record(s)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    limb = ctx.N * 8
    key_b = 3 * 2 * (L + ctx.K(L)) * limb
    hb = 31 * (key_b + 2 * L * limb) + 2 * L * limb
    keys.close()
    gbs = hb / (ms * 1e-3) / 1e9
    return {"key_switches_per_s": round(31 / (ms * 1e-3), 1), "ms_per_batch": round(ms, 4), "L": L, "dnum": 3, "rotations": 31,
            "achieved_gbs": round(gbs, 1), "hbm_frac": round(gbs / hbm, 4),
            "note": "hoisted N1=32 batch at P16 L=24; algorithmic bytes 31 (key + ct) + ct per batch / device time vs MEASURED_PEAKS hbm_gbs"}


# ------------------------------------------------------------------------------------ CPU baseline (the oracle)
def oracle_sample():
    """Time the oracle (as it stands) on a bounded sample of the layer: one hoisted rotation and one
    single rotation at L = 8 of P16 plus one 64-term plaintext MAC unit.  Returns per-op seconds."""
    from oracle import ckks as O
    from oracle import kernels as K
    import synth
    P = O.Params("P16")
    L = L_QKV
    g = [O.galois_rot(P, 128), O.galois_rot(P, 256)]
    t0 = time.time()
    keys = O.Keys(P, synth.SEED_KEYS, galois=g, max_level=L)
    t_keys = time.time() - t0
    ct = O.encrypt_sk(P, keys, O.encode(P, synth.uniform(P.n, 1), 2.0 ** 40, L), 1)
    t0 = time.time()
    O.rotate_hoisted(P, keys, ct, [128])
    t_hoist = time.time() - t0
    t0 = time.time()
    O.rotate(P, keys, ct, 256)
    t_rot = time.time() - t0
    ev = K.Ev(P, keys, M)
    pts = [O.Pt(O.sample_uniform(5, 7 + i, P.q[:L], list(range(L)), P.N), 2.0 ** 40) for i in range(8)]
    t0 = time.time()
    ev.mac_ptmul([ct] * 8, pts)
    t_mac8 = time.time() - t0
    return {"keygen_s": t_keys, "rot_hoisted_s": t_hoist, "rot_single_s": t_rot, "ptmul_term_s": t_mac8 / 8}


def oracle_layer_counts():
    """Key switches and plaintext-product terms of one BERT-base layer from the ORACLE's own schedule run in
    count-only mode (oracle/kernels.py CountEv at N = 2^16): QKV, score + export stream, value, decomplexify,
    out-projection, FF1, FF2 -- independent of the GPU's counters."""
    from oracle import kernels as K
    n = 32768
    ev = K.CountEv(n)
    nblk = 2 * -(-(H * DH) // C_QK) + -(-D // 256)
    fake_w = lambda L: (lambda *a: K.FakeCt(L, 1.0, 1))            # noqa: E731
    for d_in, d_out, L in ((D, nblk * 256, L_QKV), (D, D, L_V_P - 2), (D, DFF, L_FF), (DFF, D, L_FF)):
        pl = K.ProjPlan(n, M, d_in, d_out)
        K.projection(ev, pl, [K.FakeCt(L)] * pl.U, fake_w(L))
    sp = K.ScorePlan(n, M, H, DH, C_qk=C_QK, beta=BETA)
    K.score_export(ev, sp, K.score(ev, sp, [K.FakeCt(L_QKV - 1)] * sp.B, [K.FakeCt(L_QKV - 1)] * sp.B))
    vp = K.ValuePlan(n, M, H, DH)
    K.value(ev, vp, [K.FakeCt(L_V_P)] * vp.B_V, [K.FakeCt(L_QKV - 1)] * vp.B_V)
    ev.ledger["conj"] += vp.B_V                     # decomplexify O (G11)
    return {"keyswitch": ev.ledger["rot"] + ev.ledger["conj"] + ev.ledger["relin"], "ptmul_terms": ev.ledger["ptmul"]}


def oracle_anchored_layer():
    """The oracle on ONE COMPLETE unit of the workload -- a BERT-base QKV output block at P16, L = 8 (the full bank:
    2 x 31 hoisted rotations; 8 giant units of 64 plaintext MAC terms; 7 giant rotations, ModDown, conj, merged
    ModDown + rescale; tools/oracle_baseline.py) on every host core -- and the layer time EXTRAPOLATED from it by the
    oracle's own schedule counts: T_layer = T_block x cost(layer) / cost(block), cost = #KS t_KS + #terms t_term with
    the per-op costs of a bounded sample (one L = 8 rotation, 8 MAC terms)."""
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import oracle_baseline
    s = oracle_sample()
    t0 = time.time()
    blk = oracle_baseline.qkv_block()
    t_block = blk["kernel_s"]
    led = blk["ledger"]
    cost = lambda ks, pt: ks * s["rot_single_s"] + pt * s["ptmul_term_s"]      # noqa: E731
    lay = oracle_layer_counts()
    c_blk = cost(led.get("rot", 0) + led.get("conj", 0) + led.get("relin", 0), led.get("ptmul", 0))
    c_lay = cost(lay["keyswitch"], lay["ptmul_terms"])
    est_ms = t_block * c_lay / c_blk * 1e3
    return est_ms, {"qkv_block_measured_s": round(t_block, 2), "qkv_block_wall_s": round(time.time() - t0, 1),
                    "block_ledger": led, "layer_counts_from_oracle_schedule": lay,
                    "per_op_sample_s": {k: round(v, 4) for k, v in s.items()},
                    "modelled_block_s": round(c_blk, 2)}


def cpu_baseline(layer, stats, steps):
    est_ms, info = oracle_anchored_layer()
    return {"value": round(est_ms, 1), "unit": "ms/layer", "cores": os.cpu_count(), "kind": "oracle",
            "sample": "one COMPLETE BERT-base QKV output block (P16, L = 8) run by the oracle on %d threads in %.1f s; the layer "
                      "value is EXTRAPOLATED from it by the oracle's own schedule counts (%d key switches, %d MAC terms per "
                      "layer; tools/oracle_baseline.py times complete config-1 and QKV-block units single-threaded too)" % (
                          os.cpu_count(), info["qkv_block_measured_s"], info["layer_counts_from_oracle_schedule"]["keyswitch"],
                          info["layer_counts_from_oracle_schedule"]["ptmul_terms"]),
            "detail": info}


def run_reference(args):
    """--impl reference: the oracle (CPU) on the same workload: each step runs one complete QKV output block and
    the layer time is extrapolated from it by the oracle's schedule counts (oracle_anchored_layer)."""
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    times, ests, info = [], [], None
    for _ in range(max(args.steps, 1)):
        t0 = time.time()
        est, info = oracle_anchored_layer()
        times.append(time.time() - t0)
        ests.append(est)
    est_ms = statistics.median(ests)
    line = {"impl": "reference", "metric": "BERT-base layer CKKS linear latency (ms) & key-switches/s at N=2^16; HBM roofline %",
            "value": round(est_ms, 1), "unit": "ms/layer", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(statistics.mean(times) * 1e3, 1), "higher_is_better": False, "scaling": "weak",
            "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": {"workload": "bert-base-layer", "N": 65536, "m": M, "d": D, "H": H, "d_ff": DFF},
            "cpu_baseline": {"value": round(est_ms, 1), "unit": "ms/layer", "cores": os.cpu_count(), "kind": "oracle",
                             "sample": "per step: one complete QKV output block (P16, L=8) on every host core; layer EXTRAPOLATED "
                                       "by the oracle's own schedule counts", "detail": info},
            "e2e": {"value": round(est_ms, 1), "unit": "ms/layer", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
