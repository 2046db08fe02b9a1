// encformer.cuh -- plans and schedule entry points of the EncFormer kernels.
#pragma once
#include <algorithm>
#include <vector>
#include "eval.cuh"

struct encf_proj_plan {
    int n, m, d_in, d_out, N_seg, C, G, U, B_out, N1, N2;
    uint32_t flags;
    bool restricted;        // C < N_seg: Phi_C = RotFirst_{Cm} bank and giant fold (Alg A.4), 3 levels (R-PHIC)
};

struct encf_attn_plan {
    int n, m, H, d_h, N_seg, C, B, beta, g, n_out, H_blk, B_V, seg_stride;
    int k_route;            // ceil(C / H) channel groups folded onto the H head segments
    bool aligned;           // some block has head phase r_l = l C mod H != 0 (Align_r, App. A.3)
    std::vector<int> phases;
};

// A masked shift request on input i: rot(x; rot[0]) (.) mk[0] + rot(x; rot[1]) (.) mk[1] (Psi^t, RotFirst), or
// x (.) mk[0] alone (plain).  Masks are the descriptors of encf_mask_desc (rows [r0, r1) of segments s0 + k ss,
// k < sc, on an m-row grid).
struct MaskD { int m, r0, r1, s0, ss, sc; };
struct ShiftReq { int i; bool plain; long rot[2]; MaskD mk[2]; };
ShiftReq rotfirst_req(int i, long Ls, long tau, int m);
void shift_ext_many(Ev& ev, const std::vector<const DCt*>& xs, const std::vector<ShiftReq>& reqs, std::vector<DCt>& ly);
void shift_many(Ev& ev, const std::vector<const DCt*>& xs, const std::vector<ShiftReq>& reqs, std::vector<DCt>& outs);
void shift_sum_ext_many(Ev& ev, const std::vector<const DCt*>& xs, const std::vector<std::vector<ShiftReq>>& terms,
                        std::vector<DCt>& outs_ext);

void proj_plan_init(encf_proj_plan& p, int n, int m, int d_in, int d_out, int C, int N1, uint32_t flags);
std::vector<uint32_t> proj_galois(Ev& ev, const encf_proj_plan& p);
void proj_phase1(Ev& ev, const encf_proj_plan& p, const std::vector<DCt>& x, const u64* w /* unit u0 */, double w_scale, int u0,
                 int u1, std::vector<DCt>& accs);
void proj_finalize_many(Ev& ev, const encf_proj_plan& p, const std::vector<DCt>& accs, std::vector<DCt>& ys);

void attn_plan_init(encf_attn_plan& a, int n, int m, int H, int d_h, int C_qk, int beta, int H_blk);
std::vector<uint32_t> attn_galois(Ev& ev, const encf_attn_plan& a);
void psi_many(Ev& ev, const std::vector<const DCt*>& xs, const std::vector<std::vector<int>>& ts, int m, int seg0, int nseg,
              std::vector<std::vector<DCt>>& outs);
void score_run(Ev& ev, const encf_attn_plan& a, const std::vector<DCt>& qs, const std::vector<DCt>& ks, int t0, int t1,
               std::vector<DCt>& S);
void score_export_run(Ev& ev, const encf_attn_plan& a, const std::vector<DCt>& S, std::vector<DCt>& outs);
void value_partial_run(Ev& ev, const encf_attn_plan& a, const std::vector<DCt>& ps, const std::vector<DCt>& vs, int u0, int u1,
                       std::vector<int>& blocks, std::vector<DCt>& o3);
void value_run(Ev& ev, const encf_attn_plan& a, const std::vector<DCt>& ps, const std::vector<DCt>& vs,
               std::vector<DCt>& outs);
int l_conv_rule(const encf_ctx& c, int ell, int sigma, double scale, double B_max);
void repack_rma_run(Ev& ev, const std::vector<DCt>& xs, int m, std::vector<DCt>& outs);
void gelu_preeval_run(Ev& ev, const std::vector<DCt>& xs, const double coef[5], std::vector<DCt>& f0, std::vector<DCt>& f1);
