// Causal prefill attention on tcgen05 (sm_100a): the attention of the prefill phase of module-based
// batching (reference: prefill is a phase of the same schedule with tokens_per_seq_in_flight = P and
// no KV copy-in, pkg/src/moe_planner/memory_model.py:53-60, offload_dag.py:359-372; prefill batch B
// is searched, plan_search.py:202-209; paper prefill numbers PAPER.md:547-569).
//
// Semantics: HF transformers 5.5.0 causal attention (sdpa: fp32 scores / softmax / accumulation,
// one bf16 rounding of the output): o_i = sum_{j <= i} softmax_j(q_i . k_j * scale) v_j, for every
// position i of every equal-length prompt.  GQA (Mixtral): query head h reads kv head h / G.  MLA
// (DeepSeek-V2 prefill, modeling_deepseek_v2.py:337-396): per-head K = [k_nope_h | k_pe] with k_pe
// shared by all heads, V = v_h, so K comes from two tensors (the up-projected kv rows and the
// rotated k_pe rows) without being materialised.
//
// One work item = (prompt, query head, 128-query tile); persistent grid, one CTA per SM:
//   warp 4  Q / K producer (TMA, 128B swizzle): Q tile once per item, K tiles through a KS-stage ring
//   warp 5  V producer (TMA): V tiles through a VS-stage ring
//   warp 6  MMA issuer: S_j = Q K_j^T (M 128 queries, N 128 keys, K = head dim) into one of two TMEM
//           S buffers, issued one tile ahead of O += P_j V_j (M 128, N = HD_V, K = 128 keys; V is the
//           MN-major B operand straight from the TMA tile), O accumulating in TMEM
//   warps 0-3 softmax (thread = query row = TMEM lane): pass 1 row max over S_j (causal mask on the
//           diagonal tile); once the previous P.V has landed, rescale O in TMEM by exp2(m_old - m_new)
//           (skipped by a warp whose rows' maxima did not move); pass 2 P = exp2(S - m) as bf16 into
//           shared memory (UMMA A layout), row sum in fp32; after the last tile O / l -> bf16 -> global.
// TMEM: 2 x 128 S columns + HD_V O columns (512 allocated).
#include <cstdlib>

#include "common.cuh"

namespace mgb {

constexpr int kPfTile = 128;                 // queries per item = keys per tile = UMMA M / N
constexpr int kPfBlock = kPfTile * 128;      // one [128 rows][64 bf16] 128B-swizzled block (16 KB)
constexpr int kPfThreads = 7 * 32;

template <int HD_QK, int HD_V, int KS, int VS>
struct PfCfg {
  static constexpr int NQB = HD_QK / 64;     // 64-dim blocks of Q / K
  static constexpr int NVB = HD_V / 64;      // of V
  static constexpr int kQBytes = NQB * kPfBlock;
  static constexpr int kKBytes = NQB * kPfBlock;
  static constexpr int kVBytes = NVB * kPfBlock;
  static constexpr int kPBytes = 2 * kPfBlock;  // P [128 q][128 keys] bf16 as two 64-key blocks
  static constexpr int kOffK = kQBytes;
  static constexpr int kOffV = kOffK + KS * kKBytes;
  static constexpr int kOffP = kOffV + VS * kVBytes;
  static constexpr int kOffBar = kOffP + kPBytes;
  static constexpr int kBars = 2 + 2 * KS + 2 * VS + 2 + 2 + 1 + 1;
  static constexpr size_t kSmem = kOffBar + kBars * 8 + 16 + 1024;  // + 1024: base alignment
  static_assert(HD_QK % 64 == 0 && HD_V % 64 == 0 && HD_V <= 256, "prefill attention head dims");
  static_assert(kSmem <= 227 * 1024, "prefill attention smem");
};

struct PfArgs {
  int n_seq, P, Hq, G, n_qt;
  int q_head_cols, k_head_cols, v_head_cols, v_col0;  // column of head h: h * q_head_cols, (h / G) * k_head_cols, ...
  int kr_col0;                                        // rope part of K (MLA): column of the shared k_pe rows
  int nkb_main;                                       // K blocks from tmK (the rest from tmKr)
  float scale_log2;
  __nv_bfloat16* out;
  int out_cols;                                       // out row stride (elements); head h at h * HD_V
};

MGB_DEVINL void pf_item(int it, const PfArgs& a, int& s, int& h, int& qt) {
  // heaviest items (most key tiles) first; neighbouring items share (prompt, q-tile) and walk the
  // heads, so the G query heads of one kv head read its K / V tiles while they are in L2
  const int per = a.n_seq * a.Hq;
  qt = a.n_qt - 1 - it / per;
  const int r = it - (a.n_qt - 1 - qt) * per;
  s = r / a.Hq;
  h = r - s * a.Hq;
}

template <int HD_QK, int HD_V, int KS, int VS>
__global__ void __launch_bounds__(kPfThreads, 1)
prefill_attn_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                    const __grid_constant__ CUtensorMap tmKr, const __grid_constant__ CUtensorMap tmV, PfArgs a) {
  mgb::pdl_enter();
  using C = PfCfg<HD_QK, HD_V, KS, VS>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
  uint64_t* q_full = bars;
  uint64_t* q_empty = bars + 1;
  uint64_t* k_full = bars + 2;
  uint64_t* k_empty = k_full + KS;
  uint64_t* v_full = k_empty + KS;
  uint64_t* v_empty = v_full + VS;
  uint64_t* s_full = v_empty + VS;
  uint64_t* s_empty = s_full + 2;
  uint64_t* p_full = s_empty + 2;
  uint64_t* o_full = p_full + 1;  // one P.V completed (P buffer free, O up to date)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_full + 1);

  const uint32_t warp = warp_id(), lane = threadIdx.x & 31;
  const int items = a.n_qt * a.n_seq * a.Hq;
  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int i = 0; i < KS; ++i) { mbar_init(&k_full[i], 1); mbar_init(&k_empty[i], 1); }
    for (int i = 0; i < VS; ++i) { mbar_init(&v_full[i], 1); mbar_init(&v_empty[i], 1); }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_empty[i], 128);
    }
    mbar_init(p_full, 128);
    mbar_init(o_full, 1);
    fence_mbar_init();
  }
  if (warp == 6) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 4) {
    // ---------------- Q / K producer ----------------
    if (elect_one()) {
      const uint64_t pol = policy_evict_normal();
      int g = 0, n_it = 0;
      for (int it = blockIdx.x; it < items; it += gridDim.x, ++n_it) {
        int s, h, qt;
        pf_item(it, a, s, h, qt);
        const int row0 = s * a.P;
        mbar_wait(q_empty, (n_it & 1) ^ 1);
        mbar_arrive_expect_tx(q_full, C::kQBytes);
        for (int b = 0; b < C::NQB; ++b)
          tma_load_2d(smem + b * kPfBlock, &tmQ, q_full, h * a.q_head_cols + b * 64, row0 + qt * kPfTile, pol);
        const int kcol = (h / a.G) * a.k_head_cols;
        for (int j = 0; j <= qt; ++j, ++g) {
          const int st = g % KS;
          mbar_wait(&k_empty[st], ((g / KS) & 1) ^ 1);
          mbar_arrive_expect_tx(&k_full[st], C::kKBytes);
          uint8_t* dst = smem + C::kOffK + st * C::kKBytes;
          for (int b = 0; b < C::NQB; ++b) {
            if (b < a.nkb_main)
              tma_load_2d(dst + b * kPfBlock, &tmK, &k_full[st], kcol + b * 64, row0 + j * kPfTile, pol);
            else
              tma_load_2d(dst + b * kPfBlock, &tmKr, &k_full[st], a.kr_col0 + (b - a.nkb_main) * 64, row0 + j * kPfTile, pol);
          }
        }
      }
    }
  } else if (warp == 5) {
    // ---------------- V producer ----------------
    if (elect_one()) {
      const uint64_t pol = policy_evict_normal();
      int g = 0;
      for (int it = blockIdx.x; it < items; it += gridDim.x) {
        int s, h, qt;
        pf_item(it, a, s, h, qt);
        const int vcol = a.v_col0 + (h / a.G) * a.v_head_cols;
        for (int j = 0; j <= qt; ++j, ++g) {
          const int st = g % VS;
          mbar_wait(&v_empty[st], ((g / VS) & 1) ^ 1);
          mbar_arrive_expect_tx(&v_full[st], C::kVBytes);
          uint8_t* dst = smem + C::kOffV + st * C::kVBytes;
          for (int b = 0; b < C::NVB; ++b)
            tma_load_2d(dst + b * kPfBlock, &tmV, &v_full[st], vcol + b * 64, s * a.P + j * kPfTile, pol);
        }
      }
    }
  } else if (warp == 6) {
    // ---------------- MMA issuer ----------------
    if (elect_one()) {
      const uint32_t idesc_s = make_idesc_bf16(kPfTile, kPfTile);
      const uint32_t idesc_o = make_idesc_bf16(kPfTile, HD_V) | kIdescBMajorMN;
      const uint32_t q_addr = smem_u32(smem), p_addr = smem_u32(smem + C::kOffP);
      int g = 0, n_it = 0;
      auto issue_pv = [&](int gp, bool acc) {  // O (+)= P_gp V_gp
        const int vst = gp % VS;
        mbar_wait(p_full, gp & 1);
        mbar_wait(&v_full[vst], (gp / VS) & 1);
        tc_fence_after();
        const uint32_t v_addr = smem_u32(smem + C::kOffV + vst * C::kVBytes);
#pragma unroll
        for (int ks = 0; ks < kPfTile / 16; ++ks)
          umma_bf16(tmem + 256, make_sdesc_sw128(p_addr + (ks >> 2) * kPfBlock) + 2 * (ks & 3),
                    make_sdesc_sw128_mn(v_addr + ks * 2048, kPfBlock, 1024), idesc_o, (acc || ks > 0) ? 1u : 0u);
        umma_commit(o_full);
        umma_commit(&v_empty[vst]);
      };
      for (int it = blockIdx.x; it < items; it += gridDim.x, ++n_it) {
        int s, h, qt;
        pf_item(it, a, s, h, qt);
        mbar_wait(q_full, n_it & 1);
        for (int j = 0; j <= qt; ++j, ++g) {
          const int sb = g & 1, kst = g % KS;
          mbar_wait(&k_full[kst], (g / KS) & 1);
          mbar_wait(&s_empty[sb], ((g >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t k_addr = smem_u32(smem + C::kOffK + kst * C::kKBytes);
#pragma unroll
          for (int ks = 0; ks < HD_QK / 16; ++ks)
            umma_bf16(tmem + sb * 128, make_sdesc_sw128(q_addr + (ks >> 2) * kPfBlock) + 2 * (ks & 3),
                      make_sdesc_sw128(k_addr + (ks >> 2) * kPfBlock) + 2 * (ks & 3), idesc_s, ks > 0);
          umma_commit(&s_full[sb]);
          umma_commit(&k_empty[kst]);
          if (j == qt) umma_commit(q_empty);
          if (j > 0) issue_pv(g - 1, j > 1);  // the previous tile's P.V, behind this tile's S
        }
        issue_pv(g - 1, qt > 0);
      }
    }
  } else {
    // ---------------- softmax (warps 0-3; thread = query row = TMEM lane) ----------------
    const int row = warp * 32 + lane;
    const uint32_t lane_off = (warp * 32) << 16;
    const uint32_t tO = tmem + lane_off + 256;
    uint8_t* P = smem + C::kOffP;
    int g = 0;
    for (int it = blockIdx.x; it < items; it += gridDim.x) {
      int s, h, qt;
      pf_item(it, a, s, h, qt);
      const int qi = qt * kPfTile + row;  // query position in the prompt
      float m_run = -INFINITY, l_run = 0.f;
      for (int j = 0; j <= qt; ++j, ++g) {
        const int sb = g & 1;
        const bool diag = j == qt;
        const uint32_t tS = tmem + lane_off + sb * 128;
        mbar_wait(&s_full[sb], (g >> 1) & 1);
        tc_fence_after();
        // pass 1: row max
        float mt = -INFINITY;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t v[32];
          tmem_ld32(tS + c * 32, v);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const int kj = j * kPfTile + c * 32 + i;
            if (!diag || kj <= qi) mt = fmaxf(mt, __uint_as_float(v[i]) * a.scale_log2);
          }
        }
        const float m_new = fmaxf(m_run, mt);
        const float m_use = m_new == -INFINITY ? 0.f : m_new;
        const float alpha = m_run == -INFINITY ? 0.f : exp2f(m_run - m_use);
        if (j > 0) {
          // the previous P.V has landed in O (and released the P buffer): rescale O to the new max
          mbar_wait(o_full, (g - 1) & 1);
          tc_fence_after();
          if (__any_sync(0xffffffffu, alpha != 1.f)) {
#pragma unroll 1
            for (int c = 0; c < HD_V / 32; ++c) {
              uint32_t v[32];
              tmem_ld32(tO + c * 32, v);
              tmem_ld_wait();
#pragma unroll
              for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * alpha);
              tmem_st32(tO + c * 32, v);
            }
            tmem_st_wait();
          }
        }
        // pass 2: P = exp2(S - m) as bf16 into the UMMA A tile
        float sum = 0.f;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t v[32];
          tmem_ld32(tS + c * 32, v);
          tmem_ld_wait();
#pragma unroll
          for (int x = 0; x < 4; ++x) {  // 16-byte chunk cc = 4c + x of the row (8 keys)
            uint32_t pk[4];
#pragma unroll
            for (int i = 0; i < 8; i += 2) {
              const int kk = 8 * x + i, kj = j * kPfTile + c * 32 + kk;
              const float p0 = (!diag || kj <= qi) ? exp2f(__uint_as_float(v[kk]) * a.scale_log2 - m_use) : 0.f;
              const float p1 = (!diag || kj + 1 <= qi) ? exp2f(__uint_as_float(v[kk + 1]) * a.scale_log2 - m_use) : 0.f;
              sum += p0 + p1;
              pk[i >> 1] = pack_bf16x2(p0, p1);
            }
            const int cc = 4 * c + x, blk = cc >> 3, w = (cc & 7) ^ (row & 7);
            *reinterpret_cast<uint4*>(P + blk * kPfBlock + (row >> 3) * 1024 + (row & 7) * 128 + w * 16) =
                make_uint4(pk[0], pk[1], pk[2], pk[3]);
          }
        }
        l_run = l_run * alpha + sum;
        m_run = m_new;
        tc_fence_before();
        mbar_arrive(&s_empty[sb]);
        fence_proxy_async_smem();
        mbar_arrive(p_full);
      }
      // the last P.V, then the output row O / l
      mbar_wait(o_full, (g - 1) & 1);
      tc_fence_after();
      const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
      uint4* dst = reinterpret_cast<uint4*>(a.out + (size_t)(s * a.P + qi) * a.out_cols + (size_t)h * HD_V);
#pragma unroll 1
      for (int c = 0; c < HD_V / 32; ++c) {
        uint32_t v[32];
        tmem_ld32(tO + c * 32, v);
        tmem_ld_wait();
        if (qi < a.P) {
#pragma unroll
          for (int x = 0; x < 4; ++x) {
            const float* f = reinterpret_cast<const float*>(v + 8 * x);
            dst[4 * c + x] = make_uint4(pack_bf16x2(f[0] * inv, f[1] * inv), pack_bf16x2(f[2] * inv, f[3] * inv),
                                        pack_bf16x2(f[4] * inv, f[5] * inv), pack_bf16x2(f[6] * inv, f[7] * inv));
          }
        }
      }
      tc_fence_before();  // O is read before the next item's first P.V overwrites it
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 6) tmem_dealloc<512>(tmem);
}

template <int HD_QK, int HD_V, int KS, int VS>
int launch_prefill(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tkr, const CUtensorMap& tv,
                   const PfArgs& a, cudaStream_t st) {
  using C = PfCfg<HD_QK, HD_V, KS, VS>;
  if (const int rc = mgb_host::ensure_max_smem((const void*)prefill_attn_kernel<HD_QK, HD_V, KS, VS>, (int)C::kSmem))
    return rc;
  const int items = a.n_qt * a.n_seq * a.Hq;
  int grid = mgb_host::num_sms();
  if (grid > items) grid = items;
  mgb_host::launch(prefill_attn_kernel<HD_QK, HD_V, KS, VS>, dim3(grid), dim3(kPfThreads), C::kSmem, st, nullptr,
      tq, tk, tkr, tv, a);
  return mgb_host::launch_status();
}

}  // namespace mgb

extern "C" {

// Head dims the kernel is instantiated for (others: MGB_EINVAL).
int mgb_prefill_attn_supported(int hd_qk, int hd_v) {
  return (hd_qk == 128 && hd_v == 128) || (hd_qk == 192 && hd_v == 128) || (hd_qk == 64 && hd_v == 64);
}

// Causal attention of n_seq equal-length prompts of P tokens (rows s*P .. s*P+P-1 of every tensor).
//   q   [n_seq*P, q_cols]  query head h at columns [h*q_head_cols, +hd_qk)
//   k   [n_seq*P, k_cols]  kv head g = h / (Hq/Hkv) at columns [g*k_head_cols, +kd) where kd = hd_qk, or
//                          (MLA) kd = hd_qk - kr_dim and the last kr_dim dims come from
//   kr  [n_seq*P, kr_cols] columns [0, kr_dim) (shared by all heads; NULL when kr_dim = 0)
//   v   [n_seq*P, v_cols]  kv head g at columns [v_col0 + g*v_head_cols, +hd_v)
//   out [n_seq*P, out_cols] head h at columns [h*hd_v, +hd_v)
int mgb_prefill_attn(const void* q, int q_cols, int q_head_cols, const void* k, int k_cols, int k_head_cols,
                     const void* kr, int kr_cols, int kr_dim, const void* v, int v_cols, int v_head_cols, int v_col0,
                     int n_seq, int P, int Hq, int Hkv, int hd_qk, int hd_v, float scale, void* out, int out_cols,
                     void* stream) {
  if (n_seq < 1 || P < 1 || Hq < 1 || Hkv < 1 || Hq % Hkv || !mgb_prefill_attn_supported(hd_qk, hd_v)) return MGB_EINVAL;
  if (kr_dim % 64 || kr_dim >= hd_qk || (kr_dim && !kr) || q_cols % 8 || k_cols % 8 || v_cols % 8 || out_cols % 8 ||
      (kr && kr_cols % 8))
    return MGB_EINVAL;
  const uint64_t T = (uint64_t)n_seq * P;
  CUtensorMap tq, tk, tkr, tv;
  if (mgb_host::encode_tmap_2d_bf16(&tq, q, q_cols, T, (uint64_t)q_cols * 2, 64, mgb::kPfTile) != CUDA_SUCCESS ||
      mgb_host::encode_tmap_2d_bf16(&tk, k, k_cols, T, (uint64_t)k_cols * 2, 64, mgb::kPfTile) != CUDA_SUCCESS ||
      mgb_host::encode_tmap_2d_bf16(&tv, v, v_cols, T, (uint64_t)v_cols * 2, 64, mgb::kPfTile) != CUDA_SUCCESS)
    return MGB_ECUDA;
  if (kr_dim) {
    if (mgb_host::encode_tmap_2d_bf16(&tkr, kr, kr_cols, T, (uint64_t)kr_cols * 2, 64, mgb::kPfTile) != CUDA_SUCCESS)
      return MGB_ECUDA;
  } else {
    tkr = tk;
  }
  mgb::PfArgs a{n_seq, P, Hq, Hq / Hkv, (P + mgb::kPfTile - 1) / mgb::kPfTile, q_head_cols, k_head_cols, v_head_cols,
                v_col0, 0, (hd_qk - kr_dim) / 64, scale * 1.4426950408889634f, reinterpret_cast<__nv_bfloat16*>(out),
                out_cols};
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (hd_qk == 128) return mgb::launch_prefill<128, 128, 2, 2>(tq, tk, tkr, tv, a, st);
  if (hd_qk == 192) return mgb::launch_prefill<192, 128, 2, 1>(tq, tk, tkr, tv, a, st);
  return mgb::launch_prefill<64, 64, 2, 2>(tq, tk, tkr, tv, a, st);
}

}  // extern "C"
