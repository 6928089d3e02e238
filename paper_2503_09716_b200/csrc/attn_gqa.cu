// Paged GQA decode attention (Mixtral) on sm_100a — the ATTN_MECH_GPU job of the module-based
// batching schedule (reference: pkg/src/moe_planner/offload_dag.py:393-402; cost model
// hw_profile.py:269-270,285-287).  Semantics: softmax(q k^T / sqrt(hd)) v with key/value head
// i // G for query head i (HF transformers 5.5.0 attention with repeat_kv,
// modeling_mixtral.py:257-291), computed with fp32 scores / softmax / accumulation and one bf16
// rounding of the output (HF's default sdpa path), so it matches the oracle within tolerance.
//
// KV layout (owned by this framework, chosen for the decode access pattern): pages of
// kPage = 64 tokens; per (page, kv-head) one contiguous block for K and one for V, both
// "chunk-major": [hd/8 chunks][64 tokens][8 dims].  Eight consecutive tokens of one 8-dim chunk
// are 128 contiguous bytes, so every ldmatrix (K) / ldmatrix.trans (V) is bank-conflict free.
//
// Persistent kernel, 2 CTAs per SM: warp 4 is a bulk-copy producer streaming the pages of the
// CTA's (sequence, kv-head) work items through a 3-stage shared-memory ring (cp.async.bulk +
// mbarrier), running ahead across work-item boundaries; warps 0-3 consume, each owning 16 tokens
// of every page: S = Q K^T and O += P V on the tensor cores (mma.sync m16n8k16, the G query heads
// of the group are rows 0..G-1 of the 16-row tile), online softmax per warp, then a 4-way merge
// per work item.  HBM-bound by construction: ~1 MMA per 128 B of KV.
#include "common.cuh"

namespace mgb {

constexpr int kPage = 64;
constexpr int kAttnStages = 3;
constexpr int kConsumerWarps = 4;
constexpr int kAttnThreads = (kConsumerWarps + 1) * 32;

template <int HD, int G>
struct GqaSmem {
  static constexpr int kTileElems = HD * kPage;
  static constexpr int kTileBytes = kTileElems * 2;                 // one K (or V) page-head block
  static constexpr int kStageBytes = 2 * kTileBytes;
  static constexpr int kMergeStride = G * HD + 16;                  // per warp: O (G rows) + m[8] + l[8]
  static constexpr int kMergeBytes = kConsumerWarps * kMergeStride * 4;
  static constexpr size_t kBytes = (size_t)kAttnStages * kStageBytes + kMergeBytes + 128;
};

MGB_DEVINL void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
MGB_DEVINL void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
// D(16x8 f32) += A(16x16 bf16, row) * B(16x8 bf16, col)
MGB_DEVINL void mma_bf16_16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                               uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
// 8x8 b16 register transpose across the warp (thread (g, t) gets rows 2t, 2t+1 of column g)
MGB_DEVINL uint32_t movmatrix_trans(uint32_t a) {
  uint32_t d;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(d) : "r"(a));
  return d;
}
MGB_DEVINL void named_bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

template <int HD, int G>
__global__ void __launch_bounds__(kAttnThreads, 2)
decode_attn_gqa_kernel(const __nv_bfloat16* __restrict__ q,       // [B, Hkv*G, HD]
                       const __nv_bfloat16* __restrict__ k_cache,  // pages, chunk-major
                       const __nv_bfloat16* __restrict__ v_cache,
                       const int* __restrict__ block_table, int max_pages,
                       const int* __restrict__ seq_lens, int B, int Hkv, float scale_log2,
                       __nv_bfloat16* __restrict__ out) {          // [B, Hkv*G*HD]
  static_assert(G <= 8 && HD % 16 == 0, "GQA tile: G <= 8 query heads per kv head");
  using S = GqaSmem<HD, G>;
  constexpr int KSTEPS = HD / 16;   // k-steps of QK^T
  constexpr int NT = HD / 8;        // n-tiles of PV (8 dims each)
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* ring = smem;
  float* merge = reinterpret_cast<float*>(smem + kAttnStages * S::kStageBytes);  // [warp][8][HD] + m,l
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kAttnStages * S::kStageBytes + S::kMergeBytes);
  uint64_t* empty = full + kAttnStages;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_items = B * Hkv;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kAttnStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == kConsumerWarps) {
    // ------------------------------ producer ------------------------------
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      int stage = 0;
      uint32_t phase = 0;
      for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
        const int b = it / Hkv, h = it - b * Hkv;
        const int np = (seq_lens[b] + kPage - 1) / kPage;
        const int* bt = block_table + (size_t)b * max_pages;
        for (int p = 0; p < np; ++p) {
          mbar_wait(&empty[stage], phase ^ 1);
          const size_t blk = ((size_t)bt[p] * Hkv + h) * S::kTileElems;
          uint8_t* dst = ring + stage * S::kStageBytes;
          mbar_arrive_expect_tx(&full[stage], S::kStageBytes);
          bulk_load(dst, k_cache + blk, S::kTileBytes, &full[stage], pol);
          bulk_load(dst + S::kTileBytes, v_cache + blk, S::kTileBytes, &full[stage], pol);
          if (++stage == kAttnStages) { stage = 0; phase ^= 1; }
        }
      }
    }
    return;
  }

  // ------------------------------ consumers (warps 0..3) ------------------------------
  // "Swap-AB" tiles: the 16 tokens of the warp's page slice are the MMA M dimension and the G query
  // heads the N dimension (8, heads >= G zero), so S^T = K Q^T and O^T += V^T P^T each take half the
  // mma.sync of the head-rows-as-M form (G <= 8 of 16 rows used there), and the softmax runs on half
  // as many dead lanes.  P^T goes from the S^T accumulator layout to the B-operand layout with two
  // register transposes (movmatrix).  The running max of a head is only raised when a page exceeds it
  // by 2^8 (P <= 256 stays exact enough in bf16 / fp32), so O is rescaled on a few pages per item.
  const int g = lane >> 2, t = lane & 3;   // mma fragment coordinates
  const bool head_ok = g < G;              // B-operand column (query head) g exists
  const bool h0_ok = 2 * t < G, h1_ok = 2 * t + 1 < G;  // this thread's accumulator heads 2t, 2t+1
  constexpr int DT = HD / 16;              // 16-dim tiles of O^T
  int stage = 0;
  uint32_t phase = 0;
  for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
    const int b = it / Hkv, h = it - b * Hkv;
    const int len = seq_lens[b];
    const int np = (len + kPage - 1) / kPage;
    // Q^T B-fragments: column n = head g, k = 2t.. of each 16-dim step (heads >= G are zero)
    uint32_t qb[KSTEPS][2];
    const __nv_bfloat16* qrow = q + ((size_t)b * Hkv * G + (size_t)h * G + (head_ok ? g : 0)) * HD;
#pragma unroll
    for (int ks = 0; ks < KSTEPS; ++ks) {
      qb[ks][0] = head_ok ? *reinterpret_cast<const uint32_t*>(qrow + ks * 16 + 2 * t) : 0u;
      qb[ks][1] = head_ok ? *reinterpret_cast<const uint32_t*>(qrow + ks * 16 + 8 + 2 * t) : 0u;
    }
    float o[DT][4];
#pragma unroll
    for (int n = 0; n < DT; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
    float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;  // heads 2t, 2t+1

    for (int p = 0; p < np; ++p) {
      mbar_wait(&full[stage], phase);
      const uint32_t kbase = smem_u32(ring + stage * S::kStageBytes);
      const uint32_t vbase = kbase + S::kTileBytes;
      const int tok0 = warp * 16;  // this warp's 16 tokens of the page
      const int mi = lane >> 3, r = lane & 7;
      // ---- S^T = K Q^T: 16 tokens x 8 heads; two accumulators (even / odd k-steps) break the chain ----
      float sa[4] = {0.f, 0.f, 0.f, 0.f}, sb[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int ks = 0; ks < KSTEPS; ++ks) {
        // A matrices: (tok 0-7, chunk 2ks), (tok 8-15, chunk 2ks), (tok 0-7, chunk 2ks+1), (tok 8-15, chunk 2ks+1)
        const int chunk = 2 * ks + (mi >> 1);
        const int tok = tok0 + ((mi & 1) << 3) + r;
        uint32_t a0, a1, a2, a3;
        ldsm_x4(kbase + (uint32_t)((chunk * kPage + tok) * 16), a0, a1, a2, a3);
        if (ks & 1) mma_bf16_16816(sb, a0, a1, a2, a3, qb[ks][0], qb[ks][1]);
        else mma_bf16_16816(sa, a0, a1, a2, a3, qb[ks][0], qb[ks][1]);
      }
      // ---- online softmax: c0/c1 = token g (heads 2t, 2t+1), c2/c3 = token g + 8 ----
      const int n_valid = len - p * kPage - tok0;  // tokens of this warp that exist
      const bool v_lo = g < n_valid, v_hi = g + 8 < n_valid;
      const float x0 = (v_lo && h0_ok) ? (sa[0] + sb[0]) * scale_log2 : -INFINITY;
      const float x1 = (v_lo && h1_ok) ? (sa[1] + sb[1]) * scale_log2 : -INFINITY;
      const float x2 = (v_hi && h0_ok) ? (sa[2] + sb[2]) * scale_log2 : -INFINITY;
      const float x3 = (v_hi && h1_ok) ? (sa[3] + sb[3]) * scale_log2 : -INFINITY;
      float mx0 = fmaxf(x0, x2), mx1 = fmaxf(x1, x3);  // over this warp's 16 tokens (lanes with equal t)
#pragma unroll
      for (int o_ = 4; o_ < 32; o_ <<= 1) {
        mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, o_));
        mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, o_));
      }
      float al0 = 1.f, al1 = 1.f;
      if (mx0 > m0 + 8.f) { al0 = exp2f(m0 - mx0); m0 = mx0; }
      if (mx1 > m1 + 8.f) { al1 = exp2f(m1 - mx1); m1 = mx1; }
      if (__any_sync(0xffffffffu, al0 != 1.f || al1 != 1.f)) {
        l0 *= al0;
        l1 *= al1;
#pragma unroll
        for (int n = 0; n < DT; ++n) {
          o[n][0] *= al0;
          o[n][1] *= al1;
          o[n][2] *= al0;
          o[n][3] *= al1;
        }
      }
      const float mu0 = m0 == -INFINITY ? 0.f : m0, mu1 = m1 == -INFINITY ? 0.f : m1;
      const float p0 = exp2f(x0 - mu0), p1 = exp2f(x1 - mu1), p2 = exp2f(x2 - mu0), p3 = exp2f(x3 - mu1);
      l0 += p0 + p2;
      l1 += p1 + p3;
      // V rows past the sequence end (last, partial page) may hold any bits -- an offloaded host
      // page store or a reused staging page -- and P = 0 there would still give 0 * NaN = NaN in
      // the MMA: zero this warp's invalid V rows in the stage before P.V reads them
      if (n_valid < 16) {
        const int first = n_valid < 0 ? 0 : n_valid;
        uint8_t* vb = ring + stage * S::kStageBytes + S::kTileBytes;
        for (int i = lane; i < (16 - first) * (HD / 8); i += 32) {
          const int tk = tok0 + first + i / (HD / 8), c = i % (HD / 8);
          *reinterpret_cast<uint4*>(vb + (c * kPage + tk) * 16) = make_uint4(0u, 0u, 0u, 0u);
        }
        // generic-proxy writes, then the producer's next bulk copy (async proxy) into this stage
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
      }
      // P^T as the B operand (k = 16 tokens, n = 8 heads): transpose the two 8x8 accumulator blocks
      const uint32_t pb0 = movmatrix_trans(pack_bf16x2(p0, p1));
      const uint32_t pb1 = movmatrix_trans(pack_bf16x2(p2, p3));
      // ---- O^T += V^T P^T : one 16-dim tile per ldmatrix.x4.trans ----
#pragma unroll
      for (int d2 = 0; d2 < DT; ++d2) {
        // A matrices (V^T, rows = dims): (chunk 2d2, tok 0-7), (chunk 2d2+1, tok 0-7), (chunk 2d2, tok 8-15), (chunk 2d2+1, tok 8-15)
        const int chunk = 2 * d2 + (mi & 1);
        const int tok = tok0 + ((mi >> 1) << 3) + r;
        uint32_t a0, a1, a2, a3;
        ldsm_x4_t(vbase + (uint32_t)((chunk * kPage + tok) * 16), a0, a1, a2, a3);
        mma_bf16_16816(o[d2], a0, a1, a2, a3, pb0, pb1);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (++stage == kAttnStages) { stage = 0; phase ^= 1; }
    }

    // ---- merge the 4 warps' partial (m, l, O) and store ----
#pragma unroll
    for (int o_ = 4; o_ < 32; o_ <<= 1) {
      l0 += __shfl_xor_sync(0xffffffffu, l0, o_);
      l1 += __shfl_xor_sync(0xffffffffu, l1, o_);
    }
    constexpr int MS = S::kMergeStride;
    float* mo = merge + warp * MS;
#pragma unroll
    for (int n = 0; n < DT; ++n) {
      if (h0_ok) {
        mo[(2 * t) * HD + 16 * n + g] = o[n][0];
        mo[(2 * t) * HD + 16 * n + g + 8] = o[n][2];
      }
      if (h1_ok) {
        mo[(2 * t + 1) * HD + 16 * n + g] = o[n][1];
        mo[(2 * t + 1) * HD + 16 * n + g + 8] = o[n][3];
      }
    }
    if (g == 0) {
      if (h0_ok) {
        mo[G * HD + 2 * t] = m0;
        mo[G * HD + 8 + 2 * t] = l0;
      }
      if (h1_ok) {
        mo[G * HD + 2 * t + 1] = m1;
        mo[G * HD + 8 + 2 * t + 1] = l1;
      }
    }
    named_bar_sync(1, kConsumerWarps * 32);
    for (int i = threadIdx.x; i < G * HD; i += kConsumerWarps * 32) {
      const int row = i / HD, col = i - row * HD;
      float M = -INFINITY;
#pragma unroll
      for (int w = 0; w < kConsumerWarps; ++w) M = fmaxf(M, merge[w * MS + G * HD + row]);
      float num = 0.f, den = 0.f;
#pragma unroll
      for (int w = 0; w < kConsumerWarps; ++w) {
        const float* mw = merge + w * MS;
        const float mw_row = mw[G * HD + row];
        const float sc = (mw_row == -INFINITY) ? 0.f : exp2f(mw_row - M);
        num += sc * mw[row * HD + col];
        den += sc * mw[G * HD + 8 + row];
      }
      out[((size_t)b * Hkv * G + (size_t)h * G + row) * HD + col] = __float2bfloat16_rn(den > 0.f ? num / den : 0.f);
    }
    named_bar_sync(1, kConsumerWarps * 32);  // merge buffer reused by the next item
  }
}

template <int HD, int G>
int launch_gqa(const void* q, const void* kc, const void* vc, const int* bt, int max_pages, const int* lens, int B,
               int Hkv, float scale, void* out, cudaStream_t st) {
  using S = GqaSmem<HD, G>;
  if (const int rc = mgb_host::ensure_max_smem((const void*)decode_attn_gqa_kernel<HD, G>, (int)S::kBytes)) return rc;
  const int items = B * Hkv;
  int grid = 2 * mgb_host::num_sms();
  if (grid > items) grid = items;
  decode_attn_gqa_kernel<HD, G><<<grid, kAttnThreads, S::kBytes, st>>>(
      reinterpret_cast<const __nv_bfloat16*>(q), reinterpret_cast<const __nv_bfloat16*>(kc),
      reinterpret_cast<const __nv_bfloat16*>(vc), bt, max_pages, lens, B, Hkv, scale * 1.4426950408889634f,
      reinterpret_cast<__nv_bfloat16*>(out));
  return mgb_host::launch_status();
}

}  // namespace mgb

extern "C" {

int mgb_kv_page_size(void) { return mgb::kPage; }

// Decode attention for B sequences, one new query token each (already RoPE'd and appended to
// the cache by mgb_rope_append_gqa).  seq_lens[b] counts the cached tokens including the new one.
int mgb_decode_attn_gqa(const void* q, const void* k_cache, const void* v_cache, const int* block_table,
                        int max_pages, const int* seq_lens, int B, int Hq, int Hkv, int head_dim, float scale,
                        void* out, void* stream) {
  if (B < 1 || Hkv < 1 || Hq % Hkv) return MGB_EINVAL;
  const int G = Hq / Hkv;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
#define MGB_GQA_CASE(HD_, G_) \
  if (head_dim == HD_ && G == G_) return mgb::launch_gqa<HD_, G_>(q, k_cache, v_cache, block_table, max_pages, seq_lens, B, Hkv, scale, out, st);
  MGB_GQA_CASE(128, 4)
  MGB_GQA_CASE(128, 6)
  MGB_GQA_CASE(128, 8)
  MGB_GQA_CASE(64, 4)
  MGB_GQA_CASE(32, 4)
#undef MGB_GQA_CASE
  return MGB_EINVAL;
}

}  // extern "C"
