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

// Optional per-page timeline of CTA 0 (build with -DMGB_GQA_TRACE; tools/gqa_trace.py):
// g_gqa_trace[ev * 512 + i] = %globaltimer of event ev at the CTA's i-th page (or item)
#ifdef MGB_GQA_TRACE
__device__ unsigned long long g_gqa_trace[8 * 512];
MGB_DEVINL void gqa_trace(int ev, int i) {
  if (blockIdx.x == 0 && i < 512) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_gqa_trace[ev * 512 + i] = t;
  }
}
#else
MGB_DEVINL void gqa_trace(int, int) {}
#endif

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
MGB_DEVINL void named_bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// Fused RoPE + KV append (mgb_decode_attn_gqa_rope): the kernel takes the raw fused qkv rows
// [Hq | Hkv | Hkv] x HD instead of RoPE'd q, rotates the item's G query heads while loading them,
// and its producer warp rotates the item's new k row, copies its v row into the token's slot of
// the last K / V page (same arithmetic as rope_append_gqa_kernel, mgb::rope_rot8) and fences the
// stores into the async proxy before it issues that item's page loads.  Cache length = position + 1.
struct GqaRope {
  const __nv_bfloat16* qkv;  // [B, (Hq + 2 Hkv) * HD]; null: plain decode (q RoPE'd, KV appended)
  const int* positions;      // [B] position of the new token
  const float* cos_t;        // [max_pos, HD / 2]
  const float* sin_t;
  __nv_bfloat16* k_cache;    // the same pages as k_cache / v_cache, written at the new token's slot
  __nv_bfloat16* v_cache;
  int* seq_lens;             // [B] written = position + 1 (by the kv-head-0 item)
};

template <int HD, int G>
__global__ void __launch_bounds__(kAttnThreads, 2)
decode_attn_gqa_kernel(const __nv_bfloat16* __restrict__ q,       // [B, Hkv*G, HD]
                       const __nv_bfloat16* __restrict__ k_cache,  // pages, chunk-major
                       const __nv_bfloat16* __restrict__ v_cache,
                       const int* __restrict__ block_table, int max_pages,
                       const int* __restrict__ seq_lens, int B, int Hkv, float scale_log2,
                       __nv_bfloat16* __restrict__ out,            // [B, Hkv*G*HD]
                       int* __restrict__ sched,   // optional {next item, exit ticket}
                       const GqaRope rp) {
  mgb::pdl_enter();
  static_assert(G <= 8 && HD % 16 == 0, "GQA tile: G <= 8 query heads per kv head");
  using S = GqaSmem<HD, G>;
  constexpr int KSTEPS = HD / 16;   // k-steps of QK^T
  constexpr int NT = HD / 8;        // n-tiles of PV (8 dims each)
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* ring = smem;
  float* merge = reinterpret_cast<float*>(smem + kAttnStages * S::kStageBytes);  // [warp][8][HD] + m,l
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kAttnStages * S::kStageBytes + S::kMergeBytes);
  uint64_t* empty = full + kAttnStages;
  // Work items reach the consumers through a 4-slot ring: with `sched`, the producer takes the next
  // item from a global counter as it starts loading it (dynamic: every CTA keeps streaming until the
  // work runs out, instead of the static share of 22-23 items leaving the last wave part-idle); without
  // it, the static round-robin share.  Item -1 ends the CTA.
  __shared__ int s_item[4];
  __shared__ __align__(8) uint64_t item_full[4], item_empty[4], appended[4];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_items = B * Hkv;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kAttnStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
    }
    for (int s = 0; s < 4; ++s) {
      mbar_init(&item_full[s], 1);
      mbar_init(&item_empty[s], kConsumerWarps);
      mbar_init(&appended[s], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == kConsumerWarps) {
    // ------------------------------ producer ------------------------------
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      int stage = 0, gp = 0;
      uint32_t phase = 0;
      for (int k = 0;; ++k) {
        int it = sched ? atomicAdd(sched, 1) : (int)blockIdx.x + k * (int)gridDim.x;
        if (it >= n_items) it = -1;
        mbar_wait(&item_empty[k & 3], ((k >> 2) & 1) ^ 1);
        s_item[k & 3] = it;
        mbar_arrive(&item_full[k & 3]);
        if (it < 0) break;
        const int b = it / Hkv, h = it - b * Hkv;
        int len;
        if (rp.qkv) {
          const int pos = rp.positions[b];
          len = pos < 0 ? 0 : min(pos + 1, max_pages * kPage);
        } else {
          len = seq_lens[b];
        }
        const int np = (len + kPage - 1) / kPage;
        const int* bt = block_table + (size_t)b * max_pages;
        for (int p = 0; p < np; ++p) {
          // fused append: the last page holds the new token, which the consumers store at the item's
          // start -- by then this producer is normally still a few pages behind
          if (rp.qkv && p == np - 1) mbar_wait(&appended[k & 3], (k >> 2) & 1);
          mbar_wait(&empty[stage], phase ^ 1);
          gqa_trace(0, gp++);  // 0: stage free, page load issued
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
  const int g = lane >> 2, t = lane & 3;   // mma fragment coordinates
  const bool row_ok = g < G;
  int stage = 0, gc = 0, item = 0;
  uint32_t phase = 0;
  for (;; ++item) {
    mbar_wait(&item_full[item & 3], (item >> 2) & 1);
    const int it = s_item[item & 3];
    if (it < 0) break;
    const int b = it / Hkv, h = it - b * Hkv;
    int len;
    if (rp.qkv) {
      const int pos = rp.positions[b];
      len = pos < 0 ? 0 : min(pos + 1, max_pages * kPage);
    } else {
      len = seq_lens[b];
    }
    if (threadIdx.x == 0) gqa_trace(4, item);  // 4: item start (consumers)
    if (rp.qkv && warp == 0) {
      // the item's new token: k rotated, v copied into its slot of the last K / V page (lanes
      // 0..HD/16-1: one k rotation pair of 8-dim chunks each, the next HD/16 lanes: v), fenced into
      // the async proxy, then the producer may load that page
      const int pos = rp.positions[b];
      if (pos >= 0 && pos < max_pages * kPage) {
        constexpr int half = HD / 16;
        if (lane < 2 * half) {
          const int Hq = Hkv * G;
          const bool is_k = lane < half;
          const int j = is_k ? lane : lane - half;
          const uint4* src = reinterpret_cast<const uint4*>(rp.qkv + (size_t)b * (Hq + 2 * Hkv) * HD +
                                                            (size_t)(Hq + (is_k ? 0 : Hkv) + h) * HD);
          uint4 ol = src[j], oh = src[j + half];
          const int page = block_table[(size_t)b * max_pages + pos / kPage], slot = pos % kPage;
          if (is_k)
            rope_rot8(ol, oh, rp.cos_t + (size_t)pos * (HD / 2) + j * 8, rp.sin_t + (size_t)pos * (HD / 2) + j * 8,
                      ol, oh);
          __nv_bfloat16* blk = (is_k ? rp.k_cache : rp.v_cache) + ((size_t)page * Hkv + h) * HD * kPage;
          *reinterpret_cast<uint4*>(blk + ((size_t)j * kPage + slot) * 8) = ol;
          *reinterpret_cast<uint4*>(blk + ((size_t)(j + half) * kPage + slot) * 8) = oh;
          asm volatile("fence.proxy.async.global;" ::: "memory");  // generic stores -> the page's bulk copy
        }
        if (h == 0 && lane == 0) rp.seq_lens[b] = pos + 1;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&appended[item & 3]);
    }
    const int np = (len + kPage - 1) / kPage;
    // Q A-fragments (rows = the G query heads of this kv head; rows >= G are zero)
    uint32_t qa[KSTEPS][2];
    if (rp.qkv) {
      // raw q rows, rotated here: fragment dims d and d + HD/2 (k-steps ks and ks + KSTEPS/2) are one
      // rotation pair, so every lane holds both halves it needs
      const int Hq = Hkv * G;
      const int pos = min(max(rp.positions[b], 0), max_pages * kPage - 1);
      const __nv_bfloat16* qrow = rp.qkv + (size_t)b * (Hq + 2 * Hkv) * HD + ((size_t)h * G + (row_ok ? g : 0)) * HD;
      const float* cr = rp.cos_t + (size_t)pos * (HD / 2);
      const float* sr = rp.sin_t + (size_t)pos * (HD / 2);
#pragma unroll
      for (int ks = 0; ks < KSTEPS / 2; ++ks) {
#pragma unroll
        for (int hv = 0; hv < 2; ++hv) {
          const int dd = ks * 16 + 8 * hv + 2 * t;  // dims dd, dd + 1 (< HD/2) and their partners + HD/2
          if (row_ok) {
            const uint32_t lo = *reinterpret_cast<const uint32_t*>(qrow + dd);
            const uint32_t hi = *reinterpret_cast<const uint32_t*>(qrow + dd + HD / 2);
            const float2 c = *reinterpret_cast<const float2*>(cr + dd), sn = *reinterpret_cast<const float2*>(sr + dd);
            const float a0 = bf16lo(lo), a1 = bf16hi(lo), b0 = bf16lo(hi), b1 = bf16hi(hi);
            qa[ks][hv] = pack_bf16x2(bf16_round(a0 * c.x) + bf16_round(-b0 * sn.x),
                                     bf16_round(a1 * c.y) + bf16_round(-b1 * sn.y));
            qa[ks + KSTEPS / 2][hv] = pack_bf16x2(bf16_round(b0 * c.x) + bf16_round(a0 * sn.x),
                                                  bf16_round(b1 * c.y) + bf16_round(a1 * sn.y));
          } else {
            qa[ks][hv] = 0u;
            qa[ks + KSTEPS / 2][hv] = 0u;
          }
        }
      }
    } else {
      const __nv_bfloat16* qrow = q + ((size_t)b * Hkv * G + (size_t)h * G + (row_ok ? g : 0)) * HD;
#pragma unroll
      for (int ks = 0; ks < KSTEPS; ++ks) {
        qa[ks][0] = row_ok ? *reinterpret_cast<const uint32_t*>(qrow + ks * 16 + 2 * t) : 0u;
        qa[ks][1] = row_ok ? *reinterpret_cast<const uint32_t*>(qrow + ks * 16 + 8 + 2 * t) : 0u;
      }
    }
    float o[NT][4];
#pragma unroll
    for (int n = 0; n < NT; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
    float m_run = -INFINITY, l_run = 0.f;

    for (int p = 0; p < np; ++p, ++gc) {
      mbar_wait(&full[stage], phase);
      if (threadIdx.x == 0) gqa_trace(1, gc);  // 1: page landed at consumer warp 0
      const uint32_t kbase = smem_u32(ring + stage * S::kStageBytes);
      const uint32_t vbase = kbase + S::kTileBytes;
      const int tok0 = warp * 16;  // this warp's 16 tokens of the page
      // ---- S = Q K^T for 16 tokens (two n-tiles of 8) ----
      float s0[4] = {0.f, 0.f, 0.f, 0.f}, s1[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int ks = 0; ks < KSTEPS; ++ks) {
        // matrices: (chunk 2ks, tok0..+7), (chunk 2ks+1, tok0..+7), (chunk 2ks, tok0+8..), (chunk 2ks+1, tok0+8..)
        const int mi = lane >> 3, r = lane & 7;
        const int chunk = 2 * ks + (mi & 1);
        const int tok = tok0 + ((mi >> 1) << 3) + r;
        uint32_t b00, b01, b10, b11;
        ldsm_x4(kbase + (uint32_t)((chunk * kPage + tok) * 16), b00, b01, b10, b11);
        mma_bf16_16816(s0, qa[ks][0], 0u, qa[ks][1], 0u, b00, b01);
        mma_bf16_16816(s1, qa[ks][0], 0u, qa[ks][1], 0u, b10, b11);
      }
      // ---- online softmax over this warp's tokens (row g; columns 2t,2t+1 and 8+2t,8+2t+1) ----
      const int n_valid = len - p * kPage - tok0;  // tokens of this warp that exist
      float x0 = (2 * t < n_valid) ? s0[0] * scale_log2 : -INFINITY;
      float x1 = (2 * t + 1 < n_valid) ? s0[1] * scale_log2 : -INFINITY;
      float x2 = (8 + 2 * t < n_valid) ? s1[0] * scale_log2 : -INFINITY;
      float x3 = (8 + 2 * t + 1 < n_valid) ? s1[1] * scale_log2 : -INFINITY;
      float mt = fmaxf(fmaxf(x0, x1), fmaxf(x2, x3));
      mt = fmaxf(mt, __shfl_xor_sync(0xffffffffu, mt, 1));
      mt = fmaxf(mt, __shfl_xor_sync(0xffffffffu, mt, 2));
      const float m_new = fmaxf(m_run, mt);
      const float m_use = (m_new == -INFINITY) ? 0.f : m_new;
      const float alpha = exp2f(m_run - m_use);
      const float p0 = exp2f(x0 - m_use), p1 = exp2f(x1 - m_use), p2 = exp2f(x2 - m_use), p3 = exp2f(x3 - m_use);
      l_run = l_run * alpha + (p0 + p1 + p2 + p3);
      m_run = m_new;
#pragma unroll
      for (int n = 0; n < NT; ++n) {
        o[n][0] *= alpha;
        o[n][1] *= alpha;
      }
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
      // P as the A operand (k = 16 tokens): rows >= G are zero
      const uint32_t pa0 = row_ok ? pack_bf16x2(p0, p1) : 0u;
      const uint32_t pa2 = row_ok ? pack_bf16x2(p2, p3) : 0u;
      // ---- O += P V : two dim-chunks (n-tiles) per ldmatrix.x4.trans ----
#pragma unroll
      for (int n2 = 0; n2 < NT / 2; ++n2) {
        const int mi = lane >> 3, r = lane & 7;
        const int chunk = 2 * n2 + (mi >> 1);
        const int tok = tok0 + ((mi & 1) << 3) + r;
        uint32_t v0a, v0b, v1a, v1b;
        ldsm_x4_t(vbase + (uint32_t)((chunk * kPage + tok) * 16), v0a, v0b, v1a, v1b);
        mma_bf16_16816(o[2 * n2], pa0, 0u, pa2, 0u, v0a, v0b);
        mma_bf16_16816(o[2 * n2 + 1], pa0, 0u, pa2, 0u, v1a, v1b);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (threadIdx.x == 0) gqa_trace(2, gc);  // 2: page released by consumer warp 0
      if (++stage == kAttnStages) { stage = 0; phase ^= 1; }
    }

    // ---- merge the 4 warps' partial (m, l, O) and store ----
    if (threadIdx.x == 0) gqa_trace(5, item);  // 5: merge start
    l_run += __shfl_xor_sync(0xffffffffu, l_run, 1);
    l_run += __shfl_xor_sync(0xffffffffu, l_run, 2);
    constexpr int MS = S::kMergeStride;
    float* mo = merge + warp * MS;
    if (row_ok) {
#pragma unroll
      for (int n = 0; n < NT; ++n) {
        mo[g * HD + n * 8 + 2 * t] = o[n][0];
        mo[g * HD + n * 8 + 2 * t + 1] = o[n][1];
      }
      if (t == 0) {
        mo[G * HD + g] = m_run;
        mo[G * HD + 8 + g] = l_run;
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
    if (lane == 0) mbar_arrive(&item_empty[item & 3]);
    if (threadIdx.x == 0) gqa_trace(6, item);  // 6: merge done
  }
  // the last CTA out (all grabs of every CTA done) resets the scheduler for the next launch
  if (sched && threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(sched + 1, 1) == (int)gridDim.x - 1) {
      sched[0] = 0;
      sched[1] = 0;
    }
  }
}

template <int HD, int G>
int launch_gqa(const void* q, const void* kc, const void* vc, const int* bt, int max_pages, const int* lens, int B,
               int Hkv, float scale, void* out, cudaStream_t st, int* sched, const GqaRope& rp) {
  using S = GqaSmem<HD, G>;
  if (const int rc = mgb_host::ensure_max_smem((const void*)decode_attn_gqa_kernel<HD, G>, (int)S::kBytes)) return rc;
  const int items = B * Hkv;
  int sms = mgb_host::num_sms();
  if (const char* e = getenv("MGB_ATTN_SMS")) {  // leave SMs to a concurrent stream (overlap experiments)
    const int cap = atoi(e);
    if (cap > 0 && cap < sms) sms = cap;
  }
  int grid = 2 * sms;
  if (grid > items) grid = items;
  mgb_host::launch(decode_attn_gqa_kernel<HD, G>, dim3(grid), dim3(kAttnThreads), S::kBytes, st, nullptr,
      reinterpret_cast<const __nv_bfloat16*>(q), reinterpret_cast<const __nv_bfloat16*>(kc),
      reinterpret_cast<const __nv_bfloat16*>(vc), bt, max_pages, lens, B, Hkv, scale * 1.4426950408889634f,
      reinterpret_cast<__nv_bfloat16*>(out), sched, rp);
  return mgb_host::launch_status();
}

}  // namespace mgb

namespace {
int gqa_dispatch(const void* q, const void* k_cache, const void* v_cache, const int* block_table, int max_pages,
                 const int* seq_lens, int B, int Hq, int Hkv, int head_dim, float scale, void* out, int* sched,
                 const mgb::GqaRope& rp, cudaStream_t st) {
  const int G = Hq / Hkv;
#define MGB_GQA_CASE(HD_, G_) \
  if (head_dim == HD_ && G == G_)                                                                                  \
    return mgb::launch_gqa<HD_, G_>(q, k_cache, v_cache, block_table, max_pages, seq_lens, B, Hkv, scale, out, st, \
                                    sched, rp);
  MGB_GQA_CASE(128, 4)
  MGB_GQA_CASE(128, 6)
  MGB_GQA_CASE(128, 8)
  MGB_GQA_CASE(64, 4)
  MGB_GQA_CASE(32, 4)
#undef MGB_GQA_CASE
  return MGB_EINVAL;
}
}  // namespace

extern "C" {

int mgb_kv_page_size(void) { return mgb::kPage; }

// Copy the GQA trace buffer (MGB_GQA_TRACE builds) to host_out[8 * 512]; MGB_EINVAL otherwise.
int mgb_gqa_trace_read(unsigned long long* host_out) {
#ifdef MGB_GQA_TRACE
  return cudaMemcpyFromSymbol(host_out, mgb::g_gqa_trace, sizeof(mgb::g_gqa_trace)) == cudaSuccess ? MGB_OK : MGB_ECUDA;
#else
  (void)host_out;
  return MGB_EINVAL;
#endif
}

// Decode attention for B sequences, one new query token each (already RoPE'd and appended to
// the cache by mgb_rope_append_gqa).  seq_lens[b] counts the cached tokens including the new one.
int mgb_decode_attn_gqa_sched(const void* q, const void* k_cache, const void* v_cache, const int* block_table,
                              int max_pages, const int* seq_lens, int B, int Hq, int Hkv, int head_dim, float scale,
                              void* out, int* sched, void* stream);

int mgb_decode_attn_gqa(const void* q, const void* k_cache, const void* v_cache, const int* block_table,
                        int max_pages, const int* seq_lens, int B, int Hq, int Hkv, int head_dim, float scale,
                        void* out, void* stream) {
  return mgb_decode_attn_gqa_sched(q, k_cache, v_cache, block_table, max_pages, seq_lens, B, Hq, Hkv, head_dim, scale,
                                   out, nullptr, stream);
}

// Same, with dynamic item scheduling through `sched` (2 ints, zero before the first launch and left
// zero by every launch; one per stream).
int mgb_decode_attn_gqa_sched(const void* q, const void* k_cache, const void* v_cache, const int* block_table,
                              int max_pages, const int* seq_lens, int B, int Hq, int Hkv, int head_dim, float scale,
                              void* out, int* sched, void* stream) {
  if (B < 1 || Hkv < 1 || Hq % Hkv) return MGB_EINVAL;
  return gqa_dispatch(q, k_cache, v_cache, block_table, max_pages, seq_lens, B, Hq, Hkv, head_dim, scale, out, sched,
                      mgb::GqaRope{}, reinterpret_cast<cudaStream_t>(stream));
}

// Decode attention with the step's RoPE + KV append fused in (replaces mgb_rope_append_gqa +
// mgb_decode_attn_gqa_sched for resident paged KV): qkv [B, (Hq + 2 Hkv) * head_dim] are the raw
// projections of the B new tokens, positions[b] their positions; the new k (rotated) and v land in
// the token's slot of its page, seq_lens[b] = positions[b] + 1, out = attention over positions
// 0..positions[b].  Same numerics as the two-launch path (tests/test_kernels_gpu.py).
int mgb_decode_attn_gqa_rope(const void* qkv, const int* positions, const float* cos_t, const float* sin_t,
                             void* k_cache, void* v_cache, const int* block_table, int max_pages, int* seq_lens, int B,
                             int Hq, int Hkv, int head_dim, float scale, void* out, int* sched, void* stream) {
  if (B < 1 || Hkv < 1 || Hq % Hkv || !qkv || !positions || !cos_t || !sin_t || !seq_lens) return MGB_EINVAL;
  const mgb::GqaRope rp{reinterpret_cast<const __nv_bfloat16*>(qkv), positions, cos_t, sin_t,
                        reinterpret_cast<__nv_bfloat16*>(k_cache), reinterpret_cast<__nv_bfloat16*>(v_cache), seq_lens};
  return gqa_dispatch(nullptr, k_cache, v_cache, block_table, max_pages, seq_lens, B, Hq, Hkv, head_dim, scale, out,
                      sched, rp, reinterpret_cast<cudaStream_t>(stream));
}

}  // extern "C"
