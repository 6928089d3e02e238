// Fused MoE routing front end for the decode step (sm_100a): the post-attention residual add +
// RMSNorm, the router logits (tensor cores, mma.sync), softmax / top-k, the per-expert counts and
// offsets, and the stable expert-major permutation -- ONE launch where the unfused path runs four
// (add_rmsnorm, a cuBLAS logits GEMM, router_topk, permute).
//
// Replaces the ROUTER job of the module-based batching schedule and the token grouping in front
// of EXPERT_COMPUTE (reference: pkg/src/moe_planner/offload_dag.py:418-463; cost model
// hw_profile.py:273-275,291-292).  Semantics are those of routing.cu (HF transformers 5.5.0
// Mixtral / DeepSeek-V2 routing, pinned selection order) and elementwise.cu's add_rmsnorm (HF
// MixtralRMSNorm rounding); the permutation is the same stable sort of (t, j) entries by expert.
//
// Structure: a persistent grid of G co-resident CTAs (G <= half the device's resident capacity, so
// two such kernels on different streams can never starve each other), each owning <= kMaxOwn
// 8-token chunks:
//   phase 1 (per chunk): residual add + RMSNorm (warp per token, the normalised rows stay in smem),
//            logits = H_chunk W_r^T on mma.sync m16n8k16 (16 tokens x 8 experts per tile, K split
//            across warps when E is small), softmax + top-k (warp per token), chunk histogram and
//            stable in-chunk ranks;
//   grid barrier (the only one; one atomic per CTA on its critical path);
//   phase 2: every CTA scans the chunk histograms it needs (its chunks' exclusive bases and the
//            expert totals -> offsets), then copies its tokens' normalised rows to their permuted
//            positions (from smem for its last chunk).
#include <algorithm>

#include "common.cuh"

namespace mgb {

constexpr int kRteTPC = 8;        // tokens per chunk (half the MMA M: rows 8-15 of the A tile alias 0-7)
constexpr int kRteThreads = 256;  // 8 warps: one token of a chunk per warp
constexpr int kRteWarps = kRteThreads / 32;
constexpr int kRteMaxE = 256;
constexpr int kRteMaxK = 8;
constexpr int kRteMaxOwn = 4;     // chunks per CTA
constexpr int kRteU = 4;          // 16-byte vectors per lane in flight in the permutation copies
constexpr int kRteDU = 8;         // delta vectors per lane in flight per batch
constexpr int kRteKB = 8;         // k-steps of router-weight fragments per batch beyond the preload
constexpr int kRteKPre = 24;      // k-steps of router-weight fragments preloaded per warp (8 before the
                                  // norm, the rest while the norm's smem pass runs; 32 spills next to
                                  // the 8 delta vectors per lane in flight)

struct RouteArgs {
  const __nv_bfloat16* x;      // [T, d] residual stream
  const __nv_bfloat16* delta;  // optional [T, d] (attention output): x <- bf16(x + delta)
  const __nv_bfloat16* ln_w;   // [d]
  float eps;
  int T, d, E, k, mode;
  float scaling;
  int n_group, topk_group;
  const __nv_bfloat16* wr;     // [E, d] router weight
  __nv_bfloat16* x_out;        // optional [T, d] (may alias x)
  __nv_bfloat16* h_out;        // optional [T, d] normalised rows (required when a CTA owns > 1 chunk)
  float* logits_out;           // optional [T, E]
  int* topk_idx;               // [T, k]
  float* topk_w;               // [T, k]
  int* local_rank;             // [T, k] rank among same-expert entries of the chunk
  int* chunk_hist;             // [nchunks, E]
  int* counts;                 // [E]
  int* offsets;                // [E + 1]
  __nv_bfloat16* x_perm;       // [T * k, d]
  int* src_token;              // [T * k]
  int* dst_pos;                // [T * k]
  int* sync;                   // [2] grid barrier {arrivals, generation}, zero on first use
  int nchunks;
  long long* stamps;           // optional [G][16] globaltimer per phase (tools/route_bench.py --phases)
  int bulk_perm;               // permuted rows leave smem as TMA bulk stores (else st.global.v4 per lane)
};

MGB_DEVINL long long rte_globaltimer() {
  long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define MGB_RTE_STAMP(i) \
  if (a.stamps && threadIdx.x == 0) a.stamps[blockIdx.x * 16 + (i)] = rte_globaltimer()

MGB_DEVINL bool rte_better(float va, int ia, float vb, int ib) { return va > vb || (va == vb && ia < ib); }

MGB_DEVINL void rte_argbest(float& v, int& i) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, v, o);
    const int oi = __shfl_xor_sync(0xffffffffu, i, o);
    if (rte_better(ov, oi, v, i)) { v = ov; i = oi; }
  }
}
MGB_DEVINL float rte_wmax(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
MGB_DEVINL float rte_wsum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

MGB_DEVINL void rte_ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
MGB_DEVINL void rte_mma(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
MGB_DEVINL int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Grid barrier over G co-resident CTAs with ONE atomic per CTA on the critical path: CTA 0 adds
// 2^31 - (G - 1), every other CTA adds 1, so the word's top bit flips exactly when the last CTA
// arrives and every CTA waits for that flip (no reset / generation round trips).  The low 31 bits
// return to their value each launch, so the workspace is reusable by the next launch with any G
// (and by graph replays); only sync[0] is used.
MGB_DEVINL void grid_barrier(int* sync, int G) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned add = blockIdx.x == 0 ? 0x80000000u - (unsigned)(G - 1) : 1u;
    __threadfence();  // release this CTA's phase-1 writes
    const unsigned old = atomicAdd(reinterpret_cast<unsigned*>(sync), add);
    while (((old ^ (unsigned)ld_acquire_gpu(sync)) & 0x80000000u) == 0) __nanosleep(20);
    __threadfence();
  }
  __syncthreads();
}

struct RteSmem {
  int hstride;  // bf16 elements per smem row (d + 8: rows 16 B apart in bank terms)
  __nv_bfloat16* h;  // [16][hstride]
  float* logit;      // [16][E]
  float* part;       // [8 warps][16][8]
  int* exp;          // [16 * k]
  __nv_bfloat16* lnw;  // [d] norm weight (staged once per CTA)
};

__global__ void __launch_bounds__(kRteThreads, 2) moe_route_kernel(RouteArgs a) {
  mgb::pdl_enter();
  extern __shared__ __align__(16) uint8_t smem[];
  const int d = a.d, E = a.E, k = a.k;
  MGB_RTE_STAMP(9);
  RteSmem s;
  s.hstride = d + 8;
  s.h = reinterpret_cast<__nv_bfloat16*>(smem);
  s.logit = reinterpret_cast<float*>(smem + (size_t)kRteTPC * s.hstride * 2);
  s.part = s.logit + kRteTPC * E;
  s.exp = reinterpret_cast<int*>(s.part + kRteWarps * kRteTPC * 8);
  s.lnw = reinterpret_cast<__nv_bfloat16*>(s.exp + kRteTPC * kRteMaxK);
  __shared__ __align__(8) uint64_t s_xbar;  // the chunk's x rows landed (bulk copies)
  for (int i = threadIdx.x; i < d / 8; i += kRteThreads)
    reinterpret_cast<uint4*>(s.lnw)[i] = ld_nc_v4(reinterpret_cast<const uint4*>(a.ln_w) + i);
  if (threadIdx.x == 0) {
    mbar_init(&s_xbar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  __shared__ int s_tot[kRteMaxE];
  __shared__ int s_off[kRteMaxE + 1];
  __shared__ int s_base[kRteMaxOwn][kRteMaxE];
  __shared__ int s_red[kRteThreads];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = gridDim.x;
  const int nvec = d / 8;
  int n_own = 0;

  // ======================= phase 1: per owned chunk =======================
  MGB_RTE_STAMP(0);
  for (int c = blockIdx.x; c < a.nchunks; c += G, ++n_own) {
    const int t0 = c * kRteTPC;
    const int ntok = min(kRteTPC, a.T - t0);
    // ---- logits work split (fixed per warp): n-tile nt0 (+8, +16, ...) over k-steps [ks0, ks1) ----
    const int ntiles = (E + 7) / 8;
    const int ksplit = ntiles >= kRteWarps ? 1 : kRteWarps / ntiles;
    const int ksteps = d / 16;
    const int kper = (ksteps + ksplit - 1) / ksplit;
    const int kpart = ntiles >= kRteWarps ? 0 : warp / ntiles;
    const int nt0 = ntiles >= kRteWarps ? warp : warp % ntiles;
    const bool mma_warp = kpart < ksplit && nt0 < ntiles;
    const int ks0 = kpart * kper, ks1 = min(ksteps, ks0 + kper);
    // router-weight fragments of the warp's first n-tile do not depend on the norm: the first 8
    // k-steps are requested before it, the next 24 once the delta loads have landed (the norm's smem
    // pass hides them), so a d <= 4096 row waits for one fragment batch in the logits phase instead of three
    uint32_t bpre[kRteKPre][2];
    auto load_b = [&](uint32_t (&b)[kRteKB][2], int nt, int ks) {
      const int n = nt * 8 + (lane >> 2);
      const uint32_t* wrow = reinterpret_cast<const uint32_t*>(a.wr + (size_t)(n < E ? n : 0) * d) + (lane & 3);
#pragma unroll
      for (int u = 0; u < kRteKB; ++u) {
        const bool ok = n < E && ks + u < ks1;
        b[u][0] = ok ? __ldg(wrow + (ks + u) * 8) : 0u;
        b[u][1] = ok ? __ldg(wrow + (ks + u) * 8 + 4) : 0u;
      }
    };
    auto load_pre = [&](int u0, int u1) {
      const int n = nt0 * 8 + (lane >> 2);
      const uint32_t* wrow = reinterpret_cast<const uint32_t*>(a.wr + (size_t)(n < E ? n : 0) * d) + (lane & 3);
#pragma unroll
      for (int u = 0; u < kRteKPre; ++u) {
        if (u < u0 || u >= u1) continue;
        const bool ok = mma_warp && n < E && ks0 + u < ks1;
        bpre[u][0] = ok ? __ldg(wrow + (ks0 + u) * 8) : 0u;
        bpre[u][1] = ok ? __ldg(wrow + (ks0 + u) * 8 + 4) : 0u;
      }
    };
    load_pre(0, kRteKB);
    bool pre_rest = false;

    // ---- residual add + RMSNorm, warp per token; rows land in smem (and h_out) ----
    // the chunk's x rows arrive by bulk copy (TMA engine) while every lane has all of its delta
    // vectors in flight: one memory round trip per chunk instead of one per vector batch
    if (threadIdx.x == 0) {
      fence_proxy_async_smem();  // the previous chunk's generic writes to s.h precede the async-proxy fill
      mbar_arrive_expect_tx(&s_xbar, (uint32_t)ntok * d * 2);
      for (int tl = 0; tl < ntok; ++tl)
        bulk_load(s.h + (size_t)tl * s.hstride, a.x + (size_t)(t0 + tl) * d, (uint32_t)d * 2, &s_xbar,
                  policy_evict_normal());
    }
    for (int tl = warp; tl < kRteTPC; tl += kRteWarps) {
      uint4* srow = reinterpret_cast<uint4*>(s.h + (size_t)tl * s.hstride);
      if (tl >= ntok) {  // tail rows of the last chunk: zeros (they never leave smem)
        for (int cc = lane; cc < nvec; cc += 32) srow[cc] = make_uint4(0, 0, 0, 0);
        continue;
      }
      const size_t t = (size_t)(t0 + tl);
      const uint4* dr = a.delta ? reinterpret_cast<const uint4*>(a.delta + t * d) : nullptr;
      float ss = 0.f;
      bool landed = false;
      for (int c0 = lane; c0 < nvec; c0 += 32 * kRteDU) {
        uint4 dv[kRteDU];
        if (dr) {
#pragma unroll
          for (int u = 0; u < kRteDU; ++u)
            if (c0 + 32 * u < nvec) dv[u] = ld_nc_v4(dr + c0 + 32 * u);
        }
        if (!landed) {
          mbar_wait(&s_xbar, n_own & 1);
          landed = true;
        }
#pragma unroll
        for (int u = 0; u < kRteDU; ++u) {
          const int cc = c0 + 32 * u;
          if (cc >= nvec) continue;
          uint4 v = srow[cc];
          if (dr) {
            v.x = pack_bf16x2(bf16lo(v.x) + bf16lo(dv[u].x), bf16hi(v.x) + bf16hi(dv[u].x));
            v.y = pack_bf16x2(bf16lo(v.y) + bf16lo(dv[u].y), bf16hi(v.y) + bf16hi(dv[u].y));
            v.z = pack_bf16x2(bf16lo(v.z) + bf16lo(dv[u].z), bf16hi(v.z) + bf16hi(dv[u].z));
            v.w = pack_bf16x2(bf16lo(v.w) + bf16lo(dv[u].w), bf16hi(v.w) + bf16hi(dv[u].w));
            srow[cc] = v;
          }
          if (a.x_out) reinterpret_cast<uint4*>(a.x_out + t * d)[cc] = v;
          const float f[8] = {bf16lo(v.x), bf16hi(v.x), bf16lo(v.y), bf16hi(v.y),
                              bf16lo(v.z), bf16hi(v.z), bf16lo(v.w), bf16hi(v.w)};
#pragma unroll
          for (int i = 0; i < 8; ++i) ss = fmaf(f[i], f[i], ss);
        }
      }
      if (!pre_rest) {  // the delta registers are dead: the remaining preloaded fragments go in flight
        load_pre(kRteKB, kRteKPre);
        pre_rest = true;
      }
      const float inv = 1.0f / sqrtf(rte_wsum(ss) / (float)d + a.eps);
      const uint4* wr = reinterpret_cast<const uint4*>(s.lnw);
      uint4* hr = a.h_out ? reinterpret_cast<uint4*>(a.h_out + t * d) : nullptr;
      for (int cc = lane; cc < nvec; cc += 32) {  // smem only: no memory round trip per vector
        const uint4 v = srow[cc], wv = wr[cc];
        uint4 o;
        o.x = pack_bf16x2(bf16lo(wv.x) * bf16_round(bf16lo(v.x) * inv), bf16hi(wv.x) * bf16_round(bf16hi(v.x) * inv));
        o.y = pack_bf16x2(bf16lo(wv.y) * bf16_round(bf16lo(v.y) * inv), bf16hi(wv.y) * bf16_round(bf16hi(v.y) * inv));
        o.z = pack_bf16x2(bf16lo(wv.z) * bf16_round(bf16lo(v.z) * inv), bf16hi(wv.z) * bf16_round(bf16hi(v.z) * inv));
        o.w = pack_bf16x2(bf16lo(wv.w) * bf16_round(bf16lo(v.w) * inv), bf16hi(wv.w) * bf16_round(bf16hi(v.w) * inv));
        srow[cc] = o;
        if (hr) hr[cc] = o;
      }
    }
    if (!pre_rest) load_pre(kRteKB, kRteKPre);  // warps whose token row is a tail row
    if (a.bulk_perm) fence_proxy_async_smem();  // the normalised rows leave smem by bulk stores
    __syncthreads();

    MGB_RTE_STAMP(1);
    // ---- logits[16 tokens][E] = H W_r^T on mma.sync (bf16 in, fp32 accumulate) ----
    {
      const uint32_t hbase = smem_u32(s.h);
      // ldmatrix.x4 row address of this lane: rows 0-15, the lane's 8-column half
      // (rows 8-15 of the 16-row A tile alias rows 0-7: their results are discarded)
      const uint32_t arow = hbase + (uint32_t)((lane & 7) * s.hstride + (lane >> 4) * 8) * 2;
      for (int nt = nt0; mma_warp && nt < ntiles; nt += kRteWarps) {
        float acc[4] = {0.f, 0.f, 0.f, 0.f};
        int ks = ks0;
        if (nt == nt0) {  // the preloaded fragments
#pragma unroll
          for (int u = 0; u < kRteKPre; ++u) {
            if (ks0 + u < ks1) {
              uint32_t a0, a1, a2, a3;
              rte_ldsm_x4(arow + (ks0 + u) * 32, a0, a1, a2, a3);
              rte_mma(acc, a0, a1, a2, a3, bpre[u][0], bpre[u][1]);
            }
          }
          ks = ks0 + kRteKPre;
        }
        for (; ks < ks1; ks += kRteKB) {  // wider rows / further n-tiles: kRteKB k-steps per batch
          uint32_t bcur[kRteKB][2];
          load_b(bcur, nt, ks);
#pragma unroll
          for (int u = 0; u < kRteKB; ++u) {
            if (ks + u < ks1) {
              uint32_t a0, a1, a2, a3;
              rte_ldsm_x4(arow + (ks + u) * 32, a0, a1, a2, a3);
              rte_mma(acc, a0, a1, a2, a3, bcur[u][0], bcur[u][1]);
            }
          }
        }
        // c0,c1: token lane/4, experts 2*(lane%4)+{0,1}; c2,c3: token lane/4 + 8
        const int r = lane >> 2, cn = 2 * (lane & 3);
        if (ksplit == 1) {
          const int e0 = nt * 8 + cn;
          if (e0 < E) s.logit[r * E + e0] = acc[0];
          if (e0 + 1 < E) s.logit[r * E + e0 + 1] = acc[1];
        } else {
          float* p = s.part + warp * kRteTPC * 8;
          p[r * 8 + cn] = acc[0];
          p[r * 8 + cn + 1] = acc[1];
        }
      }
      if (ksplit > 1) {
        __syncthreads();
        for (int i = threadIdx.x; i < kRteTPC * E; i += kRteThreads) {
          const int r = i / E, e = i - r * E, nt = e >> 3;
          float v = 0.f;
          for (int kp = 0; kp < ksplit; ++kp) v += s.part[(kp * ntiles + nt) * kRteTPC * 8 + r * 8 + (e & 7)];
          s.logit[r * E + e] = v;
        }
      }
    }
    __syncthreads();

    MGB_RTE_STAMP(2);
    // ---- softmax + pinned-order top-k, warp per token ----
    for (int tl = warp; tl < ntok; tl += kRteWarps) {
      const int t = t0 + tl;
      float* lg = s.logit + tl * E;
      if (a.mode == 0)  // Mixtral's router linear is a bf16 GEMM (modeling_mixtral.py:111)
        for (int e = lane; e < E; e += 32) lg[e] = bf16_round(lg[e]);
      __syncwarp();
      if (a.logits_out)
        for (int e = lane; e < E; e += 32) a.logits_out[(size_t)t * E + e] = lg[e];
      float m = -INFINITY;
      for (int e = lane; e < E; e += 32) m = fmaxf(m, lg[e]);
      m = rte_wmax(m);
      float sum = 0.f;
      for (int e = lane; e < E; e += 32) sum += expf(lg[e] - m);
      sum = rte_wsum(sum);
      const float inv = 1.0f / sum;
      uint32_t group_ok = 0xffffffffu;
      const int gsz = (a.mode == 2) ? E / a.n_group : E;
      if (a.mode == 2) {
        float gbest = -INFINITY;
        int gi = 0x7fffffff;
        if (lane < a.n_group) {
          for (int e = lane * gsz; e < (lane + 1) * gsz; ++e) gbest = fmaxf(gbest, lg[e]);
          gi = lane;
        }
        group_ok = 0;
        for (int r = 0; r < a.topk_group; ++r) {
          float v = (group_ok >> lane) & 1u ? -INFINITY : gbest;
          int i = (group_ok >> lane) & 1u ? 0x7fffffff : gi;
          if (lane >= a.n_group) { v = -INFINITY; i = 0x7fffffff; }
          rte_argbest(v, i);
          group_ok |= 1u << i;
        }
      }
      uint32_t taken[kRteMaxE / 32] = {0, 0, 0, 0, 0, 0, 0, 0};
      float psel[kRteMaxK];
      int isel[kRteMaxK];
      for (int r = 0; r < k; ++r) {
        float bv = -INFINITY;
        int bi = 0x7fffffff;
        for (int e = lane, w = 0; e < E; e += 32, ++w) {
          if ((taken[w] >> lane) & 1u) continue;
          if (a.mode == 2 && !((group_ok >> (e / gsz)) & 1u)) continue;
          if (rte_better(lg[e], e, bv, bi)) { bv = lg[e]; bi = e; }
        }
        rte_argbest(bv, bi);
        if ((bi & 31) == lane) taken[bi >> 5] |= 1u << lane;
        isel[r] = bi;
        psel[r] = expf(lg[bi] - m) * inv;
      }
      if (lane == 0) {
        float denom = 0.f;
        for (int r = 0; r < k; ++r) denom += psel[r];
        for (int r = 0; r < k; ++r) {
          a.topk_idx[(size_t)t * k + r] = isel[r];
          a.topk_w[(size_t)t * k + r] = (a.mode == 0) ? psel[r] / denom : psel[r] * a.scaling;
          s.exp[tl * k + r] = isel[r];
        }
      }
    }
    __syncthreads();

    MGB_RTE_STAMP(3);
    // ---- chunk histogram + stable in-chunk ranks ----
    const int nent = ntok * k;
    for (int i = threadIdx.x; i < nent; i += kRteThreads) {
      const int e = s.exp[i];
      int r = 0;
      for (int j = 0; j < i; ++j) r += (s.exp[j] == e);
      a.local_rank[(size_t)t0 * k + i] = r;
    }
    for (int e = threadIdx.x; e < E; e += kRteThreads) {
      int cnt = 0;
      for (int j = 0; j < nent; ++j) cnt += (s.exp[j] == e);
      a.chunk_hist[(size_t)c * E + e] = cnt;
    }
    MGB_RTE_STAMP(4);
    __syncthreads();  // s.h / s.exp are reused by the next chunk
  }

  // ======================= grid barrier =======================
  MGB_RTE_STAMP(5);
  grid_barrier(a.sync, G);
  MGB_RTE_STAMP(6);

  // ======================= phase 2: bases, offsets, permutation =======================
  {
    // thread (e, part): sums column e over chunks part, part + nparts, ...; the bases of this CTA's
    // chunks are the sums over earlier chunks
    const int nparts = kRteThreads / E;  // >= 1 (E <= 256)
    const int e = threadIdx.x % E, part = threadIdx.x / E;
    int tot = 0;
    int pre[kRteMaxOwn] = {0, 0, 0, 0};
    if (part < nparts) {
#pragma unroll 8
      for (int c = part; c < a.nchunks; c += nparts) {
        const int v = __ldcg(a.chunk_hist + (size_t)c * E + e);
        tot += v;
#pragma unroll
        for (int i = 0; i < kRteMaxOwn; ++i)
          if (c < (int)blockIdx.x + i * G) pre[i] += v;
      }
    }
    // reduce over parts (in part order), one quantity at a time
    for (int q = 0; q <= n_own; ++q) {
      int mine = q == 0 ? tot : 0;
#pragma unroll
      for (int i = 0; i < kRteMaxOwn; ++i)
        if (q == i + 1) mine = pre[i];
      s_red[threadIdx.x] = (part < nparts) ? mine : 0;
      __syncthreads();
      if (threadIdx.x < E) {
        int v = 0;
        for (int p = 0; p < nparts; ++p) v += s_red[p * E + threadIdx.x];
        if (q == 0) s_tot[threadIdx.x] = v;
        else s_base[q - 1][threadIdx.x] = v;
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      int run = 0;
      for (int i = 0; i < E; ++i) {
        s_off[i] = run;
        run += s_tot[i];
      }
      s_off[E] = run;
    }
    __syncthreads();
    if (blockIdx.x == 0) {
      for (int i = threadIdx.x; i <= E; i += kRteThreads) {
        a.offsets[i] = s_off[i];
        if (i < E) a.counts[i] = s_tot[i];
      }
    }
  }
  MGB_RTE_STAMP(7);
  // permutation: warp per (token, slot) entry; the last chunk's rows are still in smem
  for (int i = 0; i < n_own; ++i) {
    const int c = blockIdx.x + i * G;
    const int t0 = c * kRteTPC;
    const int nent = min(kRteTPC, a.T - t0) * k;
    const bool in_smem = i == n_own - 1;
    for (int q = warp; q < nent; q += kRteWarps) {
      const int gi = t0 * k + q;
      const int t = gi / k;
      const int e = a.topk_idx[gi];
      const int pos = s_off[e] + s_base[i][e] + a.local_rank[gi];
      if (lane == 0) {
        a.dst_pos[gi] = pos;
        a.src_token[pos] = t;
      }
      const uint4* src = in_smem ? reinterpret_cast<const uint4*>(s.h + (size_t)(t - t0) * s.hstride)
                                 : reinterpret_cast<const uint4*>(a.h_out + (size_t)t * d);
      uint4* dst = reinterpret_cast<uint4*>(a.x_perm + (size_t)pos * d);
      if (in_smem && a.bulk_perm) {  // one TMA bulk store per (token, slot) row
        if (lane == 0) bulk_store(dst, src, (uint32_t)d * 2);
        continue;
      }
      for (int c0 = lane; c0 < nvec; c0 += 32 * kRteU) {
        uint4 v[kRteU];
#pragma unroll
        for (int u = 0; u < kRteU; ++u)
          if (c0 + 32 * u < nvec) v[u] = src[c0 + 32 * u];
#pragma unroll
        for (int u = 0; u < kRteU; ++u)
          if (c0 + 32 * u < nvec) dst[c0 + 32 * u] = v[u];
      }
    }
  }
  if (a.bulk_perm && lane == 0) {  // smem must outlive the bulk stores' reads
    bulk_commit();
    bulk_wait_read_all();
  }
  MGB_RTE_STAMP(8);
}

// Allow the largest dynamic smem the device offers once per device (the attribute is per kernel and
// device, and a smaller value set for a narrow d would cap the occupancy query of a wider one).
int route_prepare() {
  int dev = 0, optin = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess)
    return mgb_host::launch_status(), MGB_ECUDA;
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, moe_route_kernel) != cudaSuccess) return mgb_host::launch_status(), MGB_ECUDA;
  return mgb_host::ensure_max_smem((const void*)moe_route_kernel, optin - (int)fa.sharedSizeBytes);
}

size_t route_smem(int d, int E) {
  return (size_t)kRteTPC * (d + 8) * 2 + sizeof(float) * (kRteTPC * E + kRteWarps * kRteTPC * 8) +
         sizeof(int) * kRteTPC * kRteMaxK + (size_t)d * 2;
}

}  // namespace mgb

namespace {
long long* g_route_stamps = nullptr;  // phase timestamps of the next launches (profiling only)
}

extern "C" {

// Profiling hook: record per-CTA globaltimer stamps of mgb_moe_route's phases into stamps[G][16]
// (device memory) on subsequent launches; NULL turns it off.
int mgb_moe_route_stamps(long long* stamps) {
  g_route_stamps = stamps;
  return MGB_OK;
}

// Rows of the chunk_hist workspace mgb_moe_route needs for T tokens (8-token chunks).
int mgb_moe_route_chunks(int T) { return (T + mgb::kRteTPC - 1) / mgb::kRteTPC; }

// Fused decode routing front end (see the file comment).  sync: 2 ints, zero before first use, left
// reusable.  Returns MGB_EINVAL when T exceeds what one co-resident grid covers (the caller then
// runs mgb_add_rmsnorm + mgb_router_topk + mgb_permute).
int mgb_moe_route(const void* x, const void* delta, const void* ln_w, float eps, int T, int d, void* x_out,
                  void* h_out, const void* w_router, int E, int k, int mode, float scaling, int n_group,
                  int topk_group, float* logits_out, int* topk_idx, float* topk_w, int* local_rank, int* chunk_hist,
                  int* counts, int* offsets, void* x_perm, int* src_token, int* dst_pos, int* sync, void* stream) {
  if (T < 1 || d % 16 || d < 16 || E < 1 || E > mgb::kRteMaxE || k < 1 || k > mgb::kRteMaxK || k > E || mode < 0 ||
      mode > 2 || !sync || !x_perm)
    return MGB_EINVAL;
  if (mode == 2 && (n_group < 1 || n_group > 32 || E % n_group || topk_group < 1 || topk_group > n_group ||
                    topk_group * (E / n_group) < k))
    return MGB_EINVAL;
  const size_t smem = mgb::route_smem(d, E);
  if (smem > 227 * 1024) return MGB_EINVAL;
  if (const int rc = mgb::route_prepare()) return rc;
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, mgb::moe_route_kernel, mgb::kRteThreads, smem) !=
          cudaSuccess ||
      occ < 1)
    return mgb_host::launch_status(), MGB_ECUDA;
  const int nchunks = mgb_moe_route_chunks(T);
  const int cap = std::max(1, mgb_host::num_sms() * occ / 2);  // half the resident capacity
  const int G = std::min(nchunks, cap);
  if (nchunks > G * mgb::kRteMaxOwn) return MGB_EINVAL;
  if (!h_out && nchunks > G) return MGB_EINVAL;  // a CTA owning > 1 chunk permutes from h_out
  // MGB_ROUTE_BULK=1: permuted rows leave smem as TMA bulk stores.  Measured equal to the per-lane
  // st.global.v4 copies (tools/route_bench.py: 22.9 us both at Mixtral B=827/909), so off by default
  static const int bulk_perm = [] {
    const char* e = getenv("MGB_ROUTE_BULK");
    return e ? atoi(e) : 0;
  }();
  mgb::RouteArgs a{reinterpret_cast<const __nv_bfloat16*>(x), reinterpret_cast<const __nv_bfloat16*>(delta),
                   reinterpret_cast<const __nv_bfloat16*>(ln_w), eps, T, d, E, k, mode, scaling, n_group, topk_group,
                   reinterpret_cast<const __nv_bfloat16*>(w_router), reinterpret_cast<__nv_bfloat16*>(x_out),
                   reinterpret_cast<__nv_bfloat16*>(h_out), logits_out, topk_idx, topk_w, local_rank, chunk_hist,
                   counts, offsets, reinterpret_cast<__nv_bfloat16*>(x_perm), src_token, dst_pos, sync, nchunks,
                   g_route_stamps, bulk_perm};
  mgb_host::launch(mgb::moe_route_kernel, dim3(G), dim3(mgb::kRteThreads), smem, reinterpret_cast<cudaStream_t>(stream), nullptr,
      a);
  return mgb_host::launch_status();
}

// 1 if mgb_moe_route covers T tokens of width d routed over E experts on the current device (else the
// unfused path); 2 if it covers them in one pass (every CTA owns one chunk, so h_out may be NULL).
int mgb_moe_route_supported(int T, int d, int E) {
  if (T < 1 || d % 16 || E < 1 || E > mgb::kRteMaxE) return 0;
  const size_t smem = mgb::route_smem(d, E);
  if (smem > 227 * 1024) return 0;
  if (mgb::route_prepare()) return 0;
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, mgb::moe_route_kernel, mgb::kRteThreads, smem) !=
          cudaSuccess || occ < 1)
    return 0;
  const int cap = std::max(1, mgb_host::num_sms() * occ / 2);
  const int nchunks = mgb_moe_route_chunks(T);
  return nchunks <= cap ? 2 : nchunks <= cap * mgb::kRteMaxOwn ? 1 : 0;
}

}  // extern "C"
