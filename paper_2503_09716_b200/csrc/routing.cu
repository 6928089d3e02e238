// Router top-k, stable expert-major permutation, and weighted un-permute/combine (sm_100a).
//
// Replaces the ROUTER job of the module-based batching schedule
// (reference: pkg/src/moe_planner/offload_dag.py:418-425; cost hw_profile.py:273-275,291-292) and
// the implicit token grouping in front of the per-expert EXPERT_COMPUTE chunks
// (offload_dag.py:427-463).  Routing semantics follow HF transformers 5.5.0:
//   mode 0 (Mixtral, modeling_mixtral.py:109-116): logits = bf16(x W_g^T); p = softmax_fp32(logits);
//          top-k; w = p_sel / sum(p_sel).
//   mode 1 (DeepSeek-V2 greedy, modeling_deepseek_v2.py:100-105,125): logits = fp32(x) fp32(W_g)^T;
//          p = softmax_fp32; top-k; w = p_sel * routed_scaling_factor.
//   mode 2 (DeepSeek-V2 group_limited_greedy, :106-116): as mode 1 but experts restricted to the
//          top `topk_group` of `n_group` contiguous groups ranked by their max probability.
// Selection order is pinned (value descending, lower expert index first on ties) and is done on
// the logits (softmax is monotone), so indices are bit-exact given identical logits.
// The permutation is the stable sort of token-major flat entries (t*k + j) by expert
// (= HF grouped_mm's argsort with a stable tie rule, integrations/moe.py:368).
#include "common.cuh"

namespace mgb {

constexpr int kRouterTPB = 8;        // tokens per CTA
constexpr int kRouterThreads = 256;  // 8 warps: one token per warp in the selection phase
constexpr int kMaxE = 256;
constexpr int kMaxK = 8;

struct RouterArgs {
  const __nv_bfloat16* x;  // [T, d]
  const __nv_bfloat16* wg; // [E, d]
  const float* logits_in;  // optional [T, E]: skip the GEMV and route these logits
  int T, d, E, k, mode;
  float scaling;
  int n_group, topk_group;
  float* logits_out;       // optional [T, E]
  int* topk_idx;           // [T, k]
  float* topk_w;           // [T, k]
  int* local_rank;         // [T, k] rank of the entry among same-expert entries of its CTA
  int* block_hist;         // [nblk, E] -> converted in place to per-block exclusive bases
  int* counts;             // [E]
  int* offsets;            // [E+1]
  int* ticket;             // [1], zero on entry, reset to zero by the last CTA
};

// (value desc, index asc) ordering for selection
MGB_DEVINL bool better(float va, int ia, float vb, int ib) { return va > vb || (va == vb && ia < ib); }

MGB_DEVINL void warp_argbest(float& v, int& i) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, v, o);
    const int oi = __shfl_xor_sync(0xffffffffu, i, o);
    if (better(ov, oi, v, i)) { v = ov; i = oi; }
  }
}
MGB_DEVINL float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
MGB_DEVINL float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void __launch_bounds__(kRouterThreads) router_topk_kernel(RouterArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  float* s_logit = reinterpret_cast<float*>(smem);                          // [TPB][E]
  int* s_exp = reinterpret_cast<int*>(s_logit + kRouterTPB * kMaxE);        // [TPB*k]
  __nv_bfloat16* s_x = reinterpret_cast<__nv_bfloat16*>(s_exp + kRouterTPB * kMaxK);  // [TPB][d]
  __shared__ bool s_last;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t0 = blockIdx.x * kRouterTPB;
  const int ntok = min(kRouterTPB, a.T - t0);
  const int E = a.E, d = a.d, k = a.k;

  // ---------------- phase 1: logits ----------------
  if (a.logits_in) {
    for (int i = threadIdx.x; i < ntok * E; i += blockDim.x)
      s_logit[(i / E) * kMaxE + (i % E)] = a.logits_in[(size_t)(t0 + i / E) * E + (i % E)];
  } else {
    // stage the CTA's token rows in smem (16 B vectors)
    const int vec_per_row = d / 8;
    for (int i = threadIdx.x; i < ntok * vec_per_row; i += blockDim.x) {
      const int r = i / vec_per_row, c = i - r * vec_per_row;
      reinterpret_cast<uint4*>(s_x)[r * vec_per_row + c] =
          ld_nc_v4(reinterpret_cast<const uint4*>(a.x + (size_t)(t0 + r) * d) + c);
    }
    __syncthreads();
    for (int e = warp; e < E; e += kRouterThreads / 32) {
      float acc[kRouterTPB];
#pragma unroll
      for (int t = 0; t < kRouterTPB; ++t) acc[t] = 0.f;
      const uint4* wrow = reinterpret_cast<const uint4*>(a.wg + (size_t)e * d);
      for (int c = lane; c < vec_per_row; c += 32) {
        const uint4 w = __ldg(wrow + c);
        const float w0 = bf16lo(w.x), w1 = bf16hi(w.x), w2 = bf16lo(w.y), w3 = bf16hi(w.y);
        const float w4 = bf16lo(w.z), w5 = bf16hi(w.z), w6 = bf16lo(w.w), w7 = bf16hi(w.w);
#pragma unroll
        for (int t = 0; t < kRouterTPB; ++t) {
          if (t < ntok) {
            const uint4 xv = reinterpret_cast<const uint4*>(s_x)[t * vec_per_row + c];
            float s = acc[t];
            s = fmaf(bf16lo(xv.x), w0, s); s = fmaf(bf16hi(xv.x), w1, s);
            s = fmaf(bf16lo(xv.y), w2, s); s = fmaf(bf16hi(xv.y), w3, s);
            s = fmaf(bf16lo(xv.z), w4, s); s = fmaf(bf16hi(xv.z), w5, s);
            s = fmaf(bf16lo(xv.w), w6, s); s = fmaf(bf16hi(xv.w), w7, s);
            acc[t] = s;
          }
        }
      }
#pragma unroll
      for (int t = 0; t < kRouterTPB; ++t) {
        const float s = warp_sum(acc[t]);
        if (lane == 0 && t < ntok) s_logit[t * kMaxE + e] = (a.mode == 0) ? bf16_round(s) : s;
      }
    }
  }
  __syncthreads();

  // ---------------- phase 2: softmax + top-k (one warp per token) ----------------
  if (warp < ntok) {
    const int t = t0 + warp;
    const float* lg = s_logit + warp * kMaxE;
    if (a.logits_out)
      for (int e = lane; e < E; e += 32) a.logits_out[(size_t)t * E + e] = lg[e];
    float m = -INFINITY;
    for (int e = lane; e < E; e += 32) m = fmaxf(m, lg[e]);
    m = warp_max(m);
    float s = 0.f;
    for (int e = lane; e < E; e += 32) s += expf(lg[e] - m);
    s = warp_sum(s);
    const float inv = 1.0f / s;

    // group restriction (mode 2): allowed[e] via a bitmask over groups
    uint32_t group_ok = 0xffffffffu;
    if (a.mode == 2) {
      const int gsz = E / a.n_group;
      float gbest = -INFINITY;
      int gi = 0x7fffffff;
      if (lane < a.n_group) {
        gbest = -INFINITY;
        for (int e = lane * gsz; e < (lane + 1) * gsz; ++e) gbest = fmaxf(gbest, lg[e]);
        gi = lane;
      }
      group_ok = 0;
      for (int r = 0; r < a.topk_group; ++r) {
        float v = (group_ok >> lane) & 1u ? -INFINITY : gbest;
        int i = (group_ok >> lane) & 1u ? 0x7fffffff : gi;
        if (lane >= a.n_group) { v = -INFINITY; i = 0x7fffffff; }
        warp_argbest(v, i);
        group_ok |= 1u << i;
      }
    }
    // k rounds of warp arg-best over the (allowed, unselected) logits
    uint32_t taken[kMaxE / 32] = {0, 0, 0, 0, 0, 0, 0, 0};
    float psel[kMaxK];
    int isel[kMaxK];
    const int gsz = (a.mode == 2) ? E / a.n_group : E;
    for (int r = 0; r < k; ++r) {
      float bv = -INFINITY;
      int bi = 0x7fffffff;
      for (int e = lane, w = 0; e < E; e += 32, ++w) {
        if ((taken[w] >> lane) & 1u) continue;
        if (a.mode == 2 && !((group_ok >> (e / gsz)) & 1u)) continue;
        if (better(lg[e], e, bv, bi)) { bv = lg[e]; bi = e; }
      }
      warp_argbest(bv, bi);
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
        s_exp[warp * k + r] = isel[r];
      }
    }
  }
  __syncthreads();

  // ---------------- phase 3: per-CTA histogram + stable local ranks ----------------
  const int nent = ntok * k;
  for (int i = threadIdx.x; i < nent; i += blockDim.x) {
    const int e = s_exp[i];
    int r = 0;
    for (int j = 0; j < i; ++j) r += (s_exp[j] == e);
    a.local_rank[(size_t)t0 * k + i] = r;
  }
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    int c = 0;
    for (int j = 0; j < nent; ++j) c += (s_exp[j] == e);
    a.block_hist[(size_t)blockIdx.x * E + e] = c;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = (atomicAdd(a.ticket, 1) == (int)gridDim.x - 1);
  __syncthreads();
  if (!s_last) return;

  // ---------------- last CTA: per-block bases, counts, offsets ----------------
  __threadfence();
  int* s_cnt = reinterpret_cast<int*>(smem);  // reuse
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    int run = 0;
    for (int b = 0; b < (int)gridDim.x; ++b) {
      int* p = a.block_hist + (size_t)b * E + e;
      const int c = __ldcg(p);
      *p = run;
      run += c;
    }
    a.counts[e] = run;
    s_cnt[e] = run;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int run = 0;
    for (int e = 0; e < E; ++e) {
      a.offsets[e] = run;
      run += s_cnt[e];
    }
    a.offsets[E] = run;
    *a.ticket = 0;
  }
}

// One warp per (token, slot) entry: compute the permuted row and copy x[t] there (16 B vectors).
__global__ void permute_kernel(const __nv_bfloat16* __restrict__ x, const int* __restrict__ topk_idx,
                               const int* __restrict__ local_rank, const int* __restrict__ block_base,
                               const int* __restrict__ offsets, int T, int d, int k, int E, int tpb,
                               __nv_bfloat16* __restrict__ x_perm, int* __restrict__ src_token,
                               int* __restrict__ dst_pos) {
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (gw >= T * k) return;
  const int t = gw / k;
  const int e = topk_idx[gw];
  const int pos = offsets[e] + block_base[(size_t)(t / tpb) * E + e] + local_rank[gw];
  if (lane == 0) {
    dst_pos[gw] = pos;
    src_token[pos] = t;
  }
  const uint4* src = reinterpret_cast<const uint4*>(x + (size_t)t * d);
  uint4* dst = reinterpret_cast<uint4*>(x_perm + (size_t)pos * d);
  for (int c = lane; c < d / 8; c += 32) dst[c] = ld_nc_v4(src + c);
}

// out[t] = bf16( sum_j w[t,j] * y[dst[t,j]] ) (fp32, j ascending), then optional
//          moe = bf16(moe + shared[t]), then optional out = bf16(residual[t] + moe).
// One CTA per token, 8 dims (16 B) per thread per iteration.
__global__ void combine_kernel(const __nv_bfloat16* __restrict__ y_perm, const int* __restrict__ dst_pos,
                               const float* __restrict__ topk_w, const __nv_bfloat16* __restrict__ shared_out,
                               const __nv_bfloat16* residual, int T, int d, int k,
                               __nv_bfloat16* out) {  // out may alias residual (in-place residual add)
  const int t = blockIdx.x;
  __shared__ int s_pos[kMaxK];
  __shared__ float s_w[kMaxK];
  if (threadIdx.x < k) {
    s_pos[threadIdx.x] = dst_pos[(size_t)t * k + threadIdx.x];
    s_w[threadIdx.x] = topk_w[(size_t)t * k + threadIdx.x];
  }
  __syncthreads();
  for (int c = threadIdx.x; c < d / 8; c += blockDim.x) {
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int j = 0; j < k; ++j) {
      const uint4 v = ld_nc_v4(reinterpret_cast<const uint4*>(y_perm + (size_t)s_pos[j] * d) + c);
      const float w = s_w[j];
      acc[0] += w * bf16lo(v.x); acc[1] += w * bf16hi(v.x);
      acc[2] += w * bf16lo(v.y); acc[3] += w * bf16hi(v.y);
      acc[4] += w * bf16lo(v.z); acc[5] += w * bf16hi(v.z);
      acc[6] += w * bf16lo(v.w); acc[7] += w * bf16hi(v.w);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = bf16_round(acc[i]);
    if (shared_out) {
      const uint4 s = ld_nc_v4(reinterpret_cast<const uint4*>(shared_out + (size_t)t * d) + c);
      acc[0] = bf16_round(acc[0] + bf16lo(s.x)); acc[1] = bf16_round(acc[1] + bf16hi(s.x));
      acc[2] = bf16_round(acc[2] + bf16lo(s.y)); acc[3] = bf16_round(acc[3] + bf16hi(s.y));
      acc[4] = bf16_round(acc[4] + bf16lo(s.z)); acc[5] = bf16_round(acc[5] + bf16hi(s.z));
      acc[6] = bf16_round(acc[6] + bf16lo(s.w)); acc[7] = bf16_round(acc[7] + bf16hi(s.w));
    }
    if (residual) {
      const uint4 r = reinterpret_cast<const uint4*>(residual + (size_t)t * d)[c];
      acc[0] += bf16lo(r.x); acc[1] += bf16hi(r.x); acc[2] += bf16lo(r.y); acc[3] += bf16hi(r.y);
      acc[4] += bf16lo(r.z); acc[5] += bf16hi(r.z); acc[6] += bf16lo(r.w); acc[7] += bf16hi(r.w);
    }
    uint4 o;
    o.x = pack_bf16x2(acc[0], acc[1]); o.y = pack_bf16x2(acc[2], acc[3]);
    o.z = pack_bf16x2(acc[4], acc[5]); o.w = pack_bf16x2(acc[6], acc[7]);
    reinterpret_cast<uint4*>(out + (size_t)t * d)[c] = o;
  }
}

}  // namespace mgb

extern "C" {

// Number of router CTAs (= rows of the block_hist workspace) for T tokens.
int mgb_router_num_blocks(int T) { return (T + mgb::kRouterTPB - 1) / mgb::kRouterTPB; }
int mgb_router_tokens_per_block(void) { return mgb::kRouterTPB; }

// Fused router: gate GEMV (or given logits) -> softmax -> pinned-order top-k -> weights, plus
// per-expert counts/offsets and the per-CTA data the stable permutation needs.
int mgb_router_topk(const void* x, const void* w_gate, const float* logits_in, int T, int d, int E, int k,
                    int mode, float scaling, int n_group, int topk_group, float* logits_out, int* topk_idx,
                    float* topk_w, int* local_rank, int* block_hist, int* counts, int* offsets, int* ticket,
                    void* stream) {
  if (T < 1 || E < 1 || E > mgb::kMaxE || k < 1 || k > mgb::kMaxK || k > E || mode < 0 || mode > 2)
    return MGB_EINVAL;
  if (!logits_in && (d % 8 || d < 8)) return MGB_EINVAL;
  if (mode == 2 && (n_group < 1 || n_group > 32 || E % n_group || topk_group < 1 || topk_group > n_group ||
                    topk_group * (E / n_group) < k))
    return MGB_EINVAL;
  mgb::RouterArgs a{reinterpret_cast<const __nv_bfloat16*>(x), reinterpret_cast<const __nv_bfloat16*>(w_gate),
                    logits_in, T, d, E, k, mode, scaling, n_group, topk_group, logits_out, topk_idx, topk_w,
                    local_rank, block_hist, counts, offsets, ticket};
  const int nblk = mgb_router_num_blocks(T);
  const size_t smem = sizeof(float) * mgb::kRouterTPB * mgb::kMaxE + sizeof(int) * mgb::kRouterTPB * mgb::kMaxK +
                      (logits_in ? 0 : (size_t)mgb::kRouterTPB * d * 2);
  if (smem > 48 * 1024) {
    if (cudaFuncSetAttribute(mgb::router_topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
      return MGB_ECUDA;
  }
  mgb::router_topk_kernel<<<nblk, mgb::kRouterThreads, smem, reinterpret_cast<cudaStream_t>(stream)>>>(a);
  return cudaGetLastError() == cudaSuccess ? MGB_OK : MGB_ECUDA;
}

// Stable expert-major permutation: x_perm[pos] = x[t] for every (t, j), pos = offsets[e] +
// block_base[t / tpb][e] + local_rank[t, j]; also src_token[pos] = t and dst_pos[t, j] = pos.
int mgb_permute(const void* x, const int* topk_idx, const int* local_rank, const int* block_base,
                const int* offsets, int T, int d, int k, int E, void* x_perm, int* src_token, int* dst_pos,
                void* stream) {
  if (T < 1 || d % 8 || k < 1 || k > mgb::kMaxK) return MGB_EINVAL;
  const int warps = T * k;
  const int threads = 256;
  const int blocks = (warps * 32 + threads - 1) / threads;
  mgb::permute_kernel<<<blocks, threads, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const __nv_bfloat16*>(x), topk_idx, local_rank, block_base, offsets, T, d, k, E,
      mgb::kRouterTPB, reinterpret_cast<__nv_bfloat16*>(x_perm), src_token, dst_pos);
  return cudaGetLastError() == cudaSuccess ? MGB_OK : MGB_ECUDA;
}

// Weighted un-permute + combine (fp32, j ascending, one bf16 rounding), optional shared-expert
// add and residual add (HF grouped_mm semantics, integrations/moe.py:417-429).
int mgb_unpermute_combine(const void* y_perm, const int* dst_pos, const float* topk_w, const void* shared_out,
                          const void* residual, int T, int d, int k, void* out, void* stream) {
  if (T < 1 || d % 8 || k < 1 || k > mgb::kMaxK) return MGB_EINVAL;
  const int threads = (d / 8) >= 256 ? 256 : ((d / 8 + 31) / 32) * 32;
  mgb::combine_kernel<<<T, threads, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const __nv_bfloat16*>(y_perm), dst_pos, topk_w,
      reinterpret_cast<const __nv_bfloat16*>(shared_out), reinterpret_cast<const __nv_bfloat16*>(residual), T, d,
      k, reinterpret_cast<__nv_bfloat16*>(out));
  return cudaGetLastError() == cudaSuccess ? MGB_OK : MGB_ECUDA;
}

}  // extern "C"
