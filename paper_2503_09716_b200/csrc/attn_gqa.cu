// Paged GQA decode attention (Mixtral) on sm_100a — the ATTN_MECH_GPU job of the module-based
// batching schedule (reference: pkg/src/moe_planner/offload_dag.py:393-402; cost model
// hw_profile.py:269-270,285-287).  Semantics: HF transformers 5.5.0 eager_attention_forward
// (modeling_mixtral.py:269-291): softmax(q k^T / sqrt(hd)) v with key/value head i // G for query
// head i; this kernel keeps scores and the softmax in fp32 (online softmax), so it matches HF's
// bf16-rounded scores within tolerance, not bit-exactly.
//
// KV layout (owned by this framework, chosen for the decode access pattern): pages of
// kPage = 64 tokens; per (page, kv-head) one contiguous 16 KB block for K and one for V:
//   K: [page][kvh][hd/8 chunks][64 tokens][8]  (chunk-major -> lane = token reads are coalesced)
//   V: [page][kvh][64 tokens][hd]              (row-major   -> lane = dim-pair reads are coalesced)
// Each CTA owns one (sequence, kv-head) and streams its pages through shared memory with
// double-buffered cp.async.bulk copies (TMA bulk engine), so the kernel is HBM-bound.
#include "common.cuh"

namespace mgb {

constexpr int kPage = 64;
constexpr int kAttnThreads = 128;

template <int HD, int G>
struct AttnSmem {
  static constexpr int kTileElems = HD * kPage;                 // per K (or V) page-head block
  static constexpr int kTileBytes = kTileElems * 2;
  static constexpr int kGP = (G + 3) & ~3;                      // padded G for vector reads
  static constexpr size_t kBytes = 2 * 2 * (size_t)kTileBytes   // {K,V} x 2 stages
                                   + sizeof(float) * G * HD       // q
                                   + sizeof(float) * 2 * G * kPage  // partial scores (2 halves)
                                   + sizeof(float) * kPage * kGP    // p
                                   + sizeof(float) * 4 * G          // m, l, alpha, pad
                                   + 64;                            // mbarriers
};

template <int HD, int G>
__global__ void __launch_bounds__(kAttnThreads)
decode_attn_gqa_kernel(const __nv_bfloat16* __restrict__ q,       // [B, Hkv*G, HD]
                       const __nv_bfloat16* __restrict__ k_cache,  // pages
                       const __nv_bfloat16* __restrict__ v_cache,
                       const int* __restrict__ block_table, int max_pages,
                       const int* __restrict__ seq_lens, int Hkv, float scale_log2,
                       __nv_bfloat16* __restrict__ out) {          // [B, Hkv*G*HD]
  using S = AttnSmem<HD, G>;
  constexpr int kGP = S::kGP;
  constexpr int NCH = HD / 8;            // 16 B chunks per head row
  constexpr int NPAIR = HD / 2;          // dim pairs
  constexpr int TGROUPS = kAttnThreads / NPAIR;
  constexpr int TPG = kPage / TGROUPS;   // tokens per PV group
  static_assert(kAttnThreads % NPAIR == 0 && kPage % TGROUPS == 0, "shape");

  extern __shared__ __align__(128) uint8_t smem[];
  __nv_bfloat16* kv_s = reinterpret_cast<__nv_bfloat16*>(smem);   // [stage][K|V][tile]
  float* q_s = reinterpret_cast<float*>(smem + 4 * S::kTileBytes);  // [G][HD]
  float* sp_s = q_s + G * HD;                                       // [2][G][kPage]
  float* p_s = sp_s + 2 * G * kPage;                                // [kPage][kGP]
  float* m_s = p_s + kPage * kGP;                                   // [G]
  float* l_s = m_s + G;
  float* a_s = l_s + G;
  uint64_t* bar = reinterpret_cast<uint64_t*>(
      (reinterpret_cast<uintptr_t>(a_s + 2 * G) + 15) & ~uintptr_t(15));  // [2]

  const int b = blockIdx.x / Hkv;
  const int h = blockIdx.x - b * Hkv;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int len = seq_lens[b];
  const int npages = (len + kPage - 1) / kPage;
  const int* bt = block_table + (size_t)b * max_pages;

  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  for (int i = tid; i < G * HD; i += kAttnThreads)
    q_s[i] = __bfloat162float(q[((size_t)b * Hkv * G + (size_t)h * G) * HD + i]) * scale_log2;
  if (tid < G) {
    m_s[tid] = -INFINITY;
    l_s[tid] = 0.f;
  }
  __syncthreads();

  const uint64_t pol = policy_evict_first();
  auto issue = [&](int i) {
    const int stage = i & 1;
    const size_t blk = ((size_t)bt[i] * Hkv + h) * S::kTileElems;
    mbar_arrive_expect_tx(&bar[stage], 2 * S::kTileBytes);
    bulk_load(kv_s + (size_t)stage * 2 * S::kTileElems, k_cache + blk, S::kTileBytes, &bar[stage], pol);
    bulk_load(kv_s + (size_t)stage * 2 * S::kTileElems + S::kTileElems, v_cache + blk, S::kTileBytes, &bar[stage],
              pol);
  };
  if (tid == 0 && npages > 0) issue(0);

  float o[G][2];
#pragma unroll
  for (int g = 0; g < G; ++g) o[g][0] = o[g][1] = 0.f;

  for (int i = 0; i < npages; ++i) {
    if (tid == 0 && i + 1 < npages) issue(i + 1);
    mbar_wait(&bar[i & 1], (i >> 1) & 1);
    const __nv_bfloat16* k_t = kv_s + (size_t)(i & 1) * 2 * S::kTileElems;
    const __nv_bfloat16* v_t = k_t + S::kTileElems;
    const int n = min(kPage, len - i * kPage);

    // ---- scores: thread = (token, half of the head dims) ----
    {
      const int tok = tid & (kPage - 1);
      const int half = tid / kPage;  // 0 or 1
      float s[G];
#pragma unroll
      for (int g = 0; g < G; ++g) s[g] = 0.f;
#pragma unroll
      for (int cc = 0; cc < NCH / 2; ++cc) {
        const int c = half * (NCH / 2) + cc;
        const uint4 kv = *reinterpret_cast<const uint4*>(k_t + ((size_t)c * kPage + tok) * 8);
        const float k0 = bf16lo(kv.x), k1 = bf16hi(kv.x), k2 = bf16lo(kv.y), k3 = bf16hi(kv.y);
        const float k4 = bf16lo(kv.z), k5 = bf16hi(kv.z), k6 = bf16lo(kv.w), k7 = bf16hi(kv.w);
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const float4 qa = *reinterpret_cast<const float4*>(q_s + g * HD + c * 8);
          const float4 qb = *reinterpret_cast<const float4*>(q_s + g * HD + c * 8 + 4);
          float acc = s[g];
          acc = fmaf(qa.x, k0, acc); acc = fmaf(qa.y, k1, acc); acc = fmaf(qa.z, k2, acc); acc = fmaf(qa.w, k3, acc);
          acc = fmaf(qb.x, k4, acc); acc = fmaf(qb.y, k5, acc); acc = fmaf(qb.z, k6, acc); acc = fmaf(qb.w, k7, acc);
          s[g] = acc;
        }
      }
#pragma unroll
      for (int g = 0; g < G; ++g) sp_s[(half * G + g) * kPage + tok] = s[g];
    }
    __syncthreads();

    // ---- online softmax: one warp per head ----
    for (int g = warp; g < G; g += kAttnThreads / 32) {
      const int t0 = lane, t1 = lane + 32;
      const float s0 = t0 < n ? sp_s[g * kPage + t0] + sp_s[(G + g) * kPage + t0] : -INFINITY;
      const float s1 = t1 < n ? sp_s[g * kPage + t1] + sp_s[(G + g) * kPage + t1] : -INFINITY;
      float mt = fmaxf(s0, s1);
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) mt = fmaxf(mt, __shfl_xor_sync(0xffffffffu, mt, off));
      const float m_old = m_s[g];
      const float m_new = fmaxf(m_old, mt);
      const float alpha = exp2f(m_old - m_new);
      const float p0 = exp2f(s0 - m_new), p1 = exp2f(s1 - m_new);
      float ps = p0 + p1;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) ps += __shfl_xor_sync(0xffffffffu, ps, off);
      p_s[t0 * kGP + g] = p0;
      p_s[t1 * kGP + g] = p1;
      __syncwarp();
      if (lane == 0) {
        m_s[g] = m_new;
        l_s[g] = l_s[g] * alpha + ps;
        a_s[g] = alpha;
      }
    }
    __syncthreads();

    // ---- P V: thread = (dim pair, token group) ----
    {
      const int dp = tid % NPAIR;
      const int tg = tid / NPAIR;
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const float al = a_s[g];
        o[g][0] *= al;
        o[g][1] *= al;
      }
      const int tb = tg * TPG;
      const int te = min(tb + TPG, n);
      for (int t = tb; t < te; ++t) {
        const uint32_t v2 = *reinterpret_cast<const uint32_t*>(v_t + (size_t)t * HD + 2 * dp);
        const float v0 = bf16lo(v2), v1 = bf16hi(v2);
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const float p = p_s[t * kGP + g];
          o[g][0] = fmaf(p, v0, o[g][0]);
          o[g][1] = fmaf(p, v1, o[g][1]);
        }
      }
    }
    __syncthreads();  // stage (i & 1) fully consumed before it is refilled at iteration i + 1
  }

  // ---- reduce the token groups, normalise, store ----
  float* red = reinterpret_cast<float*>(smem);  // reuse the KV stages: [TGROUPS][G][HD]
  {
    const int dp = tid % NPAIR;
    const int tg = tid / NPAIR;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      red[((size_t)tg * G + g) * HD + 2 * dp] = o[g][0];
      red[((size_t)tg * G + g) * HD + 2 * dp + 1] = o[g][1];
    }
  }
  __syncthreads();
  for (int i = tid; i < G * HD; i += kAttnThreads) {
    const int g = i / HD;
    float acc = 0.f;
#pragma unroll
    for (int tg = 0; tg < TGROUPS; ++tg) acc += red[(size_t)tg * G * HD + i];
    const float l = l_s[g];
    out[((size_t)b * Hkv * G + (size_t)h * G) * HD + i] = __float2bfloat16_rn(l > 0.f ? acc / l : 0.f);
  }
}

template <int HD, int G>
int launch_gqa(const void* q, const void* kc, const void* vc, const int* bt, int max_pages, const int* lens, int B,
               int Hkv, float scale, void* out, cudaStream_t st) {
  using S = AttnSmem<HD, G>;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(decode_attn_gqa_kernel<HD, G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)S::kBytes) != cudaSuccess)
      return MGB_ECUDA;
    attr = true;
  }
  decode_attn_gqa_kernel<HD, G><<<B * Hkv, kAttnThreads, S::kBytes, st>>>(
      reinterpret_cast<const __nv_bfloat16*>(q), reinterpret_cast<const __nv_bfloat16*>(kc),
      reinterpret_cast<const __nv_bfloat16*>(vc), bt, max_pages, lens, Hkv, scale * 1.4426950408889634f,
      reinterpret_cast<__nv_bfloat16*>(out));
  return cudaGetLastError() == cudaSuccess ? MGB_OK : MGB_ECUDA;
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
