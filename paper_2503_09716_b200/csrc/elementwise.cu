// Small HBM-bound kernels around the hot path: fused residual-add + RMSNorm, RoPE + paged KV
// append, embedding gather, greedy argmax + decode-step bookkeeping, and the counter-based weight
// generator.  Numerics follow HF transformers 5.5.0 (MixtralRMSNorm, apply_rotary_pos_emb),
// including every intermediate bf16 rounding, so these match the CPU oracle bit-exactly except
// for the RMS reduction order.
#include <algorithm>

#include "common.cuh"

namespace mgb {

constexpr int kPageTok = 64;  // must equal attn_gqa.cu kPage

MGB_DEVINL float block_sum(float v, float* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = v;
  __syncthreads();
  float t = 0.f;
  const int nw = blockDim.x >> 5;
  for (int i = 0; i < nw; ++i) t += red[i];
  __syncthreads();
  return t;
}

// x' = delta ? bf16(x + delta) : x; x_out = x'; y = bf16(w * bf16(x' * rsqrt(mean(x'^2) + eps)))
// One CTA per row; the row stays in registers between the reduction and the normalisation.
constexpr int kNormThreads = 256;
constexpr int kNormVec = 4;  // d <= 8192
__global__ void __launch_bounds__(kNormThreads)
add_rmsnorm_kernel(const __nv_bfloat16* x, const __nv_bfloat16* __restrict__ delta,
                   const __nv_bfloat16* __restrict__ w, float eps, int d, __nv_bfloat16* x_out,
                   __nv_bfloat16* __restrict__ y) {
  mgb::pdl_enter();
  __shared__ float red[32];
  const size_t row = blockIdx.x;
  const int nvec = d / 8;
  const uint4* xr = reinterpret_cast<const uint4*>(x + row * d);
  const uint4* dr = delta ? reinterpret_cast<const uint4*>(delta + row * d) : nullptr;
  uint4 v[kNormVec], dv[kNormVec];
#pragma unroll
  for (int u = 0; u < kNormVec; ++u) {
    const int c = threadIdx.x + u * kNormThreads;
    if (c < nvec) {
      v[u] = xr[c];
      if (dr) dv[u] = dr[c];
    }
  }
  float ss = 0.f;
#pragma unroll
  for (int u = 0; u < kNormVec; ++u) {
    const int c = threadIdx.x + u * kNormThreads;
    if (c >= nvec) continue;
    if (dr) {
      v[u].x = pack_bf16x2(bf16lo(v[u].x) + bf16lo(dv[u].x), bf16hi(v[u].x) + bf16hi(dv[u].x));
      v[u].y = pack_bf16x2(bf16lo(v[u].y) + bf16lo(dv[u].y), bf16hi(v[u].y) + bf16hi(dv[u].y));
      v[u].z = pack_bf16x2(bf16lo(v[u].z) + bf16lo(dv[u].z), bf16hi(v[u].z) + bf16hi(dv[u].z));
      v[u].w = pack_bf16x2(bf16lo(v[u].w) + bf16lo(dv[u].w), bf16hi(v[u].w) + bf16hi(dv[u].w));
    }
    if (x_out) reinterpret_cast<uint4*>(x_out + row * d)[c] = v[u];
    const float f[8] = {bf16lo(v[u].x), bf16hi(v[u].x), bf16lo(v[u].y), bf16hi(v[u].y),
                        bf16lo(v[u].z), bf16hi(v[u].z), bf16lo(v[u].w), bf16hi(v[u].w)};
#pragma unroll
    for (int i = 0; i < 8; ++i) ss = fmaf(f[i], f[i], ss);
  }
  const float inv = 1.0f / sqrtf(block_sum(ss, red) / (float)d + eps);
  const uint4* wr = reinterpret_cast<const uint4*>(w);
#pragma unroll
  for (int u = 0; u < kNormVec; ++u) {
    const int c = threadIdx.x + u * kNormThreads;
    if (c >= nvec) continue;
    const uint4 wv = wr[c];
    uint4 o;
    o.x = pack_bf16x2(bf16lo(wv.x) * bf16_round(bf16lo(v[u].x) * inv), bf16hi(wv.x) * bf16_round(bf16hi(v[u].x) * inv));
    o.y = pack_bf16x2(bf16lo(wv.y) * bf16_round(bf16lo(v[u].y) * inv), bf16hi(wv.y) * bf16_round(bf16hi(v[u].y) * inv));
    o.z = pack_bf16x2(bf16lo(wv.z) * bf16_round(bf16lo(v[u].z) * inv), bf16hi(wv.z) * bf16_round(bf16hi(v[u].z) * inv));
    o.w = pack_bf16x2(bf16lo(wv.w) * bf16_round(bf16lo(v[u].w) * inv), bf16hi(wv.w) * bf16_round(bf16hi(v[u].w) * inv));
    reinterpret_cast<uint4*>(y + row * d)[c] = o;
  }
}

// Warp-per-token add + RMSNorm for rows of <= 2048 dims (DeepSeek-V2-Lite's 6058-token decode batch):
// 8 tokens per CTA, the row in registers, a warp-shuffle sum instead of the block reduction, every
// load of the row (x, delta, weight) in flight together -- the CTA-per-token kernel is a chain of two
// block barriers per token over five waves of CTAs.  Same arithmetic per element.
constexpr int kNormWarpTok = 8;
template <int V>  // 16-byte vectors per lane (d = 256 * V)
__global__ void __launch_bounds__(kNormWarpTok * 32)
add_rmsnorm_warp_kernel(const __nv_bfloat16* x, const __nv_bfloat16* __restrict__ delta,
                        const __nv_bfloat16* __restrict__ w, float eps, int T, int d, __nv_bfloat16* x_out,
                        __nv_bfloat16* __restrict__ y) {
  mgb::pdl_enter();
  const int lane = threadIdx.x & 31;
  const size_t row = (size_t)blockIdx.x * kNormWarpTok + (threadIdx.x >> 5);
  if (row >= (size_t)T) return;
  const int nvec = d / 8;
  const uint4* xr = reinterpret_cast<const uint4*>(x + row * d);
  const uint4* dr = delta ? reinterpret_cast<const uint4*>(delta + row * d) : nullptr;
  const uint4* wr = reinterpret_cast<const uint4*>(w);
  uint4 v[V], dv[V], wv[V];
#pragma unroll
  for (int u = 0; u < V; ++u) {
    const int c = lane + 32 * u;
    if (c < nvec) {
      v[u] = xr[c];
      if (dr) dv[u] = dr[c];
      wv[u] = wr[c];
    }
  }
  float ss = 0.f;
#pragma unroll
  for (int u = 0; u < V; ++u) {
    const int c = lane + 32 * u;
    if (c >= nvec) continue;
    if (dr) {
      v[u].x = pack_bf16x2(bf16lo(v[u].x) + bf16lo(dv[u].x), bf16hi(v[u].x) + bf16hi(dv[u].x));
      v[u].y = pack_bf16x2(bf16lo(v[u].y) + bf16lo(dv[u].y), bf16hi(v[u].y) + bf16hi(dv[u].y));
      v[u].z = pack_bf16x2(bf16lo(v[u].z) + bf16lo(dv[u].z), bf16hi(v[u].z) + bf16hi(dv[u].z));
      v[u].w = pack_bf16x2(bf16lo(v[u].w) + bf16lo(dv[u].w), bf16hi(v[u].w) + bf16hi(dv[u].w));
    }
    if (x_out) reinterpret_cast<uint4*>(x_out + row * d)[c] = v[u];
    const float f[8] = {bf16lo(v[u].x), bf16hi(v[u].x), bf16lo(v[u].y), bf16hi(v[u].y),
                        bf16lo(v[u].z), bf16hi(v[u].z), bf16lo(v[u].w), bf16hi(v[u].w)};
#pragma unroll
    for (int i = 0; i < 8; ++i) ss = fmaf(f[i], f[i], ss);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  const float inv = 1.0f / sqrtf(ss / (float)d + eps);
#pragma unroll
  for (int u = 0; u < V; ++u) {
    const int c = lane + 32 * u;
    if (c >= nvec) continue;
    uint4 o;
    o.x = pack_bf16x2(bf16lo(wv[u].x) * bf16_round(bf16lo(v[u].x) * inv), bf16hi(wv[u].x) * bf16_round(bf16hi(v[u].x) * inv));
    o.y = pack_bf16x2(bf16lo(wv[u].y) * bf16_round(bf16lo(v[u].y) * inv), bf16hi(wv[u].y) * bf16_round(bf16hi(v[u].y) * inv));
    o.z = pack_bf16x2(bf16lo(wv[u].z) * bf16_round(bf16lo(v[u].z) * inv), bf16hi(wv[u].z) * bf16_round(bf16hi(v[u].z) * inv));
    o.w = pack_bf16x2(bf16lo(wv[u].w) * bf16_round(bf16lo(v[u].w) * inv), bf16hi(wv[u].w) * bf16_round(bf16hi(v[u].w) * inv));
    reinterpret_cast<uint4*>(y + row * d)[c] = o;
  }
}

// RoPE of one 16-byte chunk c (8 dims) of a head row: HF rotate_half with bf16 products and sum.
MGB_DEVINL uint4 rope_chunk(const uint4* src, int c, int nch, const float* cos_row, const float* sin_row) {
  const uint4 xv = src[c];
  const int half_ch = nch >> 1;
  const bool lo = c < half_ch;
  const uint4 pv = src[lo ? c + half_ch : c - half_ch];
  const float x[8] = {bf16lo(xv.x), bf16hi(xv.x), bf16lo(xv.y), bf16hi(xv.y),
                      bf16lo(xv.z), bf16hi(xv.z), bf16lo(xv.w), bf16hi(xv.w)};
  const float pr[8] = {bf16lo(pv.x), bf16hi(pv.x), bf16lo(pv.y), bf16hi(pv.y),
                       bf16lo(pv.z), bf16hi(pv.z), bf16lo(pv.w), bf16hi(pv.w)};
  const int fi0 = (lo ? c : c - half_ch) * 8;
  const float4 c0 = *reinterpret_cast<const float4*>(cos_row + fi0), c1 = *reinterpret_cast<const float4*>(cos_row + fi0 + 4);
  const float4 s0 = *reinterpret_cast<const float4*>(sin_row + fi0), s1 = *reinterpret_cast<const float4*>(sin_row + fi0 + 4);
  const float cs[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
  const float sn[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
  float r[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float rh = lo ? -pr[i] : pr[i];  // rotate_half
    r[i] = bf16_round(x[i] * cs[i]) + bf16_round(rh * sn[i]);
  }
  uint4 ov;
  ov.x = pack_bf16x2(r[0], r[1]); ov.y = pack_bf16x2(r[2], r[3]);
  ov.z = pack_bf16x2(r[4], r[5]); ov.w = pack_bf16x2(r[6], r[7]);
  return ov;
}

// One CTA per token, one thread per (head, chunk pair (j, j + hd/16)) of its fused qkv row
// [Hq | Hkv | Hkv] x hd: rotate_half pairs exactly those two 16-byte chunks, so each thread loads its
// two chunks once (no partner re-loads) and issues all of its loads before any store (one memory round
// trip per token).  q heads are rotated into q_out; k heads rotated and written into the chunk-major K
// page; v heads copied into the V page.  Same rotation arithmetic as rope_chunk.
__global__ void rope_append_gqa_kernel(const __nv_bfloat16* __restrict__ qkv, int T, int seq0,
                                       const int* __restrict__ positions, const float* __restrict__ cos_t,
                                       const float* __restrict__ sin_t, int Hq, int Hkv, int hd,
                                       const int* __restrict__ block_table, int max_pages,
                                       __nv_bfloat16* __restrict__ k_cache, __nv_bfloat16* __restrict__ v_cache,
                                       __nv_bfloat16* __restrict__ q_out, int* __restrict__ seq_lens) {
  mgb::pdl_enter();
  const int t = blockIdx.x;
  const int nch = hd >> 3, half = nch >> 1, H = Hq + 2 * Hkv;
  const int seq = seq0 + t;
  const int i = threadIdx.x;
  if (i >= H * half) return;
  const int hh = i / half, j = i - hh * half;
  const uint4* src = reinterpret_cast<const uint4*>(qkv + (size_t)t * H * hd + hh * hd);
  const uint4 xl = src[j], xh = src[j + half];  // requested before the position / page lookups land
  const int pos = positions[seq];
  // a position past the planned context has no page (and no RoPE row): write nothing rather than
  // index the next sequence's block-table row (the host refuses such steps, Engine.run_step)
  if (pos < 0 || pos >= max_pages * kPageTok) return;
  const int page = hh >= Hq ? block_table[(size_t)seq * max_pages + pos / kPageTok] : 0;
  const int slot = pos % kPageTok;
  if (seq_lens && i == 0) seq_lens[seq] = pos + 1;  // cache length after the append
  uint4 ol = xl, oh = xh;
  if (hh < Hq + Hkv)
    rope_rot8(xl, xh, cos_t + (size_t)pos * (hd / 2) + j * 8, sin_t + (size_t)pos * (hd / 2) + j * 8, ol, oh);
  if (hh < Hq) {
    uint4* dst = reinterpret_cast<uint4*>(q_out + ((size_t)t * Hq + hh) * hd);
    dst[j] = ol;
    dst[j + half] = oh;
  } else {
    const bool is_k = hh < Hq + Hkv;
    const int kh = is_k ? hh - Hq : hh - Hq - Hkv;
    __nv_bfloat16* blk = (is_k ? k_cache : v_cache) + ((size_t)page * Hkv + kh) * hd * kPageTok;
    *reinterpret_cast<uint4*>(blk + ((size_t)j * kPageTok + slot) * 8) = ol;
    *reinterpret_cast<uint4*>(blk + ((size_t)(j + half) * kPageTok + slot) * 8) = oh;
  }
}

// Prefill variant: T = n_seq * P prompt tokens, token t of the batch is position t % P of sequence
// seq0 + t / P.  q heads are rotated into q_out [T, Hq, hd]; k heads rotated and v heads copied into
// the chunk-major KV pages AND into the contiguous k_out / v_out [T, Hkv, hd] rows the causal
// prefill attention reads.  Same rotation arithmetic as rope_append_gqa_kernel.
__global__ void rope_append_gqa_prefill_kernel(const __nv_bfloat16* __restrict__ qkv, int T, int seq0, int P,
                                               const float* __restrict__ cos_t, const float* __restrict__ sin_t,
                                               int Hq, int Hkv, int hd, const int* __restrict__ block_table,
                                               int max_pages, __nv_bfloat16* __restrict__ k_cache,
                                               __nv_bfloat16* __restrict__ v_cache, __nv_bfloat16* __restrict__ q_out,
                                               __nv_bfloat16* __restrict__ k_out, __nv_bfloat16* __restrict__ v_out) {
  mgb::pdl_enter();
  const int t = blockIdx.x;
  const int nch = hd >> 3, H = Hq + 2 * Hkv;
  const int seq = seq0 + t / P, pos = t % P;
  const int page = block_table[(size_t)seq * max_pages + pos / kPageTok];
  const int slot = pos % kPageTok;
  const float* cs = cos_t + (size_t)pos * (hd / 2);
  const float* sn = sin_t + (size_t)pos * (hd / 2);
  const __nv_bfloat16* row = qkv + (size_t)t * H * hd;
  for (int i = threadIdx.x; i < H * nch; i += blockDim.x) {
    const int hh = i / nch, c = i - hh * nch;
    const uint4* src = reinterpret_cast<const uint4*>(row + hh * hd);
    const uint4 ov = hh < Hq + Hkv ? rope_chunk(src, c, nch, cs, sn) : src[c];
    if (hh < Hq) {
      reinterpret_cast<uint4*>(q_out + ((size_t)t * Hq + hh) * hd)[c] = ov;
    } else {
      const bool is_k = hh < Hq + Hkv;
      const int kh = is_k ? hh - Hq : hh - Hq - Hkv;
      const size_t blk = ((size_t)page * Hkv + kh) * hd * kPageTok;
      *reinterpret_cast<uint4*>((is_k ? k_cache : v_cache) + blk + ((size_t)c * kPageTok + slot) * 8) = ov;
      reinterpret_cast<uint4*>((is_k ? k_out : v_out) + ((size_t)t * Hkv + kh) * hd)[c] = ov;
    }
  }
}

// h = bf16(bf16(silu(g)) * u) for gu = [g | u] rows (HF DeepseekV2MLP / MixtralExperts act-mul on the
// bf16 outputs of a cuBLAS gate|up GEMM).  8 features per thread, 16 B in/out.
__global__ void silu_mul_kernel(const __nv_bfloat16* __restrict__ gu, int T, int F, __nv_bfloat16* __restrict__ h) {
  mgb::pdl_enter();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;  // 16-byte chunk of the row
  if (c >= F / 8) return;
  for (int t = blockIdx.y; t < T; t += gridDim.y) {  // tokens on grid.y (32-bit index arithmetic)
    const uint4 g = reinterpret_cast<const uint4*>(gu + (size_t)t * 2 * F)[c];
    const uint4 u = reinterpret_cast<const uint4*>(gu + (size_t)t * 2 * F + F)[c];
    const float gf[8] = {bf16lo(g.x), bf16hi(g.x), bf16lo(g.y), bf16hi(g.y), bf16lo(g.z), bf16hi(g.z), bf16lo(g.w), bf16hi(g.w)};
    const float uf[8] = {bf16lo(u.x), bf16hi(u.x), bf16lo(u.y), bf16hi(u.y), bf16lo(u.z), bf16hi(u.z), bf16lo(u.w), bf16hi(u.w)};
    float r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = bf16_round(__fdividef(gf[j], 1.0f + __expf(-gf[j]))) * uf[j];
    uint4 o;
    o.x = pack_bf16x2(r[0], r[1]); o.y = pack_bf16x2(r[2], r[3]); o.z = pack_bf16x2(r[4], r[5]); o.w = pack_bf16x2(r[6], r[7]);
    reinterpret_cast<uint4*>(h + (size_t)t * F)[c] = o;
  }
}

__global__ void embed_kernel(const int* __restrict__ ids, const __nv_bfloat16* __restrict__ table, int d,
                             __nv_bfloat16* __restrict__ out) {
  mgb::pdl_enter();
  const size_t t = blockIdx.x;
  const uint4* src = reinterpret_cast<const uint4*>(table + (size_t)ids[t] * d);
  uint4* dst = reinterpret_cast<uint4*>(out + t * d);
  for (int c = threadIdx.x; c < d / 8; c += blockDim.x) dst[c] = src[c];
}

// Greedy argmax over a bf16 logits row (first maximal index wins, like torch.argmax).
__global__ void argmax_kernel(const __nv_bfloat16* __restrict__ logits, int V, int* __restrict__ out) {
  mgb::pdl_enter();
  const size_t row = blockIdx.x;
  const __nv_bfloat16* lr = logits + row * V;
  float bv = -INFINITY;
  int bi = 0x7fffffff;
  if ((V & 7) == 0) {  // 16 B vectors; all of a thread's loads issued before the compares
    const uint4* lv = reinterpret_cast<const uint4*>(lr);
    const int nv = V / 8;
    constexpr int U = 4;
    for (int c0 = threadIdx.x; c0 < nv; c0 += blockDim.x * U) {
      uint4 w[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (c0 + u * (int)blockDim.x < nv) w[u] = ld_nc_v4(lv + c0 + u * blockDim.x);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int c = c0 + u * blockDim.x;
        if (c >= nv) break;
        const float f[8] = {bf16lo(w[u].x), bf16hi(w[u].x), bf16lo(w[u].y), bf16hi(w[u].y),
                            bf16lo(w[u].z), bf16hi(w[u].z), bf16lo(w[u].w), bf16hi(w[u].w)};
#pragma unroll
        for (int i = 0; i < 8; ++i)
          if (f[i] > bv) { bv = f[i]; bi = c * 8 + i; }  // ascending index within a thread: first max kept
      }
    }
  } else {
    for (int i = threadIdx.x; i < V; i += blockDim.x) {
      const float v = __bfloat162float(lr[i]);
      if (v > bv || (v == bv && i < bi)) { bv = v; bi = i; }
    }
  }
  __shared__ float sv[32];
  __shared__ int si[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) { sv[w] = bv; si[w] = bi; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < (int)(blockDim.x >> 5); ++i)
      if (sv[i] > bv || (sv[i] == bv && si[i] < bi)) { bv = sv[i]; bi = si[i]; }
    out[row] = bi;
  }
}

// out_tokens[b * ld + *step] = next[b]; positions[b] += 1; then ++*step.
__global__ void decode_advance_kernel(const int* __restrict__ next, int B, long long* __restrict__ out_tokens,
                                      int ld, int* __restrict__ step, int* __restrict__ positions) {
  mgb::pdl_enter();
  const int s = *step;
  for (int b = threadIdx.x; b < B; b += blockDim.x) {
    if (out_tokens && s < ld) out_tokens[(size_t)b * ld + s] = next[b];
    positions[b] += 1;
  }
  __syncthreads();
  if (threadIdx.x == 0) *step = s + 1;
}

// Counter-based weight generator (mirrored bit-exactly by oracle/rng.py):
//   x = (seed * K1 + tensor_id) * K2 + i;  z = splitmix64_mix(x);
//   u = int(z >> 40) - 2^23  (uniform over [-2^23, 2^23));  value = bf16(float(u) * scale)
// with scale = fp32(std * sqrt(3) / 2^23): a uniform distribution with standard deviation `std`.
MGB_DEVINL uint64_t splitmix64_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__global__ void fill_uniform_kernel(__nv_bfloat16* __restrict__ out, size_t n, uint64_t seed, uint64_t tensor_id,
                                    float scale, float constant, int mode, uint64_t first) {
  mgb::pdl_enter();
  const uint64_t base = (seed * 0x9E3779B97F4A7C15ull + tensor_id) * 0xD1B54A32D192ED03ull;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    if (mode == 1) {
      out[i] = __float2bfloat16_rn(constant);
    } else {
      const uint64_t z = splitmix64_mix(base + first + i);  // element first + i of the tensor's stream
      const int u = (int)(z >> 40) - (1 << 23);
      out[i] = __float2bfloat16_rn(__fmul_rn((float)u, scale));
    }
  }
}

}  // namespace mgb

extern "C" {

int mgb_add_rmsnorm(const void* x, const void* delta, const void* weight, float eps, int T, int d, void* x_out,
                    void* y, void* stream) {
  if (T < 1 || d % 8 || d > 8 * mgb::kNormThreads * mgb::kNormVec) return MGB_EINVAL;
  if (T >= 1024 && d <= 2048) {  // large decode batches of narrow rows: warp per token
    const int blocks = (T + mgb::kNormWarpTok - 1) / mgb::kNormWarpTok;
    auto kern = d <= 1024 ? mgb::add_rmsnorm_warp_kernel<4> : mgb::add_rmsnorm_warp_kernel<8>;
    mgb_host::launch(kern, dim3(blocks), dim3(mgb::kNormWarpTok * 32), 0, reinterpret_cast<cudaStream_t>(stream), nullptr,
        reinterpret_cast<const __nv_bfloat16*>(x), reinterpret_cast<const __nv_bfloat16*>(delta),
        reinterpret_cast<const __nv_bfloat16*>(weight), eps, T, d, reinterpret_cast<__nv_bfloat16*>(x_out),
        reinterpret_cast<__nv_bfloat16*>(y));
    return mgb_host::launch_status();
  }
  mgb_host::launch(mgb::add_rmsnorm_kernel, dim3(T), dim3(mgb::kNormThreads), 0, reinterpret_cast<cudaStream_t>(stream), nullptr,
      reinterpret_cast<const __nv_bfloat16*>(x), reinterpret_cast<const __nv_bfloat16*>(delta),
      reinterpret_cast<const __nv_bfloat16*>(weight), eps, d, reinterpret_cast<__nv_bfloat16*>(x_out),
      reinterpret_cast<__nv_bfloat16*>(y));
  return mgb_host::launch_status();
}

namespace {
// 256 threads per token CTA (a few (head, chunk) items each): 8 CTAs per SM put a whole decode batch
// in one wave (Mixtral B=827: 0.44 vs 0.47 ms per forward with one item per thread)
int rope_threads(int H, int hd) { return std::min(256, (H * (hd / 8) + 31) / 32 * 32); }
int rope_pair_threads(int H, int hd) { return (H * (hd / 16) + 31) / 32 * 32; }  // one thread per chunk pair
}  // namespace

int mgb_rope_append_gqa(const void* qkv, int T, int seq0, const int* positions, const float* cos_t,
                        const float* sin_t, int Hq, int Hkv, int head_dim, const int* block_table, int max_pages,
                        void* k_cache, void* v_cache, void* q_out, int* seq_lens, void* stream) {
  if (T < 1 || head_dim % 16 || Hq % Hkv) return MGB_EINVAL;
  const int threads = rope_pair_threads(Hq + 2 * Hkv, head_dim);
  if (threads > 1024) return MGB_EINVAL;
  mgb_host::launch(mgb::rope_append_gqa_kernel, dim3(T), dim3(threads), 0, reinterpret_cast<cudaStream_t>(stream), nullptr,
      reinterpret_cast<const __nv_bfloat16*>(qkv), T, seq0, positions, cos_t, sin_t, Hq, Hkv, head_dim, block_table,
      max_pages, reinterpret_cast<__nv_bfloat16*>(k_cache), reinterpret_cast<__nv_bfloat16*>(v_cache),
      reinterpret_cast<__nv_bfloat16*>(q_out), seq_lens);
  return mgb_host::launch_status();
}

int mgb_rope_append_gqa_prefill(const void* qkv, int T, int seq0, int P, const float* cos_t, const float* sin_t,
                                int Hq, int Hkv, int head_dim, const int* block_table, int max_pages, void* k_cache,
                                void* v_cache, void* q_out, void* k_out, void* v_out, void* stream) {
  if (T < 1 || P < 1 || T % P || head_dim % 16 || Hq % Hkv) return MGB_EINVAL;
  const int threads = rope_threads(Hq + 2 * Hkv, head_dim);
  mgb_host::launch(mgb::rope_append_gqa_prefill_kernel, dim3(T), dim3(threads), 0, reinterpret_cast<cudaStream_t>(stream), nullptr,
      reinterpret_cast<const __nv_bfloat16*>(qkv), T, seq0, P, cos_t, sin_t, Hq, Hkv, head_dim, block_table, max_pages,
      reinterpret_cast<__nv_bfloat16*>(k_cache), reinterpret_cast<__nv_bfloat16*>(v_cache),
      reinterpret_cast<__nv_bfloat16*>(q_out), reinterpret_cast<__nv_bfloat16*>(k_out),
      reinterpret_cast<__nv_bfloat16*>(v_out));
  return mgb_host::launch_status();
}

int mgb_silu_mul(const void* gate_up, int T, int F, void* h, void* stream) {
  if (T < 1 || F % 8) return MGB_EINVAL;
  mgb_host::launch(mgb::silu_mul_kernel, dim3(dim3((F / 8 + 255) / 256, std::min(T, 65535))), dim3(256), 0, reinterpret_cast<cudaStream_t>(stream), nullptr,
      reinterpret_cast<const __nv_bfloat16*>(gate_up), T, F, reinterpret_cast<__nv_bfloat16*>(h));
  return mgb_host::launch_status();
}

int mgb_embed(const int* ids, const void* table, int T, int d, void* out, void* stream) {
  if (T < 1 || d % 8) return MGB_EINVAL;
  mgb_host::launch(mgb::embed_kernel, dim3(T), dim3(128), 0, reinterpret_cast<cudaStream_t>(stream), nullptr,
      ids, reinterpret_cast<const __nv_bfloat16*>(table), d, reinterpret_cast<__nv_bfloat16*>(out));
  return mgb_host::launch_status();
}

int mgb_argmax(const void* logits, int T, int V, int* out, void* stream) {
  if (T < 1 || V < 1) return MGB_EINVAL;
  mgb_host::launch(mgb::argmax_kernel, dim3(T), dim3(512), 0, reinterpret_cast<cudaStream_t>(stream), nullptr,
      reinterpret_cast<const __nv_bfloat16*>(logits), V, out);
  return mgb_host::launch_status();
}

int mgb_decode_advance(const int* next, int B, long long* out_tokens, int ld, int* step, int* positions,
                       void* stream) {
  if (B < 1) return MGB_EINVAL;
  mgb_host::launch(mgb::decode_advance_kernel, dim3(1), dim3(1024), 0, reinterpret_cast<cudaStream_t>(stream), nullptr,
      next, B, out_tokens, ld, step,
                                                                                     positions);
  return mgb_host::launch_status();
}

// mode 0: counter-based uniform with standard deviation `std`; mode 1: constant fill.
int mgb_fill_uniform_bf16(void* out, long long n, unsigned long long seed, unsigned long long tensor_id, float std,
                          float constant, int mode, void* stream) {
  if (n < 0) return MGB_EINVAL;
  if (n == 0) return MGB_OK;
  const float scale = (float)((double)std * 1.7320508075688772 / 8388608.0);
  const int threads = 256;
  long long blocks = (n + threads - 1) / threads;
  if (blocks > 148 * 64) blocks = 148 * 64;
  mgb_host::launch(mgb::fill_uniform_kernel, dim3((int)blocks), dim3(threads), 0, reinterpret_cast<cudaStream_t>(stream), nullptr,
      reinterpret_cast<__nv_bfloat16*>(out), (size_t)n, seed, tensor_id, scale, constant, mode, (uint64_t)0);
  return mgb_host::launch_status();
}

// Elements [first, first + n) of tensor `tensor_id`'s counter-based stream (the same values
// mgb_fill_uniform_bf16 writes at those indices of the whole tensor): a rank's expert shard is
// generated in place without materialising the other ranks' experts.
int mgb_fill_uniform_bf16_range(void* out, long long n, long long first, unsigned long long seed,
                                unsigned long long tensor_id, float std, void* stream) {
  if (n < 0 || first < 0) return MGB_EINVAL;
  if (n == 0) return MGB_OK;
  const float scale = (float)((double)std * 1.7320508075688772 / 8388608.0);
  const int threads = 256;
  long long blocks = (n + threads - 1) / threads;
  if (blocks > 148 * 64) blocks = 148 * 64;
  mgb_host::launch(mgb::fill_uniform_kernel, dim3((int)blocks), dim3(threads), 0, reinterpret_cast<cudaStream_t>(stream), nullptr,
      reinterpret_cast<__nv_bfloat16*>(out), (size_t)n, seed, tensor_id, scale, 0.0f, 0, (uint64_t)first);
  return mgb_host::launch_status();
}

}  // extern "C"
