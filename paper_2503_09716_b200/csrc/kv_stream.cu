// KV streaming for kv_policy="offload" (the reference's full-KV-offload mode, PAPER.md:199-203;
// memory_model.py:182-205 puts every sequence's KV in host memory).
//
// Per layer and attention micro-batch the schedule issues (offload_dag.py:359-402):
//   KV_COPY_IN   host pages of the micro-batch -> an HBM ring slot        (copy engine, cudaMemcpyAsync)
//   PRE_ATTENTION appends the new token's K/V into a small HBM staging page per sequence
//   KV_COPY_OUT  staging -> the host page store, new token only             (mgb_kv_token_copy, SM stores
//                into mapped pinned memory: exactly nt * kv bytes cross the link, positions read on the device
//                so the copy is CUDA-graph replayable)
//   ATTN_MECH    staging -> ring slot (mgb_kv_token_copy, device to device), then the attention kernel on the slot
//
// Pages are opaque to this file: a token's bytes inside a page are `n_units` runs of `unit_bytes`,
// run u of token t at byte  u * unit_stride + t * unit_bytes.  GQA chunk-major pages
// ([head][hd/8][page tok][8], attn_gqa.cu) are unit_bytes = 16, unit_stride = 16 * page_tokens; MLA
// swizzled latent pages ([64-dim block][page tok][128 B], attn_mla.cu) are unit_bytes = 128,
// unit_stride = 128 * page_tokens.  Within-row swizzles depend only on the token's in-page slot, which
// source and destination share, so rows are copied verbatim.
#include "common.cuh"

namespace mgb {

// One thread per 16-byte vector of one sequence's new token.
__global__ void kv_token_copy_kernel(const uint8_t* __restrict__ src, const int* __restrict__ src_table,
                                     int src_max_pages, uint8_t* __restrict__ dst, const int* __restrict__ dst_table,
                                     int dst_max_pages, const int* __restrict__ positions, int B, int page_tokens,
                                     long long page_bytes, int unit_bytes, int n_units, long long unit_stride) {
  mgb::pdl_enter();
  const int vec_per_unit = unit_bytes >> 4;
  const int vec_per_tok = n_units * vec_per_unit;
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (long long)B * vec_per_tok) return;
  const int b = (int)(gid / vec_per_tok);
  const int v = (int)(gid - (long long)b * vec_per_tok);
  const int u = v / vec_per_unit, w = v - u * vec_per_unit;
  const int pos = positions[b];
  const int pg = pos / page_tokens, slot = pos - pg * page_tokens;
  if (pos < 0 || pg >= src_max_pages || pg >= dst_max_pages) return;  // past the planned context
  const long long off = (long long)u * unit_stride + (long long)slot * unit_bytes + (long long)w * 16;
  const long long sp = src_table[(size_t)b * src_max_pages + pg];
  const long long dp = dst_table[(size_t)b * dst_max_pages + pg];
  const uint4 x = __ldg(reinterpret_cast<const uint4*>(src + sp * page_bytes + off));
  *reinterpret_cast<uint4*>(dst + dp * page_bytes + off) = x;
}

// Plain byte copy by SM loads/stores (16 B per thread-iteration; either side may be mapped pinned
// host memory).  Used for the small per-layer transfers of the CPU attention share, which would
// otherwise queue on a copy engine behind the multi-hundred-MB KV_COPY_IN slices.
__global__ void copy_bytes_kernel(uint4* __restrict__ dst, const uint4* __restrict__ src, long long n16) {
  mgb::pdl_enter();
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += (long long)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

}  // namespace mgb

extern "C" {

int mgb_copy_bytes(void* dst, const void* src, long long nbytes, void* stream) {
  if (nbytes < 0 || nbytes % 16 || (reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) % 16)
    return MGB_EINVAL;
  if (nbytes == 0) return MGB_OK;
  const long long n16 = nbytes / 16;
  long long blocks = (n16 + 255) / 256;
  if (blocks > 4 * 148) blocks = 4 * 148;
  mgb_host::launch(mgb::copy_bytes_kernel, dim3((int)blocks), dim3(256), 0, reinterpret_cast<cudaStream_t>(stream), nullptr,
      reinterpret_cast<uint4*>(dst), reinterpret_cast<const uint4*>(src), n16);
  return mgb_host::launch_status();
}


// Copy the token at positions[b] of every sequence b in [0, B) from page src_table[b][pos / page_tokens]
// of `src` to page dst_table[b][pos / page_tokens] of `dst` (same in-page slot).  `dst` / `src` may be
// pinned host memory (mapped; UVA pointers).
int mgb_kv_token_copy(const void* src, const int* src_table, int src_max_pages, void* dst, const int* dst_table,
                      int dst_max_pages, const int* positions, int B, int page_tokens, long long page_bytes,
                      int unit_bytes, int n_units, long long unit_stride, void* stream) {
  if (B < 1 || page_tokens < 1 || n_units < 1 || unit_bytes < 16 || unit_bytes % 16 || page_bytes % 16 ||
      unit_stride % 16 || (long long)(n_units - 1) * unit_stride + (long long)page_tokens * unit_bytes > page_bytes)
    return MGB_EINVAL;
  const long long items = (long long)B * n_units * (unit_bytes / 16);
  const int threads = 256;
  mgb_host::launch(mgb::kv_token_copy_kernel, dim3((int)((items + threads - 1) / threads)), dim3(threads), 0, reinterpret_cast<cudaStream_t>(stream), nullptr,
      reinterpret_cast<const uint8_t*>(src), src_table, src_max_pages, reinterpret_cast<uint8_t*>(dst), dst_table,
      dst_max_pages, positions, B, page_tokens, page_bytes, unit_bytes, n_units, unit_stride);
  return mgb_host::launch_status();
}

}  // extern "C"
