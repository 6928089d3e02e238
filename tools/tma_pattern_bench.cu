// Does the global layout of the expert weights limit the HBM rate the grouped GEMM's TMA loads get?
// One persistent CTA per SM streams a [rows x K] bf16 matrix through a 6-stage ring of 2 x (64 rows x
// 64 K) boxes per stage, exactly the gate/up GEMM's A-operand access order (row tiles round-robin over
// CTAs, K fastest), with the consumer releasing every stage at once (no MMA):
//   mode 0: row-major [rows][K]       -- a box is 64 slices of 128 B at a K*2-byte stride
//   mode 1: K-blocked [rows/64][K/64][64][64] -- a box is 8 KB contiguous
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tmapb tools/tma_pattern_bench.cu \
//   -I paper_2503_09716_b200/csrc paper_2503_09716_b200/csrc/host.cu && /tmp/tmapb
#include <cstdio>

#include "common.cuh"

using namespace mgb;
constexpr int kStagesB = 6, kBoxBytes = 64 * 64 * 2;

__global__ void __launch_bounds__(64, 1) stream_kernel(const __grid_constant__ CUtensorMap tm,
                                                       const __grid_constant__ CUtensorMap tmb,
                                                       const __grid_constant__ CUtensorMap tmb16,
                                                       const __grid_constant__ CUtensorMap tmb32,
                                                       const __grid_constant__ CUtensorMap tmb64,
                                                       const __grid_constant__ CUtensorMap tmb104, int mode, int row_tiles,
                                                       int KB, int b_rows, int hold_ns, int b_box, int b_spread) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int kStageB = 2 * kBoxBytes + 16 * 1024;  // A (2 boxes) + up to 128 token rows of B
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStagesB * kStageB);
  uint64_t* empty = full + kStagesB;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStagesB; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int pairs = row_tiles / 2;  // two 64-row boxes per stage (gate + up rows of one unit)
  if (threadIdx.x == 0) {
    const uint64_t pol = policy_evict_first();
    int s = 0;
    uint32_t ph = 0;
    for (int u = blockIdx.x; u < pairs; u += gridDim.x) {
      for (int kb = 0; kb < KB; ++kb) {
        mbar_wait(&empty[s], ph ^ 1);
        mbar_arrive_expect_tx(&full[s], 2 * kBoxBytes + ((b_box == 104 || b_box == 3) ? 104 : (b_rows / b_box) * b_box) * 128);
        uint8_t* dst = smem + s * kStageB;
        for (int h = 0; h < 2; ++h) {
          const int rt = 2 * u + h;
          if (mode == 0) tma_load_2d(dst + h * kBoxBytes, &tm, &full[s], kb * 64, rt * 64, pol);
          else tma_load_4d(dst + h * kBoxBytes, &tm, &full[s], 0, 0, kb, rt);
        }
        // B: the unit's token rows (an L2-resident [208 x K] slice), 8-row boxes
        const int boff = (blockIdx.x % b_spread) * 256;  // which token slice this CTA reads
        if (b_box == 104) {        // one box for the whole half tile
          tma_load_2d(dst + 2 * kBoxBytes, &tmb104, &full[s], kb * 64, boff, policy_evict_last());
        } else if (b_box == 3) {   // 64 + 32 + 8 rows
          tma_load_2d(dst + 2 * kBoxBytes, &tmb64, &full[s], kb * 64, boff, policy_evict_last());
          tma_load_2d(dst + 2 * kBoxBytes + 64 * 128, &tmb32, &full[s], kb * 64, boff + 64, policy_evict_last());
          tma_load_2d(dst + 2 * kBoxBytes + 96 * 128, &tmb, &full[s], kb * 64, boff + 96, policy_evict_last());
        } else {
          for (int j = 0; j < b_rows / b_box; ++j)
            tma_load_2d(dst + 2 * kBoxBytes + j * b_box * 128, b_box == 8 ? &tmb : &tmb16, &full[s], kb * 64,
                        boff + j * b_box, policy_evict_last());
        }
        if (++s == kStagesB) { s = 0; ph ^= 1; }
      }
    }
  } else if (threadIdx.x == 32) {
    int s = 0;
    uint32_t ph = 0;
    for (int u = blockIdx.x; u < pairs; u += gridDim.x)
      for (int kb = 0; kb < KB; ++kb) {
        mbar_wait(&full[s], ph);
        if (hold_ns) {  // stand-in for the stage's MMAs: a busy wait of hold_ns cycles
          const long long t0 = clock64();
          while (clock64() - t0 < hold_ns) {}
        }
        mbar_arrive(&empty[s]);
        if (++s == kStagesB) { s = 0; ph ^= 1; }
      }
  }
}

int main() {
  const int K = 4096, rows = 2 * 14336 * 8;  // Mixtral's W_gate_up of 8 experts: 1.88 GB
  const size_t bytes = (size_t)rows * K * 2;
  void* w;
  cudaMalloc(&w, bytes);
  cudaMemset(w, 1, bytes);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int smem = kStagesB * (2 * kBoxBytes + 16 * 1024) + 2048;
  void* xb;
  cudaMalloc(&xb, (size_t)256 * 148 * K * 2);
  cudaMemset(xb, 1, (size_t)256 * 148 * K * 2);
  CUtensorMap tmb, tmb16;
  mgb_host::encode_tmap_2d_bf16(&tmb, xb, K, 256 * 148, (uint64_t)K * 2, 64, 8);
  mgb_host::encode_tmap_2d_bf16(&tmb16, xb, K, 256 * 148, (uint64_t)K * 2, 64, 16);
  CUtensorMap tmb32, tmb64, tmb104;
  mgb_host::encode_tmap_2d_bf16(&tmb32, xb, K, 256 * 148, (uint64_t)K * 2, 64, 32);
  mgb_host::encode_tmap_2d_bf16(&tmb64, xb, K, 256 * 148, (uint64_t)K * 2, 64, 64);
  mgb_host::encode_tmap_2d_bf16(&tmb104, xb, K, 256 * 148, (uint64_t)K * 2, 64, 104);
  cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  struct Case { int mode, b_rows, hold, box, spread; const char* what; };
  const Case cases[] = {{0, 104, 0, 3, 8, "A + B 64+32+8"},
                        {0, 104, 200, 3, 8, "A + B, hold 200 cycles"},
                        {0, 104, 400, 3, 8, "A + B, hold 400 cycles"},
                        {0, 104, 600, 3, 8, "A + B, hold 600 cycles"},
                        {0, 104, 800, 3, 8, "A + B, hold 800 cycles"}};
  for (const Case& c : cases) {
    const int mode = c.mode;
    CUtensorMap tm;
    if (mode == 0) {
      mgb_host::encode_tmap_2d_bf16(&tm, w, K, rows, (uint64_t)K * 2, 64, 64);
    } else {
      const uint64_t d[4] = {64, 64, (uint64_t)K / 64, (uint64_t)rows / 64};
      const uint64_t st[3] = {128, 64 * 128, (uint64_t)64 * 128 * (K / 64)};
      const uint32_t box[4] = {64, 64, 1, 1};
      mgb_host::encode_tmap_bf16(&tm, w, 4, d, st, box, true);
    }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int it = 0; it < 2; ++it) stream_kernel<<<sms, 64, smem>>>(tm, tmb, tmb16, tmb32, tmb64, tmb104, mode, rows / 64, K / 64, c.b_rows, c.hold, c.box, c.spread);
    cudaEventRecord(e0);
    const int n = 10;
    for (int it = 0; it < n; ++it) stream_kernel<<<sms, 64, smem>>>(tm, tmb, tmb16, tmb32, tmb64, tmb104, mode, rows / 64, K / 64, c.b_rows, c.hold, c.box, c.spread);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%-34s: %.3f ms per 1.88 GB of A, %.0f GB/s of A  [%s]\n", c.what, ms / n, bytes / (ms / n * 1e-3) / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
