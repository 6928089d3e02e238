// Streaming microbenchmark: how much HBM bandwidth does one CTA per SM get from a ring of
// `stages` x `bytes` cp.async.bulk copies (consumer releases each stage immediately)?
// Used to size the attention kernels' smem rings.   nvcc -gencode arch=compute_100a,code=sm_100a
// -O3 -o /tmp/ring tools/bulk_ring_bench.cu -I paper_2503_09716_b200/csrc && /tmp/ring
#include <cstdio>
#include <vector>

#include "common.cuh"

using namespace mgb;

__global__ void ring_kernel(const uint8_t* __restrict__ src, size_t total, int stages, int bytes, int hold_ns) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)stages * bytes);
  uint64_t* empty = full + stages;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const size_t n_chunks = total / bytes;
  if (threadIdx.x == 0) {
    const uint64_t pol = policy_evict_first();
    int s = 0;
    uint32_t ph = 0;
    for (size_t c = blockIdx.x; c < n_chunks; c += gridDim.x) {
      mbar_wait(&empty[s], ph ^ 1);
      mbar_arrive_expect_tx(&full[s], bytes);
      bulk_load(smem + (size_t)s * bytes, src + c * bytes, bytes, &full[s], pol);
      if (++s == stages) { s = 0; ph ^= 1; }
    }
  } else if (threadIdx.x == 32) {
    int s = 0;
    uint32_t ph = 0;
    for (size_t c = blockIdx.x; c < n_chunks; c += gridDim.x) {
      mbar_wait(&full[s], ph);
      if (hold_ns) __nanosleep(hold_ns);
      mbar_arrive(&empty[s]);
      if (++s == stages) { s = 0; ph ^= 1; }
    }
  }
}

int main() {
  const size_t total = (size_t)4 << 30;
  uint8_t* buf;
  cudaMalloc(&buf, total);
  cudaMemset(buf, 1, total);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(ring_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  struct Cfg { int stages, bytes, ctas, hold; };
  std::vector<Cfg> cfgs = {{2, 73728, 1, 0},  {2, 73728, 1, 1000}, {3, 49152, 1, 0}, {4, 36864, 1, 0},
                           {4, 36864, 1, 500}, {6, 24576, 1, 0},   {8, 18432, 1, 0}, {2, 36864, 2, 0},
                           {2, 36864, 1, 0},   {3, 65536, 1, 0},   {3, 65536, 1, 1000}, {12, 16384, 1, 0}};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (auto c : cfgs) {
    const size_t smem = (size_t)c.stages * c.bytes + 2 * c.stages * 8;
    for (int w = 0; w < 2; ++w) ring_kernel<<<sms * c.ctas, 64, smem>>>(buf, total, c.stages, c.bytes, c.hold);
    cudaEventRecord(e0);
    const int reps = 5;
    for (int r = 0; r < reps; ++r) ring_kernel<<<sms * c.ctas, 64, smem>>>(buf, total, c.stages, c.bytes, c.hold);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double gbs = (double)(total / c.bytes * c.bytes) * reps / (ms * 1e-3) / 1e9;
    printf("stages=%d bytes=%d ctas/SM=%d hold=%dns: %.0f GB/s  (%s)\n", c.stages, c.bytes, c.ctas, c.hold, gbs,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
