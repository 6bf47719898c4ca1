// Per-SM store throughput of the GEMM epilogue's store path, measured alone:
// 148 CTAs x 8 warps; each warp repeatedly fills a 4 KB smem staging buffer and
// writes it out with a bulk copy (cp.async.bulk.global.shared::cta), keeping
// NB buffers in flight, or with plain coalesced st.global.v4 from registers.
// Output region size decides L2-resident vs DRAM.  nvcc -arch=sm_100a.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

template <int NB>
__global__ void __launch_bounds__(256, 1) bulk_store(float* out, size_t chunks_per_warp, size_t total_chunks) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* mine = sm + warp * NB * 4096;
  const size_t gw = (size_t)blockIdx.x * 8 + warp;
  const size_t nw = (size_t)gridDim.x * 8;
  int b = 0;
  for (size_t i = 0; i < chunks_per_warp; ++i) {
    const size_t chunk = (gw + i * nw) % total_chunks;
    uint8_t* buf = mine + b * 4096;
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(NB - 1) : "memory");
    __syncwarp();
    float4 v = make_float4((float)i, (float)lane, 1.f, 2.f);
#pragma unroll
    for (int c = 0; c < 8; ++c) reinterpret_cast<float4*>(buf)[c * 32 + lane] = v;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 4096;" ::"l"(out + chunk * 1024),
                   "r"(smem_u32(buf))
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    b = (b + 1) % NB;
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void __launch_bounds__(256, 1) reg_store(float4* out, size_t chunks_per_warp, size_t total_chunks) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t gw = (size_t)blockIdx.x * 8 + warp;
  const size_t nw = (size_t)gridDim.x * 8;
  for (size_t i = 0; i < chunks_per_warp; ++i) {
    const size_t chunk = (gw + i * nw) % total_chunks;
    float4 v = make_float4((float)i, (float)lane, 1.f, 2.f);
#pragma unroll
    for (int c = 0; c < 8; ++c) out[chunk * 256 + c * 32 + lane] = v;
  }
}

int main() {
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, 0);
  const int sms = prop.multiProcessorCount;
  float* out;
  const size_t maxb = 1ull << 30;
  cudaMalloc(&out, maxb);
  cudaFuncSetAttribute(bulk_store<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 2 * 4096);
  cudaFuncSetAttribute(bulk_store<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 4 * 4096);
  cudaFuncSetAttribute(bulk_store<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 8 * 4096);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (size_t region : {8ull << 20, 32ull << 20, 64ull << 20, 512ull << 20}) {
    const size_t total_chunks = region / 4096;
    const size_t bytes = 1ull << 30;  // bytes written per launch
    const size_t cpw = bytes / 4096 / ((size_t)sms * 8);
    for (int variant = 0; variant < 4; ++variant) {
      auto launch = [&]() {
        if (variant == 0) bulk_store<2><<<sms, 256, 8 * 2 * 4096>>>(out, cpw, total_chunks);
        if (variant == 1) bulk_store<4><<<sms, 256, 8 * 4 * 4096>>>(out, cpw, total_chunks);
        if (variant == 2) bulk_store<8><<<sms, 256, 8 * 8 * 4096>>>(out, cpw, total_chunks);
        if (variant == 3) reg_store<<<sms, 256>>>(reinterpret_cast<float4*>(out), cpw, total_chunks);
      };
      launch();
      cudaDeviceSynchronize();
      cudaEventRecord(a);
      for (int r = 0; r < 3; ++r) launch();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double gbs = 3.0 * cpw * sms * 8 * 4096 / (ms * 1e-3) / 1e9;
      const char* names[4] = {"bulk NB=2", "bulk NB=4", "bulk NB=8", "st.global.v4"};
      printf("region %4zu MB  %-12s  %8.1f GB/s total  %6.1f GB/s per SM\n", region >> 20, names[variant], gbs,
             gbs / sms);
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
