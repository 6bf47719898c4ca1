// L2 -> SM TMA read throughput, measured alone and together with bulk stores:
// 148 CTAs, one producer thread each streams 16 KB 2-D TMA boxes (128 rows x
// 128 B, the GEMM's operand box) from a buffer through an NB-stage ring of
// mbarriers (consumer = the same thread waiting on each stage), optionally while
// 8 warps per CTA write 4 KB bulk stores (the GEMM epilogue's store path).
// Region size decides L2-resident vs DRAM.  nvcc -arch=sm_100a -lcuda.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int NB>
__global__ void __launch_bounds__(288, 1) tma_read(const __grid_constant__ CUtensorMap tm, int rows_total,
                                                   int iters, float* out, size_t out_chunks, int do_store,
                                                   unsigned long long* tstamp, int siters) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + NB * 16384 + 8 * 2 * 4096);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NB; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  if (warp == 8) {
    if (lane == 0) {
      const int nrb = rows_total / 128;
      for (int it = 0; it < iters; ++it) {
        const int s = it % NB;
        if (it >= NB) {
          const uint32_t ph = ((it / NB) - 1) & 1;
          asm volatile("{\n.reg .pred P;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W_%=;\n}\n" ::"r"(smem_u32(&bar[s])), "r"(ph) : "memory");
        }
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 16384;" ::"r"(smem_u32(&bar[s])) : "memory");
        const int rb = (blockIdx.x * 7 + it * 13) % nrb;
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                     ::"r"(smem_u32(sm + s * 16384)), "l"(&tm), "r"(smem_u32(&bar[s])), "r"(0), "r"(rb * 128) : "memory");
      }
      for (int it = iters > NB ? iters - NB : 0; it < iters; ++it) {
        const int s = it % NB;
        const uint32_t ph = (it / NB) & 1;
        asm volatile("{\n.reg .pred P;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W_%=;\n}\n" ::"r"(smem_u32(&bar[s])), "r"(ph) : "memory");
      }
      unsigned long long t1;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
      tstamp[blockIdx.x * 2] = t1 - t0;
    }
  } else if (do_store == 2) {  // plain st.global.v4 from registers (LSU path, no TMA)
    const size_t gw = (size_t)blockIdx.x * 8 + warp, nw = (size_t)gridDim.x * 8;
    for (int i = 0; i < siters; ++i) {
      const size_t chunk = (gw + i * nw) % out_chunks;
      const float4 v = make_float4((float)i, (float)lane, 1.f, 2.f);
      float4* o = reinterpret_cast<float4*>(out + chunk * 1024);
#pragma unroll
      for (int c = 0; c < 8; ++c) o[c * 32 + lane] = v;
    }
  } else if (do_store) {
    uint8_t* mine = sm + NB * 16384 + warp * 2 * 4096;
    const size_t gw = (size_t)blockIdx.x * 8 + warp, nw = (size_t)gridDim.x * 8;
    for (int i = 0; i < siters; ++i) {
      uint8_t* buf = mine + (i & 1) * 4096;
      if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      __syncwarp();
      const float4 v = make_float4((float)i, (float)lane, 1.f, 2.f);
      for (int c = 0; c < 8; ++c) reinterpret_cast<float4*>(buf)[c * 32 + lane] = v;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        const size_t chunk = (gw + i * nw) % out_chunks;
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 4096;" ::"l"(out + chunk * 1024),
                     "r"(smem_u32(buf)) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  if (warp < 8 && do_store) {
    __syncwarp();
    asm volatile("bar.sync 1, 256;" ::: "memory");
    if (threadIdx.x == 0) {
      unsigned long long t1;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
      tstamp[blockIdx.x * 2 + 1] = t1 - t0;
    }
  }
}

int main() {
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint8_t* buf;
  float* out;
  cudaMalloc(&buf, 1ull << 30);
  cudaMalloc(&out, 1ull << 30);
  cudaMemset(buf, 1, 1ull << 30);
  const int NB = 8;
  const int smem = NB * 16384 + 8 * 2 * 4096 + 1024;
  cudaFuncSetAttribute(tma_read<NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long* ts;
  cudaMallocManaged(&ts, 2 * 1024 * sizeof(unsigned long long));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (size_t region : {16ull << 20, 64ull << 20, 1024ull << 20}) {
    for (int st = 0; st < 3; ++st) {
      CUtensorMap tm;
      const int rows = (int)(region / 128);
      cuuint64_t dims[2] = {128, (cuuint64_t)rows};
      cuuint64_t strides[1] = {128};
      cuuint32_t box[2] = {128, 128};
      cuuint32_t es[2] = {1, 1};
      enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      const int iters = 2048;
      const size_t out_chunks = (16ull << 20) / 4096;  // stores into an L2-resident 16 MB region
      const int siters = iters / 4;  // 8 KB written per 16 KB read
      tma_read<NB><<<sms, 288, smem>>>(tm, rows, 64, out, out_chunks, st, ts, 16);
      cudaDeviceSynchronize();
      for (int i = 0; i < 2 * sms; ++i) ts[i] = 0;
      tma_read<NB><<<sms, 288, smem>>>(tm, rows, iters, out, out_chunks, st, ts, siters);
      cudaDeviceSynchronize();
      unsigned long long tr = 0, tw = 0;
      for (int i = 0; i < sms; ++i) {
        tr = ts[2 * i] > tr ? ts[2 * i] : tr;
        tw = ts[2 * i + 1] > tw ? ts[2 * i + 1] : tw;
      }
      const double rd = (double)sms * iters * 16384 / (tr * 1e-9) / 1e9;
      const double wr = st ? (double)sms * 8 * siters * 4096 / (tw * 1e-9) / 1e9 : 0.0;
      printf("read region %5zu MB  stores %-9s  read %8.1f GB/s (%5.1f per SM)  write %8.1f GB/s (%5.1f per SM)\n",
             region >> 20, st == 0 ? "off" : st == 1 ? "bulk" : "st.global", rd, rd / sms, wr, wr / sms);
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
