// Packed f32x2 arithmetic (sm_100 FADD2 / FMUL2 / FFMA2, PTX add/sub/mul/fma.rn.f32x2)
// against the scalar _rn intrinsics, bit for bit, on 8.4 M random pairs (every
// other one with raw random bits: subnormals, infinities and NaNs included),
// with broadcast and negated operands.  The row kernels and GEMM epilogues rely
// on this.  Build: nvcc -gencode arch=compute_100a,code=sm_100a
// -O3 -fmad=false tools/f32x2_exactness.cu; prints the mismatch counts (all 0).
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cstring>
__device__ __forceinline__ uint64_t pk(float a, float b) { uint64_t r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ void up(uint64_t v, float& a, float& b) { asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v)); }
__global__ void k(const float* a, const float* b, const float* c, int n, unsigned* bad) {
  int i = blockIdx.x * blockDim.x + threadIdx.x; if (2 * i + 1 >= n) return;
  float a0 = a[2*i], a1 = a[2*i+1], b0 = b[2*i], b1 = b[2*i+1], c0 = c[2*i], c1 = c[2*i+1];
  uint64_t A = pk(a0, a1), B = pk(b0, b1), C = pk(c0, c1), r; float r0, r1;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(A), "l"(B)); up(r, r0, r1);
  if (__float_as_uint(r0) != __float_as_uint(__fadd_rn(a0, b0)) || __float_as_uint(r1) != __float_as_uint(__fadd_rn(a1, b1))) atomicAdd(bad + 0, 1);
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(A), "l"(B)); up(r, r0, r1);
  if (__float_as_uint(r0) != __float_as_uint(__fsub_rn(a0, b0)) || __float_as_uint(r1) != __float_as_uint(__fsub_rn(a1, b1))) atomicAdd(bad + 1, 1);
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(A), "l"(B)); up(r, r0, r1);
  if (__float_as_uint(r0) != __float_as_uint(__fmul_rn(a0, b0)) || __float_as_uint(r1) != __float_as_uint(__fmul_rn(a1, b1))) atomicAdd(bad + 2, 1);
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(A), "l"(B), "l"(C)); up(r, r0, r1);
  if (__float_as_uint(r0) != __float_as_uint(__fmaf_rn(a0, b0, c0)) || __float_as_uint(r1) != __float_as_uint(__fmaf_rn(a1, b1, c1))) atomicAdd(bad + 3, 1);
  {
    float dd = c[1];
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(pk(-dd, -dd)), "l"(A), "l"(B)); up(r, r0, r1);
    if (__float_as_uint(r0) != __float_as_uint(__fmaf_rn(-dd, a0, b0)) || __float_as_uint(r1) != __float_as_uint(__fmaf_rn(-dd, a1, b1))) atomicAdd(bad + 5, 1);
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(A), "l"(pk(dd, dd)), "l"(B)); up(r, r0, r1);
    if (__float_as_uint(r0) != __float_as_uint(__fmaf_rn(a0, dd, b0)) || __float_as_uint(r1) != __float_as_uint(__fmaf_rn(a1, dd, b1))) atomicAdd(bad + 6, 1);
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(A), "l"(pk(dd, dd))); up(r, r0, r1);
    if (__float_as_uint(r0) != __float_as_uint(__fmul_rn(a0, dd)) || __float_as_uint(r1) != __float_as_uint(__fmul_rn(a1, dd))) atomicAdd(bad + 7, 1);
  }
  // splat-constant forms
  float m = c[0];
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(A), "l"(pk(m, m))); up(r, r0, r1);
  if (__float_as_uint(r0) != __float_as_uint(__fsub_rn(a0, m)) || __float_as_uint(r1) != __float_as_uint(__fsub_rn(a1, m))) atomicAdd(bad + 4, 1);
}
int main() {
  const int n = 1 << 24; float *a, *b, *c; unsigned* bad;
  cudaMallocManaged(&a, n * 4); cudaMallocManaged(&b, n * 4); cudaMallocManaged(&c, n * 4); cudaMallocManaged(&bad, 64);
  srand(1); memset(bad, 0, 64);
  for (int i = 0; i < n; ++i) { uint32_t u = ((uint32_t)rand() << 16) ^ rand(); uint32_t v = ((uint32_t)rand() << 16) ^ rand(); uint32_t w = ((uint32_t)rand() << 16) ^ rand();
    if (i & 1) { u = (u & 0x807fffff) | ((120 + rand() % 16) << 23); v = (v & 0x807fffff) | ((120 + rand() % 16) << 23); w = (w & 0x807fffff) | ((120 + rand() % 16) << 23); }
    memcpy(a + i, &u, 4); memcpy(b + i, &v, 4); memcpy(c + i, &w, 4); }
  k<<<n / 2 / 256, 256>>>(a, b, c, n, bad); cudaDeviceSynchronize();
  printf("mismatch add %u sub %u mul %u fma %u subsplat %u fmanegsplatA %u fmasplatB %u mulsplat %u (of %d pairs)\n", bad[0], bad[1], bad[2], bad[3], bad[4], bad[5], bad[6], bad[7], n / 2);
}
