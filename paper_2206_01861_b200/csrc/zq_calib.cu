// Order-exact float32 forward for static calibration:
// the reference calibrates by running the FLOAT model (evaluate.py:168-196 ->
// transformer.model_forward with PrecisionConfig.full(), transformer.py:405-440)
// and records max / min of every GEMM input.  A calibrated scale is
// f32(max(|EMA max|, |EMA min|) / qmax), so reproducing it bit for bit needs the
// float forward bit for bit.  These kernels restate its numpy arithmetic:
//
//   tensor.matmul (tensor.py:37-56): c[i,j] = sum_p a[i,p] * b[p,j] with every
//     product and partial sum rounded to f32, p ascending from +0.0 (einsum,
//     optimize=False), then `+= bias` (transformer.py:405-410);
//   transformer.attention (transformer.py:413-440): per head scores = q k^T
//     (the same sequential matmul), `*= 1/sqrt(dh)`, causal -inf mask,
//     tensor.softmax (tensor.py:94-99): x - rowmax, numpy's float32 exp, the
//     row sum in numpy's pairwise order, one IEEE division; then probs @ v;
//   numpy's float32 exp is NOT correctly rounded (39% of results differ from
//     RN(exp)): it is numpy 2.x's SIMD kernel (simd_exp_f32: Cody-Waite range
//     reduction, a [5/2] rational minimax, scalef), restated in np_expf below
//     and pinned against np.exp on CPU (tests/test_oracle_golden.py).
// LayerNorm and GeLU use the exact quantize-on-write kernels (their f32
// outputs); the GEMM-input taps reduce max / min on device (zq_minmax_f32).
// Off the hot path (offline calibration): simple CUDA-core kernels.

#include <math.h>

#include "zq_common.cuh"

namespace zq {

static inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// numpy 2.x float32 exp (numpy/_core/src/umath/loops_exponent_log.dispatch.c.src,
// simd_exp_f32; AVX512F / AVX2 universal-intrinsics path): FMA (npyv_muladd)
// everywhere the source fuses, x * 2^k formed exactly and rounded once.
__device__ __noinline__ float np_expf(float x) {
  if (x != x) return x;
  if (x >= 88.72283935546875f) return __int_as_float(0x7f800000);
  if (x <= -103.97208404541015625f) return 0.0f;
  float quad = __fmul_rn(x, 1.442695040888963407359924681001892137f);
  quad = __fsub_rn(__fadd_rn(quad, 12582912.0f), 12582912.0f);  // rint
  float r = __fmaf_rn(quad, -6.93145752e-1f, x);                 // Cody-Waite ln2 hi
  r = __fmaf_rn(quad, -1.42860677e-6f, r);                       // ln2 lo
  r = __fmaf_rn(quad, 0.0f, r);
  float num = __fmaf_rn(5.082762527590693718096e-04f, r, 6.757896990527504603057e-03f);
  num = __fmaf_rn(num, r, 5.114512081637298353406e-02f);
  num = __fmaf_rn(num, r, 2.473615434895520810817e-01f);
  num = __fmaf_rn(num, r, 7.257664613233124478488e-01f);
  num = __fmaf_rn(num, r, 9.999999999980870924916e-01f);
  float den = __fmaf_rn(2.159509375685829852307e-02f, r, -2.742335390411667452936e-01f);
  den = __fmaf_rn(den, r, 1.0f);
  const float v = __fdiv_rn(num, den);
  return __double2float_rn(__dmul_rn((double)v, ldexp(1.0, (int)quad)));
}

// numpy's float32 pairwise sum (the order of `a.sum(axis=-1, dtype=f32)` over a
// contiguous row): n < 8 sequential from +0.0; n <= 128 eight interleaved
// accumulators + ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) + sequential tail; else
// split at (n/2) rounded down to a multiple of 8.
__device__ float np_pairwise_sum(const float* a, int64_t n) {
  if (n < 8) {
    float r = 0.0f;
    for (int64_t i = 0; i < n; ++i) r = __fadd_rn(r, a[i]);
    return r;
  }
  if (n <= 128) {
    float r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int64_t i = 8;
    for (; i < n - (n % 8); i += 8)
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = __fadd_rn(r[j], a[i + j]);
    float res = __fadd_rn(__fadd_rn(__fadd_rn(r[0], r[1]), __fadd_rn(r[2], r[3])),
                          __fadd_rn(__fadd_rn(r[4], r[5]), __fadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __fadd_rn(res, a[i]);
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return __fadd_rn(np_pairwise_sum(a, n2), np_pairwise_sum(a + n2, n - n2));
}

// out[i, j] = (sum_p a[i, p] * w[j, p]) [+ bias[j]]: weights output-major
// (the reference's x @ w.T), p ascending, separately rounded products / sums.
constexpr int kSeqTile = 32;
__global__ void __launch_bounds__(kSeqTile * 8) matmul_seq_kernel(const float* __restrict__ a, int64_t lda,
                                                                 const float* __restrict__ w, int64_t ldw,
                                                                 const float* __restrict__ bias, int64_t M,
                                                                 int64_t N, int64_t K, float* __restrict__ out,
                                                                 int64_t ldo) {
  __shared__ float sa[kSeqTile][kSeqTile + 1];
  __shared__ float sw[kSeqTile][kSeqTile + 1];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 8 row groups of 4 rows
  const int64_t i0 = (int64_t)blockIdx.y * kSeqTile, j0 = (int64_t)blockIdx.x * kSeqTile;
  float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
  for (int64_t p0 = 0; p0 < K; p0 += kSeqTile) {
    for (int r = ty; r < kSeqTile; r += 8) {
      const int64_t ia = i0 + r, jw = j0 + r, p = p0 + tx;
      sa[r][tx] = (ia < M && p < K) ? a[ia * lda + p] : 0.0f;
      sw[r][tx] = (jw < N && p < K) ? w[jw * ldw + p] : 0.0f;
    }
    __syncthreads();
    const int pn = (int)((K - p0) < kSeqTile ? (K - p0) : kSeqTile);
    for (int pp = 0; pp < pn; ++pp) {
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[q] = __fadd_rn(acc[q], __fmul_rn(sa[ty * 4 + q][pp], sw[tx][pp]));
    }
    __syncthreads();
  }
  const int64_t j = j0 + tx;
  if (j >= N) return;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int64_t i = i0 + ty * 4 + q;
    if (i < M) out[i * ldo + j] = bias ? __fadd_rn(acc[q], bias[j]) : acc[q];
  }
}

// Softmax rows of one head: block = (query row i, head h).  scores / probs in
// the caller's scratch [heads, t, t].
__global__ void __launch_bounds__(128) attn_probs_kernel(const float* __restrict__ q, const float* __restrict__ k,
                                                        int64_t ld, int t, int dh, int causal, float inv,
                                                        float* __restrict__ scratch) {
  const int i = blockIdx.x, h = blockIdx.y;
  float* row = scratch + ((int64_t)h * t + i) * t;
  __shared__ float red[4];
  __shared__ float sum_s;
  const float* qi = q + (int64_t)i * ld + (int64_t)h * dh;
  float m = -INFINITY;
  for (int j = threadIdx.x; j < t; j += blockDim.x) {
    const float* kj = k + (int64_t)j * ld + (int64_t)h * dh;
    float s = 0.0f;
    for (int p = 0; p < dh; ++p) s = __fadd_rn(s, __fmul_rn(qi[p], kj[p]));
    s = __fmul_rn(s, inv);
    if (causal && j > i) s = -INFINITY;
    row[j] = s;
    m = fmaxf(m, s);
  }
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  m = fmaxf(fmaxf(red[0], red[1]), fmaxf(red[2], red[3]));
  for (int j = threadIdx.x; j < t; j += blockDim.x) row[j] = np_expf(__fsub_rn(row[j], m));
  __syncthreads();
  if (threadIdx.x == 0) sum_s = np_pairwise_sum(row, t);
  __syncthreads();
  const float s = sum_s;
  for (int j = threadIdx.x; j < t; j += blockDim.x) row[j] = __fdiv_rn(row[j], s);
}

// ctx[i, h*dh + c] = sum_j probs[h, i, j] * v[j, h*dh + c], j ascending from +0.0.
__global__ void __launch_bounds__(128) attn_pv_kernel(const float* __restrict__ v, int64_t ld, int t, int dh,
                                                     const float* __restrict__ scratch, float* __restrict__ ctx,
                                                     int64_t ld_ctx) {
  const int i = blockIdx.x, h = blockIdx.y;
  const float* p = scratch + ((int64_t)h * t + i) * t;
  for (int c = threadIdx.x; c < dh; c += blockDim.x) {
    float acc = 0.0f;
    for (int j = 0; j < t; ++j) acc = __fadd_rn(acc, __fmul_rn(p[j], v[(int64_t)j * ld + (int64_t)h * dh + c]));
    ctx[(int64_t)i * ld_ctx + (int64_t)h * dh + c] = acc;
  }
}

// [max, min] of n floats (exact in any order) + non-finite flag.
__global__ void __launch_bounds__(1024) minmax_kernel(const float* __restrict__ x, int64_t n,
                                                     float* __restrict__ out, int32_t* __restrict__ flag) {
  __shared__ float smax[32], smin[32];
  float mx = -INFINITY, mn = INFINITY;
  bool bad = false;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const float v = x[i];
    bad |= !isfinite(v);
    mx = fmaxf(mx, v);
    mn = fminf(mn, v);
  }
  if (bad && flag) atomicOr(flag, 1);
  for (int o = 16; o > 0; o >>= 1) {
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
  }
  if ((threadIdx.x & 31) == 0) {
    smax[threadIdx.x >> 5] = mx;
    smin[threadIdx.x >> 5] = mn;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    mx = smax[threadIdx.x];
    mn = smin[threadIdx.x];
    for (int o = 16; o > 0; o >>= 1) {
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    }
    if (threadIdx.x == 0) {
      out[0] = mx;
      out[1] = mn;
    }
  }
}

__global__ void np_expf_kernel(const float* __restrict__ x, int64_t n, float* __restrict__ y) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = np_expf(x[i]);
}

}  // namespace zq

using namespace zq;

extern "C" {

int zq_matmul_f32_seq(const float* a, int64_t lda, const float* w, int64_t ldw, const float* bias, int64_t M,
                      int64_t N, int64_t K, float* out, int64_t ldo, void* stream) {
  ZQ_CHECK_ARG(M >= 1 && N >= 1 && K >= 1, ZQ_ERR_SHAPE, "empty matmul (%lld, %lld, %lld)", (long long)M,
               (long long)N, (long long)K);
  ZQ_CHECK_ARG(lda >= K && ldw >= K && ldo >= N, ZQ_ERR_USAGE, "bad leading dimension");
  dim3 grid((unsigned)((N + kSeqTile - 1) / kSeqTile), (unsigned)((M + kSeqTile - 1) / kSeqTile));
  matmul_seq_kernel<<<grid, kSeqTile * 8, 0, as_stream(stream)>>>(a, lda, w, ldw, bias, M, N, K, out, ldo);
  ZQ_LAUNCH_CHECK("sequential f32 matmul launch");
  return ZQ_OK;
}

int zq_attention_exact_f32(const float* qkv, int64_t ld_qkv, int t, int heads, int head_dim, int causal,
                           float inv_scale, float* scratch, float* ctx, int64_t ld_ctx, void* stream) {
  ZQ_CHECK_ARG(t >= 1 && heads >= 1 && head_dim >= 1, ZQ_ERR_SHAPE, "bad attention shape");
  ZQ_CHECK_ARG(ld_qkv >= 3LL * heads * head_dim, ZQ_ERR_USAGE, "qkv row stride too small");
  const int64_t d = (int64_t)heads * head_dim;
  cudaStream_t st = as_stream(stream);
  attn_probs_kernel<<<dim3((unsigned)t, (unsigned)heads), 128, 0, st>>>(qkv, qkv + d, ld_qkv, t, head_dim, causal,
                                                                        inv_scale, scratch);
  attn_pv_kernel<<<dim3((unsigned)t, (unsigned)heads), 128, 0, st>>>(qkv + 2 * d, ld_qkv, t, head_dim, scratch,
                                                                     ctx, ld_ctx);
  ZQ_LAUNCH_CHECK("exact attention launch");
  return ZQ_OK;
}

int zq_minmax_f32(const float* x, int64_t n, float* out2, int32_t* nonfinite_flag, void* stream) {
  ZQ_CHECK_ARG(n >= 1, ZQ_ERR_USAGE, "min/max of an empty tensor");
  minmax_kernel<<<1, 1024, 0, as_stream(stream)>>>(x, n, out2, nonfinite_flag);
  ZQ_LAUNCH_CHECK("minmax launch");
  return ZQ_OK;
}

int zq_np_expf(const float* x, int64_t n, float* y, void* stream) {
  ZQ_CHECK_ARG(n >= 0, ZQ_ERR_USAGE, "bad size");
  if (n == 0) return ZQ_OK;
  int64_t blocks = (n + 255) / 256;
  if (blocks > 4096) blocks = 4096;
  np_expf_kernel<<<(unsigned)blocks, 256, 0, as_stream(stream)>>>(x, n, y);
  ZQ_LAUNCH_CHECK("np_expf launch");
  return ZQ_OK;
}

}  // extern "C"
