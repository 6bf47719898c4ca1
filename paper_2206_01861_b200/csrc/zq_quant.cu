// Bandwidth-bound quantization kernels:
//   K1 token-wise activation quantize      quant.py:258-269
//   K2 static activation quantize          quant.py:272-281 / :103-113
//   K3 group-wise weight quantize (+INT4)  quant.py:236-255
//   K4 (residual +) LayerNorm + quantize   igemm.py:150-157, tensor.py:59-73
//   K5 GeLU + quantize                     igemm.py:160-161, tensor.py:76-83
// All arithmetic that decides an int8 value or a scale is written with explicit
// round-to-nearest intrinsics (no FMA contraction) so the results are
// bit-identical to the reference's numpy arithmetic.
#include <cuda_fp16.h>
#include <stdarg.h>
#include <string.h>

#include <stdlib.h>

#include <algorithm>

#include "zq_common.cuh"
#include "zq_gelu.cuh"
#include "zq_rowops.h"

namespace zq {

static thread_local char g_err[512];

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

static inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

bool pdl_enabled() {
  static int mode = -1;
  if (mode < 0) {
    const char* e = getenv("ZQ_PDL");
    mode = e ? atoi(e) : 1;
  }
  return mode != 0;
}

// ---------------------------------------------------------------------------
// Row producers: what value each activation element holds before quantization.
// ---------------------------------------------------------------------------
struct IdentityOp {
  static constexpr bool kWarpOk = true;
  __device__ __forceinline__ float operator()(float x) const { return x; }
};

// ---------------------------------------------------------------------------
// K1/K5: one CTA per row, row held in registers as float4 chunks.
// Thread t owns chunks t, t+B, ..., t+(NC-1)B.
// ---------------------------------------------------------------------------
template <int NC, class Op>
__global__ void __launch_bounds__(1024) rowquant_vec_kernel(
    const float* __restrict__ x, int64_t cols, int64_t ld_x, int qm, Op op,
    float* __restrict__ y_out, int8_t* __restrict__ q, int64_t ld_q, float* __restrict__ scales,
    int32_t* __restrict__ flag) {
  __shared__ uint32_t red[32];
  const int64_t row = blockIdx.x;
  const int cols4 = (int)(cols >> 2);
  const float4* xr = reinterpret_cast<const float4*>(x + row * ld_x);
  float4 v[NC];
  float amax = 0.0f;
  bool bad = false;
#pragma unroll
  for (int i = 0; i < NC; ++i) {
    int c = threadIdx.x + i * blockDim.x;
    if (c < cols4) {
      float4 a = __ldg(xr + c);
      a.x = op(a.x);
      a.y = op(a.y);
      a.z = op(a.z);
      a.w = op(a.w);
      bad |= !(is_finite_f(a.x) && is_finite_f(a.y) && is_finite_f(a.z) && is_finite_f(a.w));
      amax = fmaxf(amax, fmaxf(fmaxf(fabsf(a.x), fabsf(a.y)), fmaxf(fabsf(a.z), fabsf(a.w))));
      v[i] = a;
    }
  }
  if (bad && flag) atomicOr(flag, 1);
  amax = block_max_nonneg(amax, red);
  const float s = scale_from_absmax(amax, qm);
  const float inv = safe_rcp(s);
  if (threadIdx.x == 0) scales[row] = s;
  char4* qr = reinterpret_cast<char4*>(q + row * ld_q);
  float4* yr = y_out ? reinterpret_cast<float4*>(y_out + row * cols) : nullptr;
#pragma unroll
  for (int i = 0; i < NC; ++i) {
    int c = threadIdx.x + i * blockDim.x;
    if (c < cols4) {
      char4 o;
      o.x = (signed char)quantize_fast(v[i].x, s, inv, qm);
      o.y = (signed char)quantize_fast(v[i].y, s, inv, qm);
      o.z = (signed char)quantize_fast(v[i].z, s, inv, qm);
      o.w = (signed char)quantize_fast(v[i].w, s, inv, qm);
      qr[c] = o;
      if (yr) yr[c] = v[i];
    }
  }
  // zero the K padding [cols, ld_q) so tensor-core K tails contribute nothing
  const int ldq4 = (int)(ld_q >> 2);
  for (int c = cols4 + threadIdx.x; c < ldq4; c += blockDim.x) qr[c] = make_char4(0, 0, 0, 0);
}

// Generic (any cols / alignment): two passes over the row, scalar loads.
template <class Op>
__global__ void __launch_bounds__(256) rowquant_scalar_kernel(
    const float* __restrict__ x, int64_t cols, int64_t ld_x, int qm, Op op,
    float* __restrict__ y_out, int8_t* __restrict__ q, int64_t ld_q, float* __restrict__ scales,
    int32_t* __restrict__ flag) {
  __shared__ uint32_t red[32];
  const int64_t row = blockIdx.x;
  const float* xr = x + row * ld_x;
  float amax = 0.0f;
  bool bad = false;
  for (int64_t c = threadIdx.x; c < cols; c += blockDim.x) {
    float a = op(xr[c]);
    bad |= !is_finite_f(a);
    amax = fmaxf(amax, fabsf(a));
  }
  if (bad && flag) atomicOr(flag, 1);
  amax = block_max_nonneg(amax, red);
  const float s = scale_from_absmax(amax, qm);
  if (threadIdx.x == 0) scales[row] = s;
  int8_t* qr = q + row * ld_q;
  for (int64_t c = threadIdx.x; c < ld_q; c += blockDim.x) {
    if (c < cols) {
      float a = op(xr[c]);
      qr[c] = (int8_t)quantize_exact(a, s, qm);
      if (y_out) y_out[row * cols + c] = a;
    } else {
      qr[c] = 0;
    }
  }
}

template <class Op>
static int launch_rowquant(const float* x, int64_t rows, int64_t cols, int64_t ld_x, int bits,
                           Op op, float* y_out, int8_t* q, int64_t ld_q, float* scales,
                           int32_t* flag, cudaStream_t st) {
  const int qm = qmax_of(bits);
  const bool vec = (cols % 4 == 0) && (ld_x % 4 == 0) &&
                   ((reinterpret_cast<uintptr_t>(x) & 15) == 0) && (ld_q % 16 == 0) &&
                   ((reinterpret_cast<uintptr_t>(q) & 15) == 0) &&
                   (!y_out || (reinterpret_cast<uintptr_t>(y_out) & 15) == 0);
  const int64_t cols4 = cols / 4;
  if (vec && cols4 <= 1024 * 16) {
    int nc = 1;
    while ((cols4 + nc - 1) / nc > 1024 || ((cols4 + nc - 1) / nc > 256 && nc < 4)) nc *= 2;
    int threads = (int)(((cols4 + nc - 1) / nc + 31) / 32 * 32);
    if (threads < 32) threads = 32;
    dim3 grid((unsigned)rows);
    switch (nc) {
      case 1: rowquant_vec_kernel<1, Op><<<grid, threads, 0, st>>>(x, cols, ld_x, qm, op, y_out, q, ld_q, scales, flag); break;
      case 2: rowquant_vec_kernel<2, Op><<<grid, threads, 0, st>>>(x, cols, ld_x, qm, op, y_out, q, ld_q, scales, flag); break;
      case 4: rowquant_vec_kernel<4, Op><<<grid, threads, 0, st>>>(x, cols, ld_x, qm, op, y_out, q, ld_q, scales, flag); break;
      case 8: rowquant_vec_kernel<8, Op><<<grid, threads, 0, st>>>(x, cols, ld_x, qm, op, y_out, q, ld_q, scales, flag); break;
      default: rowquant_vec_kernel<16, Op><<<grid, threads, 0, st>>>(x, cols, ld_x, qm, op, y_out, q, ld_q, scales, flag); break;
    }
  } else {
    rowquant_scalar_kernel<Op><<<(unsigned)rows, 256, 0, st>>>(x, cols, ld_x, qm, op, y_out, q,
                                                                ld_q, scales, flag);
  }
  ZQ_LAUNCH_CHECK("row quantize launch");
  return ZQ_OK;
}

// ---------------------------------------------------------------------------
// K2: static quantization, one scale for the whole tensor
// ---------------------------------------------------------------------------
__global__ void static_quant_kernel(const float* __restrict__ x, int64_t rows, int64_t cols,
                                    int64_t ld_x, float s32, double s64, int use_f32, int qm,
                                    int8_t* __restrict__ q, int64_t ld_q,
                                    int32_t* __restrict__ flag) {
  const int64_t total = rows * ld_q;
  bool bad = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i / ld_q, c = i - r * ld_q;
    int8_t o = 0;
    if (c < cols) {
      float a = x[r * ld_x + c];
      bad |= !is_finite_f(a);
      o = (int8_t)(use_f32 ? quantize_exact(a, s32, qm) : quantize_f64(a, s64, qm));
    }
    q[i] = o;
  }
  if (bad && flag) atomicOr(flag, 1);
}

// ---------------------------------------------------------------------------
// Row max |x| (K3 phase 1, TP token absmax)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) row_absmax_kernel(const float* __restrict__ x,
                                                         int64_t cols, int64_t ld_x,
                                                         float* __restrict__ amax,
                                                         int32_t* __restrict__ flag) {
  __shared__ uint32_t red[32];
  const float* xr = x + (int64_t)blockIdx.x * ld_x;
  float m = 0.0f;
  bool bad = false;
  for (int64_t c = threadIdx.x; c < cols; c += blockDim.x) {
    float a = xr[c];
    bad |= !is_finite_f(a);
    m = fmaxf(m, fabsf(a));
  }
  if (bad && flag) atomicOr(flag, 1);
  m = block_max_nonneg(m, red);
  if (threadIdx.x == 0) amax[blockIdx.x] = m;
}

// K3 phase 2: group max -> scale (quant.py:249-252), expanded row scales.
__global__ void group_scale_kernel(const float* __restrict__ row_amax, int64_t rows,
                                   int64_t groups, int qm, float* __restrict__ group_scales,
                                   float* __restrict__ row_scales) {
  int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= groups) return;
  const int64_t base = rows / groups;
  const int64_t start = g * base;
  const int64_t count = (g == groups - 1) ? rows - start : base;
  float m = 0.0f;
  for (int64_t r = 0; r < count; ++r) m = fmaxf(m, row_amax[start + r]);
  float s = scale_from_absmax(m, qm);
  group_scales[g] = s;
  for (int64_t r = 0; r < count; ++r) row_scales[start + r] = s;
}

// K3 phase 3: quantize every row with its group scale; optional INT4 pack.
__global__ void rowscale_quant_kernel(const float* __restrict__ w, int64_t rows, int64_t cols,
                                      const float* __restrict__ row_scales, int qm,
                                      int8_t* __restrict__ q, int64_t ld_q) {
  const int64_t total = rows * ld_q;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i / ld_q, c = i - r * ld_q;
    q[i] = (c < cols) ? (int8_t)quantize_exact(w[r * cols + c], row_scales[r], qm) : (int8_t)0;
  }
}

__global__ void pack_int4_kernel(const int8_t* __restrict__ q, int64_t rows, int64_t ld_q,
                                 uint8_t* __restrict__ packed) {
  const int64_t half = ld_q / 2;
  const int64_t total = rows * half;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i / half, k = i - r * half;
    uint8_t lo = (uint8_t)q[r * ld_q + 2 * k] & 0xF;
    uint8_t hi = (uint8_t)q[r * ld_q + 2 * k + 1] & 0xF;
    packed[i] = (uint8_t)(lo | (hi << 4));
  }
}

// TP: quantize with a given (all-reduced) per-row absmax.
// Token-wise quantization with the all-reduced row max (tensor-parallel row-parallel
// projections): one CTA per row (grid-stride), the scale and its reciprocal once per
// row, float4 loads, the branch-free fast rounding with the exact fallback for
// near-ties (the same arithmetic as tok_quant_kernel, so bit-identical to it).
__global__ void __launch_bounds__(256) quant_with_absmax_kernel(const float* __restrict__ x, int64_t rows,
                                                                int64_t cols, int64_t ld_x,
                                                                const float* __restrict__ amax, int qm,
                                                                int8_t* __restrict__ q, int64_t ld_q,
                                                                float* __restrict__ scales) {
  pdl_trigger();
  pdl_wait();
  const bool vec = (cols & 3) == 0 && (ld_x & 3) == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(q) & 3) == 0 && (ld_q & 3) == 0;
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    const float s = scale_from_absmax(amax[r], qm);
    const float inv = safe_rcp(s);
    if (threadIdx.x == 0) scales[r] = s;
    const float* xr = x + r * ld_x;
    int8_t* qr = q + r * ld_q;
    if (vec) {
      const int64_t n4 = cols >> 2;
      for (int64_t c = threadIdx.x; c < n4; c += blockDim.x) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(xr) + c);
        bool amb = inv == 0.0f;
        int o0 = qbf(v.x, inv, qm, kQMargin, amb), o1 = qbf(v.y, inv, qm, kQMargin, amb),
            o2 = qbf(v.z, inv, qm, kQMargin, amb), o3 = qbf(v.w, inv, qm, kQMargin, amb);
        if (amb) {
          o0 = quantize_exact_slow(v.x, s, qm);
          o1 = quantize_exact_slow(v.y, s, qm);
          o2 = quantize_exact_slow(v.z, s, qm);
          o3 = quantize_exact_slow(v.w, s, qm);
        }
        reinterpret_cast<uint32_t*>(qr)[c] = pack4(o0, o1, o2, o3);
      }
      for (int64_t c = cols + threadIdx.x; c < ld_q; c += blockDim.x) qr[c] = 0;
    } else {
      for (int64_t c = threadIdx.x; c < ld_q; c += blockDim.x)
        qr[c] = c < cols ? (int8_t)quantize_exact(xr[c], s, qm) : (int8_t)0;
    }
  }
}

// ---------------------------------------------------------------------------
// K4: (residual +) LayerNorm + token-wise quantize, numpy pairwise reductions.
// ---------------------------------------------------------------------------
// numpy's float32 pairwise sum (see oracle.lowbit_oracle.pairwise_sum_f32):
// leaves of <=128 elements, each summed with 8 interleaved accumulators
// combined ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) plus a sequential tail; leaves
// combined by the binary split tree n2 = (n/2) rounded down to a multiple of 8.
// The plan (computed on the host per row width) lists the leaves and the
// internal-node combines level by level, so the tree is evaluated in parallel.
constexpr int kMaxLeaves = 256;
constexpr int kMaxNodes = 2 * kMaxLeaves;
constexpr int kMaxLevels = 24;

struct PairwisePlan {
  int n;
  int nleaves;
  int nlevels;
  int root;
  int leaf_start[kMaxLeaves];
  short leaf_len[kMaxLeaves];
  short level_begin[kMaxLevels + 1];
  short op_dst[kMaxLeaves];
  short op_a[kMaxLeaves];
  short op_b[kMaxLeaves];
};

struct PlanBuilder {
  PairwisePlan* p;
  int next_slot;
  int depth_of[kMaxNodes];
  int ops_dst[kMaxLeaves], ops_a[kMaxLeaves], ops_b[kMaxLeaves], ops_h[kMaxLeaves];
  int nops;
  bool ok;
  // returns (slot, height)
  int rec(int start, int n, int* height) {
    if (n <= 128) {
      if (p->nleaves >= kMaxLeaves) {
        ok = false;
        *height = 0;
        return 0;
      }
      int id = p->nleaves++;
      p->leaf_start[id] = start;
      p->leaf_len[id] = (short)n;
      *height = 0;
      return id;
    }
    int n2 = n / 2;
    n2 -= n2 % 8;
    int ha, hb;
    int a = rec(start, n2, &ha);
    int b = rec(start + n2, n - n2, &hb);
    int h = (ha > hb ? ha : hb) + 1;
    if (nops >= kMaxLeaves) {
      ok = false;
      *height = h;
      return 0;
    }
    ops_a[nops] = a;
    ops_b[nops] = b;
    ops_h[nops] = h;
    ops_dst[nops] = -1;
    *height = h;
    return -(++nops);  // negative: internal node index
  }
};

static bool build_plan(int n, PairwisePlan* plan) {
  memset(plan, 0, sizeof(*plan));
  plan->n = n;
  PlanBuilder b;
  b.p = plan;
  b.nops = 0;
  b.ok = true;
  int h;
  int root = b.rec(0, n, &h);
  if (!b.ok || h > kMaxLevels) return false;
  // slot numbering: leaves 0..L-1, internal node i (1-based) -> L + i - 1
  auto slot = [&](int s) { return s >= 0 ? s : plan->nleaves + (-s) - 1; };
  plan->root = slot(root);
  plan->nlevels = h;
  int k = 0;
  for (int lev = 1; lev <= h; ++lev) {
    plan->level_begin[lev - 1] = (short)k;
    for (int i = 0; i < b.nops; ++i)
      if (b.ops_h[i] == lev) {
        plan->op_dst[k] = (short)(plan->nleaves + i);
        plan->op_a[k] = (short)slot(b.ops_a[i]);
        plan->op_b[k] = (short)slot(b.ops_b[i]);
        ++k;
      }
  }
  plan->level_begin[h] = (short)k;
  return true;
}

// Pairwise sum of f(row[i]) over the plan.  All threads of the block call it.
// `slots` has >= 2*nleaves floats.
template <class F>
__device__ float pairwise_sum_block(const float* row, const PairwisePlan& plan, F f,
                                    float* slots) {
  const int n = plan.n;
  if (n < 8) {
    __syncthreads();
    if (threadIdx.x == 0) {
      float r = 0.0f;
      for (int i = 0; i < n; ++i) r = __fadd_rn(r, f(row[i]));
      slots[0] = r;
    }
    __syncthreads();
    return slots[0];
  }
  // chains: thread handles (leaf = c >> 3, j = c & 7); lanes of one leaf are an
  // aligned group of 8 so the 8-accumulator combine is a 3-step butterfly.
  const int nchains = plan.nleaves * 8;
  for (int base = 0; base < nchains; base += blockDim.x) {
    int c = base + threadIdx.x;
    float acc = 0.0f;
    int leaf = c >> 3, j = c & 7;
    bool act = c < nchains;
    int len = 0, st = 0;
    if (act) {
      len = plan.leaf_len[leaf];
      st = plan.leaf_start[leaf];
      int m = len - len % 8;
      acc = f(row[st + j]);
      for (int i = 8 + j; i < m; i += 8) acc = __fadd_rn(acc, f(row[st + i]));
    }
    // ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) : IEEE addition is commutative, so
    // the butterfly reproduces the fixed tree exactly.
    acc = __fadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, 1));
    acc = __fadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, 2));
    acc = __fadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, 4));
    if (act && j == 0) {
      int m = len - len % 8;
      for (int i = m; i < len; ++i) acc = __fadd_rn(acc, f(row[st + i]));
      slots[leaf] = acc;
    }
  }
  __syncthreads();
  for (int lev = 0; lev < plan.nlevels; ++lev) {
    int b = plan.level_begin[lev], e = plan.level_begin[lev + 1];
    for (int k = b + threadIdx.x; k < e; k += blockDim.x)
      slots[plan.op_dst[k]] = __fadd_rn(slots[plan.op_a[k]], slots[plan.op_b[k]]);
    __syncthreads();
  }
  float r = slots[plan.root];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(256) ln_quant_kernel(
    const float* __restrict__ x, const float* __restrict__ res, const float* __restrict__ gamma,
    const float* __restrict__ beta, int64_t cols, float eps, int qm,
    const __grid_constant__ PairwisePlan plan, float* __restrict__ ln_out,
    int8_t* __restrict__ q, int64_t ld_q, float* __restrict__ scales,
    int32_t* __restrict__ flag) {
  extern __shared__ float sm[];
  __shared__ uint32_t red[32];
  float* row = sm;                 // cols floats
  float* slots = sm + cols;        // 2 * nleaves floats
  const int64_t r = blockIdx.x;
  const float* xr = x + r * cols;
  const float* rr = res ? res + r * cols : nullptr;
  bool bad = false;
  for (int64_t c = threadIdx.x; c < cols; c += blockDim.x) {
    float v = xr[c];
    if (rr) v = __fadd_rn(v, rr[c]);  // (x + attn_out) / (h + f), transformer.py:477,486
    bad |= !is_finite_f(v);
    row[c] = v;
  }
  if (bad && flag) atomicOr(flag, 1);
  __syncthreads();
  const float fcols = (float)cols;
  const float sum = pairwise_sum_block(row, plan, [](float v) { return v; }, slots);
  const float mean = __fdiv_rn(sum, fcols);
  const float sq = pairwise_sum_block(
      row, plan,
      [mean](float v) {
        float d = __fsub_rn(v, mean);
        return __fmul_rn(d, d);
      },
      slots);
  const float var = __fdiv_rn(sq, fcols);
  const float den = __fsqrt_rn(__fadd_rn(var, eps));
  float amax = 0.0f;
  for (int64_t c = threadIdx.x; c < cols; c += blockDim.x) {
    float nv = __fdiv_rn(__fsub_rn(row[c], mean), den);
    float y = __fadd_rn(__fmul_rn(nv, gamma[c]), beta[c]);
    row[c] = y;
    amax = fmaxf(amax, fabsf(y));
    bad |= !is_finite_f(y);
  }
  if (bad && flag) atomicOr(flag, 1);
  amax = block_max_nonneg(amax, red);  // contains __syncthreads
  const float s = scale_from_absmax(amax, qm);
  if (threadIdx.x == 0) scales[r] = s;
  int8_t* qr = q + r * ld_q;
  for (int64_t c = threadIdx.x; c < ld_q; c += blockDim.x) {
    if (c < cols) {
      float y = row[c];
      qr[c] = (int8_t)quantize_exact(y, s, qm);
      if (ln_out) ln_out[r * cols + c] = y;
    } else {
      qr[c] = 0;
    }
  }
}

// Uniform-tree test on a host plan: 2^k equal leaves of 64..128 elements.
static bool plan_uniform(const PairwisePlan& p, int* E_out, int* nchains_out) {
  if (p.n < 256) return false;
  const int L = p.leaf_len[0];
  if (L % 8 != 0 || L < 64 || L > 128) return false;
  for (int i = 1; i < p.nleaves; ++i)
    if (p.leaf_len[i] != L) return false;
  if (p.nleaves & (p.nleaves - 1)) return false;
  const int nch = 8 * p.nleaves;
  if (nch < 32 || nch > 512) return false;  // <= 8 warps x 2 chains per lane
  *E_out = L / 8;
  *nchains_out = nch;
  return true;
}

struct PlanCache {
  int n = -1;
  PairwisePlan plan;
};
static thread_local PlanCache g_plan_cache;

}  // namespace zq

using namespace zq;

extern "C" {

const char* zq_last_error(void) { return zq::g_err; }

int zq_quantize_tokenwise(const float* x, int64_t rows, int64_t cols, int64_t ld_x, int bits,
                          int8_t* q, int64_t ld_q, float* token_scales, int32_t* flag,
                          void* stream) {
  ZQ_CHECK_ARG(bits_ok(bits), ZQ_ERR_USAGE, "unsupported bit width %d, expected one of (4, 8)", bits);
  ZQ_CHECK_ARG(rows >= 1 && cols >= 1, ZQ_ERR_USAGE, "activations must be (tokens x dim), got (%lld, %lld)",
               (long long)rows, (long long)cols);
  ZQ_CHECK_ARG(ld_x >= cols && ld_q >= cols && ld_q % 16 == 0, ZQ_ERR_USAGE, "bad leading dimensions");
  if (cols % 4 == 0 && ld_x % 4 == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0 &&
      (reinterpret_cast<uintptr_t>(q) & 15) == 0 &&
      launch_tok_quant(x, rows, cols, ld_x, qmax_of(bits), q, ld_q, token_scales, flag,
                       as_stream(stream)) == ZQ_OK) {
    ZQ_LAUNCH_CHECK("token-wise quantize launch");
    return ZQ_OK;
  }
  return launch_rowquant(x, rows, cols, ld_x, bits, IdentityOp{}, nullptr, q, ld_q, token_scales,
                         flag, as_stream(stream));
}

int zq_gelu_quantize(const float* x, int64_t rows, int64_t cols, int64_t ld_x, int bits,
                     float* gelu_out, int8_t* q, int64_t ld_q, float* token_scales, int32_t* flag,
                     void* stream) {
  ZQ_CHECK_ARG(bits_ok(bits), ZQ_ERR_USAGE, "unsupported bit width %d, expected one of (4, 8)", bits);
  ZQ_CHECK_ARG(rows >= 1 && cols >= 1, ZQ_ERR_USAGE, "activations must be (tokens x dim)");
  ZQ_CHECK_ARG(ld_x >= cols && ld_q >= cols && ld_q % 16 == 0, ZQ_ERR_USAGE, "bad leading dimensions");
  if (gelu_out == nullptr && cols % 4 == 0 && ld_x % 4 == 0 &&
      (reinterpret_cast<uintptr_t>(x) & 15) == 0 && (reinterpret_cast<uintptr_t>(q) & 15) == 0 &&
      launch_gelu_quant(x, rows, cols, ld_x, qmax_of(bits), q, ld_q, token_scales, flag,
                        as_stream(stream)) == ZQ_OK) {
    ZQ_LAUNCH_CHECK("gelu quantize launch");
    return ZQ_OK;
  }
  return launch_rowquant(x, rows, cols, ld_x, bits, GeluOp{}, gelu_out, q, ld_q, token_scales,
                         flag, as_stream(stream));
}

int zq_gelu_estimate(const float* x, int64_t n, float* est, float* bound, void* stream) {
  ZQ_CHECK_ARG(n >= 1, ZQ_ERR_USAGE, "empty input");
  launch_gelu_estimate(x, n, est, bound, as_stream(stream));
  ZQ_LAUNCH_CHECK("gelu estimate launch");
  return ZQ_OK;
}

int zq_quantize_static(const float* x, int64_t rows, int64_t cols, int64_t ld_x, double scale,
                       int bits, int8_t* q, int64_t ld_q, int32_t* flag, void* stream) {
  ZQ_CHECK_ARG(bits_ok(bits), ZQ_ERR_USAGE, "unsupported bit width %d, expected one of (4, 8)", bits);
  ZQ_CHECK_ARG(scale > 0.0, ZQ_ERR_USAGE, "calibrated scale must be > 0, got %g", scale);
  ZQ_CHECK_ARG(rows >= 0 && cols >= 0 && ld_x >= cols && ld_q >= cols, ZQ_ERR_USAGE, "bad shape");
  if (rows == 0) return ZQ_OK;
  float s32 = (float)scale;
  int use_f32 = ((double)s32 == scale) && s32 > 0.0f;
  int64_t total = rows * ld_q;
  int blocks = (int)((total + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  static_quant_kernel<<<blocks, 256, 0, as_stream(stream)>>>(x, rows, cols, ld_x, s32, scale,
                                                             use_f32, qmax_of(bits), q, ld_q, flag);
  ZQ_LAUNCH_CHECK("static quantize launch");
  return ZQ_OK;
}

int zq_row_absmax(const float* x, int64_t rows, int64_t cols, int64_t ld_x, float* amax,
                  int32_t* flag, void* stream) {
  ZQ_CHECK_ARG(rows >= 1 && cols >= 1 && ld_x >= cols, ZQ_ERR_USAGE, "bad shape");
  row_absmax_kernel<<<(unsigned)rows, 256, 0, as_stream(stream)>>>(x, cols, ld_x, amax, flag);
  ZQ_LAUNCH_CHECK("row absmax launch");
  return ZQ_OK;
}

// float64 inputs (quant.py:80-95 / :103-113 read their input as float64
// without an f32 round trip): exact row max of |x| and RHAFZ(x / scale) with
// the f64 division, +0.5 and floor of the reference (_round_half_away).
__global__ void __launch_bounds__(256) row_absmax_f64_kernel(const double* __restrict__ x, int64_t cols,
                                                             int64_t ld_x, double* __restrict__ amax,
                                                             int32_t* __restrict__ flag) {
  __shared__ double red[32];
  const double* xr = x + (int64_t)blockIdx.x * ld_x;
  double m = 0.0;
  bool bad = false;
  for (int64_t c = threadIdx.x; c < cols; c += blockDim.x) {
    const double a = xr[c];
    bad |= !isfinite(a);
    m = fmax(m, fabs(a));
  }
  if (bad && flag) atomicOr(flag, 1);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    m = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (threadIdx.x == 0) amax[blockIdx.x] = m;
  }
}

__global__ void quantize_array_f64_kernel(const double* __restrict__ x, int64_t n, double scale, int qm,
                                          int8_t* __restrict__ q, int32_t* __restrict__ flag) {
  bool bad = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double v = __ddiv_rn(x[i], scale);
    bad |= !isfinite(x[i]);
    const double a = fmin(floor(__dadd_rn(fabs(v), 0.5)), (double)qm);
    const int k = (int)a;  // inf -> qm (np.clip); NaN raises on the host
    q[i] = (int8_t)(v < 0.0 ? -k : k);
  }
  if (bad && flag) atomicOr(flag, 1);
}

int zq_row_absmax_f64(const double* x, int64_t rows, int64_t cols, int64_t ld_x, double* amax, int32_t* flag,
                      void* stream) {
  ZQ_CHECK_ARG(rows >= 1 && cols >= 1 && ld_x >= cols, ZQ_ERR_USAGE, "bad shape");
  row_absmax_f64_kernel<<<(unsigned)rows, 256, 0, as_stream(stream)>>>(x, cols, ld_x, amax, flag);
  ZQ_LAUNCH_CHECK("row absmax (f64) launch");
  return ZQ_OK;
}

int zq_quantize_array_f64(const double* x, int64_t n, double scale, int bits, int8_t* q, int32_t* flag,
                          void* stream) {
  ZQ_CHECK_ARG(bits_ok(bits), ZQ_ERR_USAGE, "unsupported bit width %d, expected one of (4, 8)", bits);
  ZQ_CHECK_ARG(scale > 0.0, ZQ_ERR_USAGE, "quantization scale must be > 0, got %g", scale);
  ZQ_CHECK_ARG(n >= 0, ZQ_ERR_USAGE, "bad size");
  if (n == 0) return ZQ_OK;
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  quantize_array_f64_kernel<<<(unsigned)blocks, 256, 0, as_stream(stream)>>>(x, n, scale, qmax_of(bits), q, flag);
  ZQ_LAUNCH_CHECK("quantize array (f64) launch");
  return ZQ_OK;
}

int zq_quantize_with_absmax(const float* x, int64_t rows, int64_t cols, int64_t ld_x,
                            const float* amax, int bits, int8_t* q, int64_t ld_q,
                            float* token_scales, void* stream) {
  ZQ_CHECK_ARG(bits_ok(bits), ZQ_ERR_USAGE, "unsupported bit width %d", bits);
  ZQ_CHECK_ARG(rows >= 1 && cols >= 1 && ld_x >= cols && ld_q >= cols && ld_q % 16 == 0,
               ZQ_ERR_USAGE, "bad shape");
  const int blocks = (int)std::min<int64_t>(rows, (int64_t)zq_num_sms() * 8);
  const cudaError_t e = launch_kernel(quant_with_absmax_kernel, dim3(blocks), dim3(256), 0, as_stream(stream), 1, x,
                                      rows, cols, ld_x, amax, qmax_of(bits), q, ld_q, token_scales);
  if (e != cudaSuccess) {
    set_error("quantize with absmax launch: %s", cudaGetErrorString(e));
    return ZQ_ERR_CUDA;
  }
  return ZQ_OK;
}

int zq_quantize_weight_groupwise(const float* w, int64_t rows, int64_t cols, int64_t groups,
                                 int bits, int8_t* q, int64_t ld_q, float* group_scales,
                                 float* row_scales, uint8_t* packed4, int32_t* flag,
                                 void* stream) {
  ZQ_CHECK_ARG(bits_ok(bits), ZQ_ERR_USAGE, "unsupported bit width %d, expected one of (4, 8)", bits);
  ZQ_CHECK_ARG(rows >= 1 && cols >= 1, ZQ_ERR_USAGE, "weight matrix must be 2-d and non-empty");
  ZQ_CHECK_ARG(groups >= 1 && groups <= rows, ZQ_ERR_USAGE, "group count %lld invalid for %lld rows",
               (long long)groups, (long long)rows);
  ZQ_CHECK_ARG(ld_q >= cols && ld_q % 16 == 0, ZQ_ERR_USAGE, "bad leading dimension");
  ZQ_CHECK_ARG(!packed4 || bits == 4, ZQ_ERR_USAGE, "int4 packing requires bits == 4");
  cudaStream_t st = as_stream(stream);
  // row maxima go to row_scales (overwritten by the expanded scales in phase 2)
  float* row_amax = nullptr;
  if (cudaMallocAsync(&row_amax, sizeof(float) * rows, st) != cudaSuccess) {
    set_error("cudaMallocAsync failed");
    return ZQ_ERR_CUDA;
  }
  row_absmax_kernel<<<(unsigned)rows, 256, 0, st>>>(w, cols, cols, row_amax, flag);
  group_scale_kernel<<<(unsigned)((groups + 127) / 128), 128, 0, st>>>(row_amax, rows, groups,
                                                                       qmax_of(bits),
                                                                       group_scales, row_scales);
  int64_t total = rows * ld_q;
  int blocks = (int)((total + 255) / 256);
  if (blocks > 148 * 32) blocks = 148 * 32;
  rowscale_quant_kernel<<<blocks, 256, 0, st>>>(w, rows, cols, row_scales, qmax_of(bits), q, ld_q);
  if (packed4) {
    int64_t tp = rows * (ld_q / 2);
    int pb = (int)((tp + 255) / 256);
    if (pb > 148 * 32) pb = 148 * 32;
    pack_int4_kernel<<<pb, 256, 0, st>>>(q, rows, ld_q, packed4);
  }
  cudaFreeAsync(row_amax, st);
  ZQ_LAUNCH_CHECK("group-wise weight quantize launch");
  return ZQ_OK;
}

int zq_pack_int4(const int8_t* q, int64_t rows, int64_t ld_q, uint8_t* packed, void* stream) {
  ZQ_CHECK_ARG(rows >= 1 && ld_q >= 2 && ld_q % 2 == 0, ZQ_ERR_USAGE, "bad shape for int4 pack");
  int64_t tp = rows * (ld_q / 2);
  int pb = (int)((tp + 255) / 256);
  if (pb > 148 * 32) pb = 148 * 32;
  pack_int4_kernel<<<pb, 256, 0, as_stream(stream)>>>(q, rows, ld_q, packed);
  ZQ_LAUNCH_CHECK("int4 pack launch");
  return ZQ_OK;
}

int zq_layer_norm_quantize(const float* x, const float* residual, const float* gamma,
                           const float* beta, int64_t rows, int64_t cols, float eps, int bits,
                           float* ln_out, int8_t* q, int64_t ld_q, float* token_scales,
                           int32_t* flag, void* stream) {
  ZQ_CHECK_ARG(bits_ok(bits), ZQ_ERR_USAGE, "unsupported bit width %d, expected one of (4, 8)", bits);
  ZQ_CHECK_ARG(rows >= 1 && cols >= 1, ZQ_ERR_USAGE, "activations must be (tokens x dim)");
  ZQ_CHECK_ARG(eps > 0.0f, ZQ_ERR_USAGE, "layer_norm eps must be > 0");
  ZQ_CHECK_ARG(ld_q >= cols && ld_q % 16 == 0, ZQ_ERR_USAGE, "bad leading dimension");
  ZQ_CHECK_ARG(cols <= 32768, ZQ_ERR_UNSUPPORTED, "layer_norm_quantize supports rows up to 32768 wide");
  if (g_plan_cache.n != (int)cols) {
    if (!build_plan((int)cols, &g_plan_cache.plan)) {
      g_plan_cache.n = -1;
      set_error("pairwise plan overflow for width %lld", (long long)cols);
      return ZQ_ERR_UNSUPPORTED;
    }
    g_plan_cache.n = (int)cols;
  }
  const PairwisePlan& plan = g_plan_cache.plan;
  int E = 0, nch = 0;
  auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (plan_uniform(plan, &E, &nch) && cols % 4 == 0 && al16(x) && al16(residual) && al16(gamma) &&
      al16(beta) && al16(ln_out) && al16(q) &&
      launch_ln_quant_uniform(x, residual, gamma, beta, rows, cols, plan.nleaves, plan.leaf_len[0],
                              eps, qmax_of(bits), ln_out, q, ld_q, token_scales, flag,
                              as_stream(stream)) == ZQ_OK) {
    ZQ_LAUNCH_CHECK("layer_norm_quantize (uniform) launch");
    return ZQ_OK;
  }
  size_t smem = sizeof(float) * (cols + 2 * (size_t)plan.nleaves + 2);
  static ZqDeviceOnce attr_set_once;
  attr_set_once([&](int) {
    cudaFuncSetAttribute(ln_quant_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  });
  int threads = cols >= 2048 ? 256 : 128;
  ln_quant_kernel<<<(unsigned)rows, threads, smem, as_stream(stream)>>>(
      x, residual, gamma, beta, cols, eps, qmax_of(bits), plan, ln_out, q, ld_q, token_scales,
      flag);
  ZQ_LAUNCH_CHECK("layer_norm_quantize launch");
  return ZQ_OK;
}

}  // extern "C"

// L2 residency control for an engine's hot activation pool (cudaStreamAttribute
// access-policy window, captured into graph kernel nodes): accesses inside
// [base, base + bytes) are marked persisting (up to the device's set-aside), the
// rest of the window streaming.  bytes == 0 clears the window.  Returns the
// persisting set-aside actually granted (bytes) through *granted when non-null.
extern "C" int zq_l2_persist(void* stream, const void* base, int64_t bytes, int64_t* granted) {
  int dev = 0;
  cudaGetDevice(&dev);
  int max_persist = 0, max_window = 0;
  cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, dev);
  cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, dev);
  cudaStreamAttrValue attr;
  memset(&attr, 0, sizeof(attr));
  int64_t setaside = 0;
  if (bytes > 0 && max_persist > 0 && max_window > 0) {
    setaside = bytes < max_persist ? bytes : max_persist;
    if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)setaside) != cudaSuccess) {
      cudaGetLastError();
      setaside = 0;
    }
  }
  if (setaside > 0) {
    const int64_t win = bytes < max_window ? bytes : max_window;
    attr.accessPolicyWindow.base_ptr = const_cast<void*>(base);
    attr.accessPolicyWindow.num_bytes = (size_t)win;
    attr.accessPolicyWindow.hitRatio = (float)((double)setaside / (double)win > 1.0 ? 1.0 : (double)setaside / (double)win);
    attr.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    attr.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  }
  const cudaError_t e = cudaStreamSetAttribute(reinterpret_cast<cudaStream_t>(stream),
                                               cudaStreamAttributeAccessPolicyWindow, &attr);
  if (granted) *granted = setaside;
  if (e != cudaSuccess) {
    set_error("L2 access policy window: %s", cudaGetErrorString(e));
    return ZQ_ERR_CUDA;
  }
  return ZQ_OK;
}

