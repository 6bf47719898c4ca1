// Float attention of the post-LN block (transformer.py:413-440) on tcgen05:
//   S = (Q K^T) * 1/sqrt(dh); causal -> -inf above the diagonal; P = softmax(S);
//   ctx = P V
// The reference computes this in float32 (sequential sums); it is outside the
// bit-exact contract (tolerance parity), but we keep ~fp32 accuracy: every
// operand x is split into hi = x with the low 13 mantissa bits cleared (exactly
// representable in tf32) and lo = x - hi (exact in f32), and each product is
// formed as hi*hi + hi*lo + lo*hi (3 tcgen05 kind::tf32 MMAs into one f32 TMEM
// accumulator) — relative error ~2^-21 instead of tf32's 2^-11.  The tensor core
// reads only the top 19 bits of a tf32 operand (measured: feeding the raw f32 as
// "hi" gives the same 3e-6 error as the explicitly truncated value), so the raw
// TMA-staged tiles serve as hi and only lo is written.
//
// Persistent CTAs (one per SM) walk the (sequence, head) pairs; seq <= 128,
// head_dim = 64 (BERT-base, GPT-3 350M heads).  256 threads, per head:
//   1. TMA brings Q, K, V of the head (6 boxes of [128 rows x 32 f32],
//      SWIZZLE_128B) straight from the fused QKV GEMM output: Q and K land in
//      the K-major layout the MMA reads;
//   2. all threads write lo(Q), lo(K) (same swizzled layout, a flat pass) and
//      transpose V into K-major V^T hi / lo (with B MN-major the kind::tf32 MMA
//      returned zeros on this build, so only K-major operands are used); the
//      next head's V load is issued as soon as V is consumed;
//   3. one warp issues 24 MMAs for S (M=128, N=128, K=64) -> TMEM cols [0,128);
//      once they complete, Q / K are dead and the next head's Q / K loads go out;
//   4. 8 warps softmax: warp w reads TMEM lanes 32*(w%4).. (query rows), column
//      half w/4; row max / sum combined through smem; P hi / lo are written back
//      to TMEM (cols [0,128) / [128,256)) with tcgen05.st;
//   5. one warp issues 48 MMAs for O with A = P read from TMEM, B = V^T
//      (M=128, N=64, K=128) -> TMEM cols [256,320);
//   6. 8 warps read O and store ctx rows (f32).
#include <cuda.h>
#include <cuda_fp16.h>
#include <string.h>

#include "zq_common.cuh"

namespace zq {

constexpr int kAttT = 128;   // max sequence (query rows = MMA M)
constexpr int kAttD = 64;    // head dim
// smem: [Qh | Ql | Kh | Kl | V | VTh | VTl], 32 KB each.  Q/K: 2 K-major atoms
// of [128 rows x 128 B] (32 head-dim columns each), as TMA lands them.  V: the
// same TMA layout (rows = tokens); VTh/VTl: V^T hi/lo as the K-major B operand
// of P.V (64 rows = head dim, 4 atoms of 32 tokens).  P hi / lo (128 x 128 f32,
// 4 K-major atoms each) overlay Qh..Kl once S is computed.
constexpr int kRegion = kAttT * kAttD * 4;         // 32 KB
constexpr uint32_t kTmemQ = 320;                   // TMEM columns of Q hi [320,384) / lo [384,448)
constexpr int kAttSmem = 7 * kRegion + 64 + 2 * 128 * 4;  // + barriers / TMEM slot / row partials

__device__ __forceinline__ uint32_t make_idesc_tf32(int M, int N, int b_mn_major) {
  return (1u << 4)                       // c_format F32
         | (2u << 7)                     // a_format TF32
         | (2u << 10)                    // b_format TF32
         | ((uint32_t)b_mn_major << 16)  // B major-ness (1 = MN-major)
         | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// MN-major SWIZZLE_128B operand (kept for reference: with kind::tf32 and B
// MN-major the MMA produced zeros on this B200 build, so V is transposed): 128-byte rows hold 32 consecutive MN elements,
// 8 rows (K) per 1024-byte swizzle atom; LBO = stride between 32-element MN
// blocks, SBO = stride between 8-row K groups.
__device__ __forceinline__ uint64_t make_sw128_mn_desc(uint32_t smem_addr, uint32_t lbo,
                                                       uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr & 0x3FFFFu) >> 4);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ float ex2_approx_f(float v) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
  return r;
}

// One elected lane of a converged warp issues the MMA (operands warp-uniform, so
// no per-lane R2UR loops around the instruction).
__device__ __forceinline__ void mma_tf32_elect(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                               uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p, e;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_commit_elect(uint64_t* bar) {
  asm volatile(
      "{\n"
      ".reg .pred e;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
      "}\n" ::"r"(smem_u32(bar))
      : "memory");
}

// hi = x with the low 13 mantissa bits cleared (a tf32 value), lo = x - hi (exact)
__device__ __forceinline__ void split_tf32(float x, float& hi, float& lo) {
  hi = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
  lo = __fsub_rn(x, hi);
}

// byte offset of element (row r, k) in a K-major SWIZZLE_128B operand of `rows`
// rows: atoms of 128 bytes along K, each [rows][128 B], 16-byte chunks XORed
// with (row & 7)
__device__ __forceinline__ uint32_t sw_off(int rows, int r, int k_bytes) {
  const int atom = k_bytes >> 7, wb = k_bytes & 127;
  return atom * rows * 128 + r * 128 + ((((wb >> 4) ^ (r & 7))) << 4) + (wb & 15);
}

__device__ __forceinline__ void mma_tf32_ts_elect(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc,
                                                  uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p, e;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void tmem_st_32x32b_x32(uint32_t taddr, const float (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]),
      "f"(v[8]), "f"(v[9]), "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15]),
      "f"(v[16]), "f"(v[17]), "f"(v[18]), "f"(v[19]), "f"(v[20]), "f"(v[21]), "f"(v[22]), "f"(v[23]),
      "f"(v[24]), "f"(v[25]), "f"(v[26]), "f"(v[27]), "f"(v[28]), "f"(v[29]), "f"(v[30]), "f"(v[31])
      : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// Persistent: CTA c handles heads c, c + grid, ...  TMEM (512 columns): S and
// then P hi in [0,128), P lo in [128,256), O in [256,320).  P never touches smem
// (the P.V MMAs read A from TMEM), so Q and K are dead as soon as the S MMAs
// complete and the next head's Q / K TMA loads are issued right then; the next
// V load goes out as soon as V has been transposed.
__global__ void __launch_bounds__(256, 1)
    attention_kernel(const __grid_constant__ CUtensorMap tm, int seq, int heads, int dmodel,
                     int causal, float scale, float* __restrict__ ctx, int64_t ld_ctx, int nheads_total,
                     unsigned long long* __restrict__ trace, const __grid_constant__ CUtensorMap tmc,
                     int tma_store) {
  // no static smem in this kernel: the dynamic window starts 1024-aligned, and
  // addressing it directly (no integer round trip) keeps every access LDS/STS
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* sQh = sm;
  uint8_t* sQl = sm + kRegion;
  uint8_t* sKh = sm + 2 * kRegion;
  uint8_t* sKl = sm + 3 * kRegion;
  uint8_t* sV = sm + 4 * kRegion;
  uint8_t* sVh = sm + 5 * kRegion;
  uint8_t* sVl = sm + 6 * kRegion;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 7 * kRegion);  // QK, V, S, O
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 4);
  float* red = reinterpret_cast<float*>(bar + 5);  // [2][128] row partials (max / sum)

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    if (smem_u32(sm) & 1023) __trap();  // SWIZZLE_128B atoms need 1024-byte alignment
    prefetch_tmap(&tm);
    for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  const int quarter = warp & 3, half = warp >> 2;
  const int row = quarter * 32 + lane;  // query index (TMEM lane)

  auto issue_qk = [&](int hd) {
    const int b = hd / heads, h = hd % heads;
    mbar_arrive_expect_tx(&bar[0], 4 * 128 * 128);
#pragma unroll
    for (int part = 0; part < 2; ++part)
#pragma unroll
      for (int j = 0; j < 2; ++j)
        tma_load_2d(sm + 2 * part * kRegion + j * (kRegion / 2), &tm, &bar[0],
                    part * dmodel + h * kAttD + 32 * j, b * seq);
  };
  auto issue_v = [&](int hd) {
    const int b = hd / heads, h = hd % heads;
    mbar_arrive_expect_tx(&bar[1], 2 * 128 * 128);
#pragma unroll
    for (int j = 0; j < 2; ++j)
      tma_load_2d(sV + j * (kRegion / 2), &tm, &bar[1], 2 * dmodel + h * kAttD + 32 * j, b * seq);
  };

  pdl_trigger();
  pdl_wait();  // the QKV GEMM output is ready (and the previous ctx reader is done)
  if (tid == 0 && (int)blockIdx.x < nheads_total) {
    issue_qk(blockIdx.x);
    issue_v(blockIdx.x);
  }
  int it = 0;
  unsigned long long* tr = (trace && tid == 0) ? trace + (size_t)blockIdx.x * 64 : nullptr;
  for (int hd = blockIdx.x; hd < nheads_total; hd += gridDim.x, ++it) {
    const uint32_t ph = it & 1;
    if (tr && it < 8) tr[it * 8 + 0] = gtime();
    const int nxt = hd + gridDim.x;
    const int b = hd / heads, h = hd % heads;
    mbar_wait(&bar[1], ph);
    mbar_wait(&bar[0], ph);
    if (tma_store && it > 0) {  // the previous head's O staging (in lo(K)) must be read out
      if (tid == 0) bulk_wait_read0();
      __syncthreads();
    }
    if (tr && it < 8) tr[it * 8 + 1] = gtime();
    // ---- Q -> TMEM as hi / lo (the S MMAs read A from TMEM: Q leaves smem once);
    //      lo(K) in place; V -> K-major V^T hi / lo ----
    {
      const uint8_t* qrow = sQh + half * (kRegion / 2) + row * 128;
      float qh[32], ql[32];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const float4 x = *reinterpret_cast<const float4*>(qrow + ((c ^ (row & 7)) << 4));
        split_tf32(x.x, qh[4 * c], ql[4 * c]);
        split_tf32(x.y, qh[4 * c + 1], ql[4 * c + 1]);
        split_tf32(x.z, qh[4 * c + 2], ql[4 * c + 2]);
        split_tf32(x.w, qh[4 * c + 3], ql[4 * c + 3]);
      }
      const uint32_t tq = tmem + ((uint32_t)(quarter * 32) << 16) + kTmemQ + half * 32;
      tmem_st_32x32b_x32(tq, qh);
      tmem_st_32x32b_x32(tq + kAttD, ql);
    }
    for (int i = tid; i < kRegion / 16; i += 256) {
      const int off = i * 16;
      const float4 x = *reinterpret_cast<const float4*>(sKh + off);
      float4 hi, lo;
      split_tf32(x.x, hi.x, lo.x);
      split_tf32(x.y, hi.y, lo.y);
      split_tf32(x.z, hi.z, lo.z);
      split_tf32(x.w, hi.w, lo.w);
      *reinterpret_cast<float4*>(sKl + off) = lo;
    }
    {
      const int j = (warp & 1) * 32 + lane;  // head-dim column
      const uint8_t* vcol = sV + (j >> 5) * (kRegion / 2) + (j & 3) * 4;
      const int jc = (j & 31) >> 2;
#pragma unroll 2
      for (int q = warp >> 1; q < kAttT / 4; q += 4) {  // token quad
        float v[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int t = 4 * q + e;
          v[e] = *reinterpret_cast<const float*>(vcol + t * 128 + ((jc ^ (t & 7)) << 4));
        }
        float4 hi, lo;
        split_tf32(v[0], hi.x, lo.x);
        split_tf32(v[1], hi.y, lo.y);
        split_tf32(v[2], hi.z, lo.z);
        split_tf32(v[3], hi.w, lo.w);
        hi = make_float4(v[0], v[1], v[2], v[3]);  // the MMA reads only the tf32 bits
        const uint32_t o = (q >> 3) * (kAttD * 128) + j * 128 + (((q & 7) ^ (j & 7)) << 4);
        *reinterpret_cast<float4*>(sVh + o) = hi;
        *reinterpret_cast<float4*>(sVl + o) = lo;
      }
    }
    tmem_st_wait();
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (tr && it < 8) tr[it * 8 + 2] = gtime();
    if (tid == 0 && nxt < nheads_total) issue_v(nxt);  // V raw is free again

    // ---- S = Q K^T (3-term split) -> TMEM [0,128) ----
    if (warp == 0) {
      const uint32_t idesc = make_idesc_tf32(128, 128, 0);
      const uint64_t dKh = make_sw128_desc(smem_u32(sKh)), dKl = make_sw128_desc(smem_u32(sKl));
#pragma unroll
      for (int t3 = 0; t3 < 3; ++t3)
#pragma unroll
        for (int ks = 0; ks < kAttD / 8; ++ks) {
          const int kb = 32 * ks;
          const uint64_t boff = (uint64_t)(((kb >> 7) * kAttT * 128 + (kb & 127)) >> 4);
          mma_tf32_ts_elect(tmem, tmem + kTmemQ + (t3 == 2 ? kAttD : 0) + 8 * ks, (t3 == 1 ? dKl : dKh) + boff,
                            idesc, (t3 | ks) != 0);
        }
      mma_commit_elect(&bar[2]);
    }
    mbar_wait(&bar[2], ph);
    tc_fence_after();
    if (tr && it < 8) tr[it * 8 + 3] = gtime();
    if (tid == 0 && nxt < nheads_total) issue_qk(nxt);  // Q / K are consumed

    // ---- softmax rows: S from TMEM, P hi / lo back into TMEM ----
    float s[64];
    {
      uint32_t r0[32], r1[32];
      const uint32_t ta = tmem + ((uint32_t)(quarter * 32) << 16) + half * 64;
      tmem_ld_32x32b_x32(ta, r0);
      tmem_ld_32x32b_x32(ta + 32, r1);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        s[j] = __uint_as_float(r0[j]);
        s[32 + j] = __uint_as_float(r1[j]);
      }
    }
    // scores * inv (transformer.py:432) is folded into the exponent: the max is
    // taken over raw scores (inv > 0) and exp(inv (s - max)) = 2^(s c - max c),
    // c = inv log2(e); the common rounding of max c cancels in the normalisation
    float mx = -INFINITY;
    if (seq == kAttT && !causal) {  // no masked keys (BERT's full 128-token rows)
#pragma unroll
      for (int j = 0; j < 64; ++j) mx = fmaxf(mx, s[j]);
    } else {
#pragma unroll
      for (int j = 0; j < 64; ++j) {
        const int key = half * 64 + j;
        if (key >= seq || (causal && key > row)) s[j] = -INFINITY;  // mask (transformer.py:433-434)
        mx = fmaxf(mx, s[j]);
      }
    }
    red[half * 128 + row] = mx;
    __syncthreads();
    mx = fmaxf(red[row], red[128 + row]);
    const float c = __fmul_rn(scale, 1.4426950408889634f);
    const float mxc = __fmul_rn(mx, c);
    // branch-free: masked scores give 2^-inf = 0; four partial sums for ILP
    float sp[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
    for (int j = 0; j < 64; ++j) {
      const float e = ex2_approx_f(__fmaf_rn(s[j], c, -mxc));
      s[j] = e;
      sp[j & 3] = __fadd_rn(sp[j & 3], e);
    }
    float sum = __fadd_rn(__fadd_rn(sp[0], sp[1]), __fadd_rn(sp[2], sp[3]));
    __syncthreads();
    red[half * 128 + row] = sum;
    __syncthreads();
    sum = __fadd_rn(red[row], red[128 + row]);
    // P is left unnormalised (entries in [0, 1]); the 1 / sum is applied to the
    // 64 outputs of the row instead of its 128 probabilities
    const float inv_sum = __frcp_rn(sum);
#pragma unroll
    for (int c2 = 0; c2 < 2; ++c2) {
      float hi[32], lo[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) split_tf32(s[32 * c2 + j], hi[j], lo[j]);
      const uint32_t ta = tmem + ((uint32_t)(quarter * 32) << 16) + half * 64 + 32 * c2;
      tmem_st_32x32b_x32(ta, hi);
      tmem_st_32x32b_x32(ta + 128, lo);
    }
    tmem_st_wait();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (tr && it < 8) tr[it * 8 + 4] = gtime();

    // ---- O = P V (3-term split), A = P from TMEM, N = 64 -> TMEM [256,320) ----
    if (warp == 0) {
      const uint32_t idesc = make_idesc_tf32(128, kAttD, 0);
      const uint64_t dVh = make_sw128_desc(smem_u32(sVh)), dVl = make_sw128_desc(smem_u32(sVl));
#pragma unroll
      for (int t3 = 0; t3 < 3; ++t3)
#pragma unroll
        for (int ks = 0; ks < kAttT / 8; ++ks) {
          const int kb = 32 * ks;
          const uint64_t boff = (uint64_t)(((kb >> 7) * kAttD * 128 + (kb & 127)) >> 4);
          mma_tf32_ts_elect(tmem + 256, tmem + (t3 == 2 ? 128 : 0) + 8 * ks, (t3 == 1 ? dVl : dVh) + boff,
                            idesc, (t3 | ks) != 0);
        }
      mma_commit_elect(&bar[3]);
    }
    mbar_wait(&bar[3], ph);
    tc_fence_after();
    if (tr && it < 8) tr[it * 8 + 5] = gtime();
    {
      uint32_t r0[32];
      tmem_ld_32x32b_x32(tmem + ((uint32_t)(quarter * 32) << 16) + 256 + half * 32, r0);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 32; ++j) r0[j] = __float_as_uint(__fmul_rn(__uint_as_float(r0[j]), inv_sum));
      if (tma_store) {
        // stage O in lo(K) (dead after S) as two [128 rows x 32 cols] SWIZZLE_128B
        // boxes; one bulk tensor store per box drains while the next head runs
        uint8_t* st = sKl + half * (kRegion / 2) + row * 128;
#pragma unroll
        for (int c = 0; c < 8; ++c)
          *reinterpret_cast<uint4*>(st + ((c ^ (row & 7)) << 4)) =
              make_uint4(r0[4 * c], r0[4 * c + 1], r0[4 * c + 2], r0[4 * c + 3]);
      } else if (row < seq) {
        float* dst = ctx + ((int64_t)b * seq + row) * ld_ctx + h * kAttD + half * 32;
#pragma unroll
        for (int j = 0; j < 32; j += 4)
          *reinterpret_cast<float4*>(dst + j) =
              make_float4(__uint_as_float(r0[j]), __uint_as_float(r0[j + 1]),
                          __uint_as_float(r0[j + 2]), __uint_as_float(r0[j + 3]));
      }
    }
    if (tma_store) fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();  // TMEM / smem of this head are free for the next one
    tc_fence_after();
    if (tma_store && tid == 0) {
      tma_store_2d(&tmc, sKl, h * kAttD, b * seq);
      tma_store_2d(&tmc, sKl + kRegion / 2, h * kAttD + 32, b * seq);
      bulk_commit();
    }
    if (tr && it < 8) tr[it * 8 + 6] = gtime();
  }
  if (tma_store && tid == 0) bulk_wait0();  // ctx stores complete before exit
  if (warp == 0) tmem_dealloc(tmem, 512);
}


// ---------------------------------------------------------------------------
// ---------------------------------------------------------------------------
// fp16 two-term variant (default for seq <= 128).  Every operand tile is scaled
// by a power of two so its max lands in [2^14, 2^15) and split as
// hi = f16(x'), lo = f16(x' - hi) (22 significant bits; products hi*hi + hi*lo +
// lo*hi, relative error ~2^-21 like the 3xTF32 kernel), and the six MMAs run as
// tcgen05 kind::f16 — twice the kind::tf32 rate, with half the shared-memory
// bytes per operand.  P (in [0, 1]) is scaled by 2^15.  The scales are exact
// powers of two, folded into the softmax exponent (S) and the output (O).
//   smem: raw Q | raw K | raw V (TMA, f32) | K hi | K lo (f16, K-major SW128) |
//         2 x (V^T hi | V^T lo) (f16, 2 atoms of [64 x 128 B]) | O staging (f32)
//   TMEM (256 cols): S [0,128) -> P hi [0,64) / P lo [64,128) (f16x2), O [128,192),
//         Q hi [192,224), Q lo [224,256) (f16x2)
// Software pipeline per CTA: split(h+1) (CUDA cores, smem) runs while the tensor
// core computes P V of head h (V^T double-buffered), and S(h+1) is issued before
// O(h) is read out.  The raw tiles are consumed by the split, so the loads of
// head h+2 go out during split(h+1).
// ---------------------------------------------------------------------------
constexpr int kH16 = 128 * 64 * 2;                    // one f16 operand tile: 16 KB
constexpr int kAtt16Smem = 3 * kRegion + 6 * kH16 + kRegion + 64 + 3 * 8 * 4 + 2 * 128 * 4;
constexpr uint32_t kT16O = 128, kT16Q = 192;

__device__ __forceinline__ uint32_t make_idesc_f16(int M, int N) {
  return (1u << 4)  // c_format F32; a_format = b_format = F16 (0); both K-major
         | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_f16_ts_elect(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc,
                                                 uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p, e;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// x -> (hi, lo) f16 halves of the pair (a, b) packed low = a, high = b
__device__ __forceinline__ void split_f16x2(float a, float b, uint32_t& hi, uint32_t& lo) {
  const __half2 h = __floats2half2_rn(a, b);
  const float2 hf = __half22float2(h);
  const __half2 l = __floats2half2_rn(__fsub_rn(a, hf.x), __fsub_rn(b, hf.y));
  hi = *reinterpret_cast<const uint32_t*>(&h);
  lo = *reinterpret_cast<const uint32_t*>(&l);
}
// power-of-two factor f with max * f in [2^14, 2^15) (clamped to normal range)
__device__ __forceinline__ float pow2_scale_for(uint32_t max_bits) {
  const int E = (int)((max_bits >> 23) & 0xFF);
  int F = 268 - E;
  F = F < 1 ? 1 : (F > 254 ? 254 : F);
  return __uint_as_float((uint32_t)F << 23);
}
__device__ __forceinline__ float pow2_inv(float f) {  // exact 1/f for a power of two
  return __uint_as_float((uint32_t)(254 - (int)(__float_as_uint(f) >> 23)) << 23);
}
__device__ __forceinline__ void tmem_st_32x32b_x16(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
      "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}
__device__ __forceinline__ void tmem_st_32x32b_x32u(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
      "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]),
      "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]),
      "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}

__global__ void __launch_bounds__(256, 1)
    attention_f16_kernel(const __grid_constant__ CUtensorMap tm, int seq, int heads, int dmodel, int causal,
                         float scale, float* __restrict__ ctx, int64_t ld_ctx, int nheads_total,
                         unsigned long long* __restrict__ trace, const __grid_constant__ CUtensorMap tmc,
                         int tma_store) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* sQ = sm;
  uint8_t* sK = sm + kRegion;
  uint8_t* sV = sm + 2 * kRegion;
  uint8_t* sKh = sm + 3 * kRegion;
  uint8_t* sKl = sKh + kH16;
  uint8_t* sVT = sKl + kH16;  // [2 buffers][hi | lo]
  uint8_t* sO = sVT + 4 * kH16;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sO + kRegion);  // raw, -, S, O
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 4);
  uint32_t* rmax = reinterpret_cast<uint32_t*>(bar + 5);     // [8 warps][3]
  float* red = reinterpret_cast<float*>(rmax + 24);          // [2][128] row partials

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    if (smem_u32(sm) & 1023) __trap();
    prefetch_tmap(&tm);
    for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(tslot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  const int quarter = warp & 3, half = warp >> 2;
  const int row = quarter * 32 + lane;
  const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;

  auto issue_raw = [&](int hd) {
    const int b = hd / heads, h = hd % heads;
    mbar_arrive_expect_tx(&bar[0], 6 * 128 * 128);  // 3 tiles x 2 boxes x 16 KB
#pragma unroll
    for (int part = 0; part < 3; ++part)
#pragma unroll
      for (int j = 0; j < 2; ++j)
        tma_load_2d(sm + part * kRegion + j * (kRegion / 2), &tm, &bar[0], part * dmodel + h * kAttD + 32 * j,
                    b * seq);
  };

  // raw tiles of head hd (landed) -> Q hi/lo in TMEM, K hi/lo and V^T hi/lo (buffer vb)
  // in smem; returns the head's three power-of-two scales.  Issues the raw loads
  // of head hd_after as soon as every thread has read the raw tiles.
  auto split = [&](int hd_after, int vb, float& fq, float& fk, float& fv) {
    float q[32], k[32], v[32];
    {
      const uint8_t* qr = sQ + half * (kRegion / 2) + row * 128;
      const uint8_t* kr = sK + half * (kRegion / 2) + row * 128;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const float4 a = *reinterpret_cast<const float4*>(qr + ((c ^ (row & 7)) << 4));
        const float4 bb = *reinterpret_cast<const float4*>(kr + ((c ^ (row & 7)) << 4));
        q[4 * c] = a.x, q[4 * c + 1] = a.y, q[4 * c + 2] = a.z, q[4 * c + 3] = a.w;
        k[4 * c] = bb.x, k[4 * c + 1] = bb.y, k[4 * c + 2] = bb.z, k[4 * c + 3] = bb.w;
      }
    }
    const int vd = tid & 63, vtb = tid >> 6;  // V^T row (head dim) and 32-token block
    {
      const uint8_t* vc = sV + (vd >> 5) * (kRegion / 2) + (vd & 3) * 4;
      const int jc = (vd & 31) >> 2;
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const int t = 32 * vtb + i;
        v[i] = *reinterpret_cast<const float*>(vc + t * 128 + ((jc ^ (t & 7)) << 4));
      }
    }
    uint32_t mq = 0, mk = 0, mv = 0;
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      mq = max(mq, __float_as_uint(q[i]) & 0x7fffffffu);
      mk = max(mk, __float_as_uint(k[i]) & 0x7fffffffu);
      mv = max(mv, __float_as_uint(v[i]) & 0x7fffffffu);
    }
    mq = __reduce_max_sync(0xffffffffu, mq);
    mk = __reduce_max_sync(0xffffffffu, mk);
    mv = __reduce_max_sync(0xffffffffu, mv);
    __syncthreads();  // rmax of the previous split has been read by everyone
    if (lane == 0) rmax[warp * 3] = mq, rmax[warp * 3 + 1] = mk, rmax[warp * 3 + 2] = mv;
    __syncthreads();  // also: every thread's raw reads are done -> the next head may land
    if (tid == 0 && hd_after < nheads_total) issue_raw(hd_after);
    {
      const uint32_t a = lane < 8 ? rmax[lane * 3] : 0u, bq = lane < 8 ? rmax[lane * 3 + 1] : 0u,
                     cq = lane < 8 ? rmax[lane * 3 + 2] : 0u;
      mq = __reduce_max_sync(0xffffffffu, a);
      mk = __reduce_max_sync(0xffffffffu, bq);
      mv = __reduce_max_sync(0xffffffffu, cq);
    }
    fq = pow2_scale_for(mq), fk = pow2_scale_for(mk), fv = pow2_scale_for(mv);
    {
      uint32_t hi[16], lo[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) split_f16x2(__fmul_rn(q[2 * j], fq), __fmul_rn(q[2 * j + 1], fq), hi[j], lo[j]);
      tmem_st_32x32b_x16(tmem + lane_base + kT16Q + 16 * half, hi);
      tmem_st_32x32b_x16(tmem + lane_base + kT16Q + 32 + 16 * half, lo);
    }
    {
      uint32_t hi[16], lo[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) split_f16x2(__fmul_rn(k[2 * j], fk), __fmul_rn(k[2 * j + 1], fk), hi[j], lo[j]);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const uint32_t off = row * 128 + ((((4 * half + c) ^ (row & 7))) << 4);
        *reinterpret_cast<uint4*>(sKh + off) = make_uint4(hi[4 * c], hi[4 * c + 1], hi[4 * c + 2], hi[4 * c + 3]);
        *reinterpret_cast<uint4*>(sKl + off) = make_uint4(lo[4 * c], lo[4 * c + 1], lo[4 * c + 2], lo[4 * c + 3]);
      }
    }
    {
      uint32_t hi[16], lo[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) split_f16x2(__fmul_rn(v[2 * j], fv), __fmul_rn(v[2 * j + 1], fv), hi[j], lo[j]);
      uint8_t* vh = sVT + vb * (2 * kH16);
      uint8_t* vl = vh + kH16;
      const uint32_t atom = (uint32_t)(vtb >> 1) * (64 * 128);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const uint32_t off = atom + vd * 128 + ((((4 * (vtb & 1) + c) ^ (vd & 7))) << 4);
        *reinterpret_cast<uint4*>(vh + off) = make_uint4(hi[4 * c], hi[4 * c + 1], hi[4 * c + 2], hi[4 * c + 3]);
        *reinterpret_cast<uint4*>(vl + off) = make_uint4(lo[4 * c], lo[4 * c + 1], lo[4 * c + 2], lo[4 * c + 3]);
      }
    }
    tmem_st_wait();
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  };
  auto issue_s = [&]() {
    if (warp == 0) {
      const uint32_t idesc = make_idesc_f16(128, 128);
      const uint64_t dKh = make_sw128_desc(smem_u32(sKh)), dKl = make_sw128_desc(smem_u32(sKl));
#pragma unroll
      for (int t3 = 0; t3 < 3; ++t3)
#pragma unroll
        for (int ks = 0; ks < kAttD / 16; ++ks)
          mma_f16_ts_elect(tmem, tmem + kT16Q + (t3 == 2 ? 32 : 0) + 8 * ks, (t3 == 1 ? dKl : dKh) + 2 * ks, idesc,
                           (t3 | ks) != 0);
      mma_commit_elect(&bar[2]);
    }
  };

  pdl_trigger();
  pdl_wait();
  // prologue: first head's split and S
  float fq = 1.0f, fk = 1.0f, fv = 1.0f;
  if ((int)blockIdx.x < nheads_total) {
    if (tid == 0) issue_raw(blockIdx.x);
    mbar_wait(&bar[0], 0);
    split((int)blockIdx.x + (int)gridDim.x, 0, fq, fk, fv);
    issue_s();
  }
  int it = 0;
  unsigned long long* tr = (trace && tid == 0) ? trace + (size_t)blockIdx.x * 64 : nullptr;
  for (int hd = blockIdx.x; hd < nheads_total; hd += gridDim.x, ++it) {
    const uint32_t ph = it & 1;
    if (tr && it < 8) tr[it * 8 + 0] = gtime();
    const int nxt = hd + gridDim.x;
    const int b = hd / heads, h = hd % heads;
    const float cfq = fq, cfk = fk, cfv = fv;  // this head's scales (split(nxt) overwrites)
    mbar_wait(&bar[2], ph);
    tc_fence_after();
    if (tr && it < 8) tr[it * 8 + 1] = gtime();

    // ---- softmax: S' from TMEM; P' = 2^15 exp(.) as f16 hi / lo back into TMEM ----
    float s[64];
    {
      uint32_t r0[32], r1[32];
      const uint32_t ta = tmem + lane_base + half * 64;
      tmem_ld_32x32b_x32(ta, r0);
      tmem_ld_32x32b_x32(ta + 32, r1);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        s[j] = __uint_as_float(r0[j]);
        s[32 + j] = __uint_as_float(r1[j]);
      }
    }
    float mx = -INFINITY;
    if (seq == kAttT && !causal) {
#pragma unroll
      for (int j = 0; j < 64; ++j) mx = fmaxf(mx, s[j]);
    } else {
#pragma unroll
      for (int j = 0; j < 64; ++j) {
        const int key = half * 64 + j;
        if (key >= seq || (causal && key > row)) s[j] = -INFINITY;  // mask (transformer.py:433-434)
        mx = fmaxf(mx, s[j]);
      }
    }
    red[half * 128 + row] = mx;
    __syncthreads();
    mx = fmaxf(red[row], red[128 + row]);
    // exp(inv (s - max)) with s = S' / (fq fk): c = inv log2(e) / (fq fk), exact powers of two
    const float c = __fmul_rn(__fmul_rn(__fmul_rn(scale, 1.4426950408889634f), pow2_inv(cfq)), pow2_inv(cfk));
    const float mxc = __fsub_rn(__fmul_rn(mx, c), 15.0f);  // P' = 2^15 exp(.): +15 in the exponent
    // row sum: per 32-key quarter four interleaved partials ((p0 + p1) + (p2 + p3)),
    // the two quarters of this half added, then the halves ((q0 + q1) + (q2 + q3));
    // qkv_attention_kernel (16 compute warps, 32 keys per thread) sums in this order
    float qsum[2];
#pragma unroll
    for (int qq = 0; qq < 2; ++qq) {
      float sp[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const float e = ex2_approx_f(__fmaf_rn(s[32 * qq + j], c, -mxc));
        s[32 * qq + j] = e;
        sp[j & 3] = __fadd_rn(sp[j & 3], e);
      }
      qsum[qq] = __fadd_rn(__fadd_rn(sp[0], sp[1]), __fadd_rn(sp[2], sp[3]));
    }
    float sum = __fadd_rn(qsum[0], qsum[1]);
    __syncthreads();
    red[half * 128 + row] = sum;
    __syncthreads();
    sum = __fadd_rn(red[row], red[128 + row]);
    // O = (P' V') / (fv sum'), sum' = 2^15 sum
    const float oscale = __fmul_rn(__frcp_rn(sum), pow2_inv(cfv));
    {
      uint32_t hi[32], lo[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) split_f16x2(s[2 * j], s[2 * j + 1], hi[j], lo[j]);
      tmem_st_32x32b_x32u(tmem + lane_base + 32 * half, hi);
      tmem_st_32x32b_x32u(tmem + lane_base + 64 + 32 * half, lo);
    }
    tmem_st_wait();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (tr && it < 8) tr[it * 8 + 2] = gtime();

    // ---- O' = P' V' (3 terms), A = P' from TMEM, B = V'^T buffer it & 1 ----
    if (warp == 0) {
      const uint32_t idesc = make_idesc_f16(128, kAttD);
      const uint8_t* vh = sVT + (it & 1) * (2 * kH16);
      const uint64_t dVh = make_sw128_desc(smem_u32(vh)), dVl = make_sw128_desc(smem_u32(vh + kH16));
#pragma unroll
      for (int t3 = 0; t3 < 3; ++t3)
#pragma unroll
        for (int ks = 0; ks < kAttT / 16; ++ks) {
          const uint64_t boff = (uint64_t)(((ks >> 2) * (64 * 128) + (ks & 3) * 32) >> 4);
          mma_f16_ts_elect(tmem + kT16O, tmem + (t3 == 2 ? 64 : 0) + 8 * ks, (t3 == 1 ? dVl : dVh) + boff, idesc,
                           (t3 | ks) != 0);
        }
      mma_commit_elect(&bar[3]);
    }
    // ---- the next head's split runs while the tensor core computes P V ----
    if (nxt < nheads_total) {
      mbar_wait(&bar[0], (it + 1) & 1);
      split(nxt + (int)gridDim.x, (it + 1) & 1, fq, fk, fv);
    }
    if (tr && it < 8) tr[it * 8 + 3] = gtime();
    mbar_wait(&bar[3], ph);
    tc_fence_after();
    if (nxt < nheads_total) issue_s();  // P of this head is consumed: S of the next may overwrite it
    if (tr && it < 8) tr[it * 8 + 4] = gtime();
    {
      uint32_t r0[32];
      tmem_ld_32x32b_x32(tmem + lane_base + kT16O + half * 32, r0);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 32; ++j) r0[j] = __float_as_uint(__fmul_rn(__uint_as_float(r0[j]), oscale));
      if (tma_store) {
        if (it > 0) {  // the previous head's O store must have read the staging buffer
          if (tid == 0) bulk_wait_read0();
          __syncthreads();
        }
        uint8_t* st = sO + half * (kRegion / 2) + row * 128;
#pragma unroll
        for (int cc = 0; cc < 8; ++cc)
          *reinterpret_cast<uint4*>(st + ((cc ^ (row & 7)) << 4)) =
              make_uint4(r0[4 * cc], r0[4 * cc + 1], r0[4 * cc + 2], r0[4 * cc + 3]);
      } else if (row < seq) {
        float* dst = ctx + ((int64_t)b * seq + row) * ld_ctx + h * kAttD + half * 32;
#pragma unroll
        for (int j = 0; j < 32; j += 4)
          *reinterpret_cast<float4*>(dst + j) =
              make_float4(__uint_as_float(r0[j]), __uint_as_float(r0[j + 1]), __uint_as_float(r0[j + 2]),
                          __uint_as_float(r0[j + 3]));
      }
    }
    if (tma_store) fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (tma_store && tid == 0) {
      tma_store_2d(&tmc, sO, h * kAttD, b * seq);
      tma_store_2d(&tmc, sO + kRegion / 2, h * kAttD + 32, b * seq);
      bulk_commit();
    }
    if (tr && it < 8) tr[it * 8 + 5] = gtime(), tr[it * 8 + 6] = gtime();
  }
  if (tma_store && tid == 0) bulk_wait0();
  if (warp == 0) tmem_dealloc(tmem, 256);
}

// ---------------------------------------------------------------------------
// Long sequences (seq > 128, head_dim 64: GPT-3 350M prefill) with the fp16
// two-term scheme of attention_f16_kernel and an online softmax over 128-key
// blocks.  Work items are (sequence, head, 128-query block), heaviest causal
// blocks first; a CTA walks the key blocks of its items as one flat sequence of
// steps with the same software pipeline (the split of step j+1 on the CUDA
// cores runs while the tensor core computes P V of step j).  Q's hi / lo stay in
// TMEM for all key blocks of an item; K and V get a power-of-two scale per
// block (fk_j, fv_j), folded exactly into the softmax exponent (S) and into the
// running O; P is split with a per-row, per-block power of two that puts the
// block's largest p in [2^14, 2^15) (a block far below the running max keeps its
// precision).  Before step j's P V, O is rescaled in TMEM by corr_j and the ratio
// of the two blocks' P and V scales, so it always carries the current block's.
// Replaces the 3xTF32 kernel (attention_long_kernel, kept under ZQ_ATT_LONG_TF32=1):
// twice the MMA rate and half the operand bytes per term.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256, 1)
    attention_f16_long_kernel(const __grid_constant__ CUtensorMap tm, int seq, int heads, int dmodel, int causal,
                              float scale, float* __restrict__ ctx, int64_t ld_ctx, int nbh, int nq) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* sQ = sm;
  uint8_t* sK = sm + kRegion;
  uint8_t* sV = sm + 2 * kRegion;
  uint8_t* sKh = sm + 3 * kRegion;
  uint8_t* sKl = sKh + kH16;
  uint8_t* sVT = sKl + kH16;  // [2 buffers][hi | lo]
  uint8_t* sO = sVT + 4 * kH16;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sO + kRegion);  // raw, -, S, O
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 4);
  uint32_t* rmax = reinterpret_cast<uint32_t*>(bar + 5);     // [8 warps][3]
  float* red = reinterpret_cast<float*>(rmax + 24);          // [2][128] row partials
  (void)sO;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    if (smem_u32(sm) & 1023) __trap();
    prefetch_tmap(&tm);
    for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(tslot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  const int quarter = warp & 3, half = warp >> 2;
  const int row = quarter * 32 + lane;
  const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
  const int nitems = nbh * nq;

  // item -> (b, h, qb), the heaviest causal query blocks first; nk key blocks
  auto decode = [&](int item, int& b, int& h, int& qb) {
    qb = nq - 1 - item / nbh;
    const int bh = item % nbh;
    b = bh / heads;
    h = bh % heads;
  };
  auto nkeys = [&](int qb) { return causal ? qb + 1 : nq; };
  // the step after (item, kb) for this CTA; item = nitems when there is none
  auto next_step = [&](int item, int kb, int& nitem, int& nkb) {
    int b, h, qb;
    decode(item, b, h, qb);
    if (kb + 1 < nkeys(qb)) {
      nitem = item, nkb = kb + 1;
    } else {
      nitem = item + (int)gridDim.x, nkb = 0;
    }
  };
  auto issue_raw = [&](int item, int kb) {
    int b, h, qb;
    decode(item, b, h, qb);
    mbar_arrive_expect_tx(&bar[0], (kb == 0 ? 6 : 4) * 128 * 128);
#pragma unroll
    for (int part = 0; part < 3; ++part) {
      if (part == 0 && kb != 0) continue;  // Q stays in TMEM for the item's later key blocks
      const int r0 = b * seq + (part == 0 ? qb : kb) * kAttT;
#pragma unroll
      for (int j = 0; j < 2; ++j)
        tma_load_2d(sm + part * kRegion + j * (kRegion / 2), &tm, &bar[0], part * dmodel + h * kAttD + 32 * j, r0);
    }
  };

  // raw tiles of a step (landed) -> [Q hi/lo into TMEM when kb == 0], K hi/lo and
  // V^T hi/lo (buffer vb) in smem, with their power-of-two scales; issues the raw
  // loads of (aitem, akb) as soon as every thread has read the raw tiles
  auto split = [&](bool with_q, int aitem, int akb, int vb, float& fq, float& fk, float& fv) {
    float q[32], k[32], v[32];
    {
      const uint8_t* qr = sQ + half * (kRegion / 2) + row * 128;
      const uint8_t* kr = sK + half * (kRegion / 2) + row * 128;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const float4 bb = *reinterpret_cast<const float4*>(kr + ((c ^ (row & 7)) << 4));
        k[4 * c] = bb.x, k[4 * c + 1] = bb.y, k[4 * c + 2] = bb.z, k[4 * c + 3] = bb.w;
        if (with_q) {
          const float4 a = *reinterpret_cast<const float4*>(qr + ((c ^ (row & 7)) << 4));
          q[4 * c] = a.x, q[4 * c + 1] = a.y, q[4 * c + 2] = a.z, q[4 * c + 3] = a.w;
        } else {
          q[4 * c] = q[4 * c + 1] = q[4 * c + 2] = q[4 * c + 3] = 0.0f;
        }
      }
    }
    const int vd = tid & 63, vtb = tid >> 6;
    {
      const uint8_t* vc = sV + (vd >> 5) * (kRegion / 2) + (vd & 3) * 4;
      const int jc = (vd & 31) >> 2;
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const int t = 32 * vtb + i;
        v[i] = *reinterpret_cast<const float*>(vc + t * 128 + ((jc ^ (t & 7)) << 4));
      }
    }
    uint32_t mq = 0, mk = 0, mv = 0;
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      mq = max(mq, __float_as_uint(q[i]) & 0x7fffffffu);
      mk = max(mk, __float_as_uint(k[i]) & 0x7fffffffu);
      mv = max(mv, __float_as_uint(v[i]) & 0x7fffffffu);
    }
    mq = __reduce_max_sync(0xffffffffu, mq);
    mk = __reduce_max_sync(0xffffffffu, mk);
    mv = __reduce_max_sync(0xffffffffu, mv);
    __syncthreads();
    if (lane == 0) rmax[warp * 3] = mq, rmax[warp * 3 + 1] = mk, rmax[warp * 3 + 2] = mv;
    __syncthreads();
    if (tid == 0 && aitem < nitems) issue_raw(aitem, akb);
    {
      const uint32_t a = lane < 8 ? rmax[lane * 3] : 0u, bq = lane < 8 ? rmax[lane * 3 + 1] : 0u,
                     cq = lane < 8 ? rmax[lane * 3 + 2] : 0u;
      mq = __reduce_max_sync(0xffffffffu, a);
      mk = __reduce_max_sync(0xffffffffu, bq);
      mv = __reduce_max_sync(0xffffffffu, cq);
    }
    fk = pow2_scale_for(mk), fv = pow2_scale_for(mv);
    if (with_q) {
      fq = pow2_scale_for(mq);
      uint32_t hi[16], lo[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) split_f16x2(__fmul_rn(q[2 * j], fq), __fmul_rn(q[2 * j + 1], fq), hi[j], lo[j]);
      tmem_st_32x32b_x16(tmem + lane_base + kT16Q + 16 * half, hi);
      tmem_st_32x32b_x16(tmem + lane_base + kT16Q + 32 + 16 * half, lo);
    }
    {
      uint32_t hi[16], lo[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) split_f16x2(__fmul_rn(k[2 * j], fk), __fmul_rn(k[2 * j + 1], fk), hi[j], lo[j]);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const uint32_t off = row * 128 + ((((4 * half + c) ^ (row & 7))) << 4);
        *reinterpret_cast<uint4*>(sKh + off) = make_uint4(hi[4 * c], hi[4 * c + 1], hi[4 * c + 2], hi[4 * c + 3]);
        *reinterpret_cast<uint4*>(sKl + off) = make_uint4(lo[4 * c], lo[4 * c + 1], lo[4 * c + 2], lo[4 * c + 3]);
      }
    }
    {
      uint32_t hi[16], lo[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) split_f16x2(__fmul_rn(v[2 * j], fv), __fmul_rn(v[2 * j + 1], fv), hi[j], lo[j]);
      uint8_t* vh = sVT + vb * (2 * kH16);
      uint8_t* vl = vh + kH16;
      const uint32_t atom = (uint32_t)(vtb >> 1) * (64 * 128);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const uint32_t off = atom + vd * 128 + ((((4 * (vtb & 1) + c) ^ (vd & 7))) << 4);
        *reinterpret_cast<uint4*>(vh + off) = make_uint4(hi[4 * c], hi[4 * c + 1], hi[4 * c + 2], hi[4 * c + 3]);
        *reinterpret_cast<uint4*>(vl + off) = make_uint4(lo[4 * c], lo[4 * c + 1], lo[4 * c + 2], lo[4 * c + 3]);
      }
    }
    tmem_st_wait();
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  };
  auto issue_s = [&]() {
    if (warp == 0) {
      const uint32_t idesc = make_idesc_f16(128, 128);
      const uint64_t dKh = make_sw128_desc(smem_u32(sKh)), dKl = make_sw128_desc(smem_u32(sKl));
#pragma unroll
      for (int t3 = 0; t3 < 3; ++t3)
#pragma unroll
        for (int ks = 0; ks < kAttD / 16; ++ks)
          mma_f16_ts_elect(tmem, tmem + kT16Q + (t3 == 2 ? 32 : 0) + 8 * ks, (t3 == 1 ? dKl : dKh) + 2 * ks, idesc,
                           (t3 | ks) != 0);
      mma_commit_elect(&bar[2]);
    }
  };

  pdl_trigger();
  pdl_wait();
  float fq = 1.0f, fk = 1.0f, fv = 1.0f;
  int item = blockIdx.x, kb = 0;
  if (item < nitems) {
    if (tid == 0) issue_raw(item, 0);
    mbar_wait(&bar[0], 0);
    int ni, nk2;
    next_step(item, 0, ni, nk2);
    split(true, ni, nk2, 0, fq, fk, fv);
    issue_s();
  }
  float m2 = -INFINITY, l = 0.0f, fv_prev = 1.0f;
  int kp_prev = 0;
  for (int it = 0; item < nitems; ++it) {
    const uint32_t ph = it & 1;
    int b, h, qb;
    decode(item, b, h, qb);
    const int nk = nkeys(qb);
    const int q0 = qb * kAttT;
    int nitem, nkb;
    next_step(item, kb, nitem, nkb);
    const float cfq = fq, cfk = fk, cfv = fv;  // this step's scales (split of the next overwrites)
    mbar_wait(&bar[2], ph);
    tc_fence_after();

    // ---- online softmax of this key block ----
    float s[64];
    {
      uint32_t r0[32], r1[32];
      const uint32_t ta = tmem + lane_base + half * 64;
      tmem_ld_32x32b_x32(ta, r0);
      tmem_ld_32x32b_x32(ta + 32, r1);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        s[j] = __uint_as_float(r0[j]);
        s[32 + j] = __uint_as_float(r1[j]);
      }
    }
    float mx = -INFINITY;
    const int k0 = kb * kAttT + half * 64;
    if ((causal && kb == qb) || k0 + 64 > seq) {
#pragma unroll
      for (int j = 0; j < 64; ++j) {
        const int key = k0 + j;
        if (key >= seq || (causal && key > q0 + row)) s[j] = -INFINITY;  // transformer.py:433-434
        mx = fmaxf(mx, s[j]);
      }
    } else {
#pragma unroll
      for (int j = 0; j < 64; ++j) mx = fmaxf(mx, s[j]);
    }
    red[half * 128 + row] = mx;
    __syncthreads();
    mx = fmaxf(red[row], red[128 + row]);
    // scores in log2 units: S' * c with c = scale log2(e) / (fq fk_j) (exact powers of two)
    const float c = __fmul_rn(__fmul_rn(__fmul_rn(scale, 1.4426950408889634f), pow2_inv(cfq)), pow2_inv(cfk));
    const float mxb = __fmul_rn(mx, c);
    const float m2_new = fmaxf(m2, mxb);
    const float corr = ex2_approx_f(__fsub_rn(m2, m2_new));  // 0 on the first block (m2 = -inf)
    // P' = p * 2^(14 - kp): the row's largest p of this block (2^(mxb - m2_new)) lands
    // in [2^14, 2^15), so blocks far below the running max keep 22 significant bits
    const int kp = max((int)floorf(__fsub_rn(mxb, m2_new)), -100);
    const float mxc = __fsub_rn(m2_new, (float)(14 - kp));
    float sp[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
    for (int j = 0; j < 64; ++j) {
      const float e = ex2_approx_f(__fmaf_rn(s[j], c, -mxc));
      s[j] = e;
      sp[j & 3] = __fadd_rn(sp[j & 3], e);
    }
    float sum = __fadd_rn(__fadd_rn(sp[0], sp[1]), __fadd_rn(sp[2], sp[3]));
    __syncthreads();
    red[half * 128 + row] = sum;
    __syncthreads();
    sum = __fmul_rn(__fadd_rn(red[row], red[128 + row]), ldexpf(1.0f, kp - 14));  // true units
    l = kb == 0 ? sum : __fadd_rn(__fmul_rn(l, corr), sum);
    m2 = m2_new;
    {
      uint32_t hi[32], lo[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) split_f16x2(s[2 * j], s[2 * j + 1], hi[j], lo[j]);
      tmem_st_32x32b_x32u(tmem + lane_base + 32 * half, hi);
      tmem_st_32x32b_x32u(tmem + lane_base + 64 + 32 * half, lo);
    }
    if (kb > 0) {  // O carries 2^(14-kp) fv of the previous block: rescale by corr * 2^(kp' - kp) fv_j / fv_{j-1}
      const float f = __fmul_rn(__fmul_rn(__fmul_rn(corr, cfv), pow2_inv(fv_prev)), ldexpf(1.0f, kp_prev - kp));
      uint32_t r0[32];
      const uint32_t ta = tmem + lane_base + kT16O + half * 32;
      tmem_ld_32x32b_x32(ta, r0);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 32; ++j) r0[j] = __float_as_uint(__fmul_rn(__uint_as_float(r0[j]), f));
      tmem_st_32x32b_x32u(ta, r0);
    }
    fv_prev = cfv;
    kp_prev = kp;
    tmem_st_wait();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();

    // ---- O' += P' V' (3 terms), A = P' from TMEM, B = V'^T buffer it & 1 ----
    if (warp == 0) {
      const uint32_t idesc = make_idesc_f16(128, kAttD);
      const uint8_t* vh = sVT + (it & 1) * (2 * kH16);
      const uint64_t dVh = make_sw128_desc(smem_u32(vh)), dVl = make_sw128_desc(smem_u32(vh + kH16));
#pragma unroll
      for (int t3 = 0; t3 < 3; ++t3)
#pragma unroll
        for (int ks = 0; ks < kAttT / 16; ++ks) {
          const uint64_t boff = (uint64_t)(((ks >> 2) * (64 * 128) + (ks & 3) * 32) >> 4);
          mma_f16_ts_elect(tmem + kT16O, tmem + (t3 == 2 ? 64 : 0) + 8 * ks, (t3 == 1 ? dVl : dVh) + boff, idesc,
                           (kb | t3 | ks) != 0);
        }
      mma_commit_elect(&bar[3]);
    }
    // ---- the next step's split runs while the tensor core computes P V ----
    if (nitem < nitems) {
      mbar_wait(&bar[0], (it + 1) & 1);
      int ai, akb;
      next_step(nitem, nkb, ai, akb);
      split(nkb == 0, ai, akb, (it + 1) & 1, fq, fk, fv);
    }
    mbar_wait(&bar[3], ph);
    tc_fence_after();
    if (nitem < nitems) issue_s();  // P of this step is consumed: S of the next may overwrite it
    if (kb == nk - 1) {
      // ---- the item's output: O' / (l * 2^(14 - kp) * fv_last) ----
      const float oscale = __fmul_rn(__fmul_rn(__frcp_rn(l), pow2_inv(cfv)), ldexpf(1.0f, kp - 14));
      uint32_t r0[32];
      tmem_ld_32x32b_x32(tmem + lane_base + kT16O + half * 32, r0);
      tmem_ld_wait();
      if (q0 + row < seq) {
        float* dst = ctx + ((int64_t)b * seq + q0 + row) * ld_ctx + h * kAttD + half * 32;
#pragma unroll
        for (int j = 0; j < 32; j += 4)
          *reinterpret_cast<float4*>(dst + j) = make_float4(
              __fmul_rn(__uint_as_float(r0[j]), oscale), __fmul_rn(__uint_as_float(r0[j + 1]), oscale),
              __fmul_rn(__uint_as_float(r0[j + 2]), oscale), __fmul_rn(__uint_as_float(r0[j + 3]), oscale));
      }
      m2 = -INFINITY;
      l = 0.0f;
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    item = nitem;
    kb = nkb;
  }
  if (warp == 0) tmem_dealloc(tmem, 256);
}

// ---------------------------------------------------------------------------
// Any head_dim (multiple of 32, <= 256) and any sequence length: CUDA-core fp32
// flash attention (GPT-J 256 / NeoX 96 prefill).  A CTA takes 32 queries of one
// (sequence, head): 4 warps x 8 query rows; per block of 32 keys lane l scores key
// l against the warp's 8 rows with 16-byte loads (K rows padded by 4 floats:
// conflict-free; Q rows are warp broadcasts), the
// online softmax runs on warp shuffles, and P V accumulates into registers
// (lane l owns head-dim columns l, l+32, ...), broadcasting p per key.  fp32 FMA
// throughout (more accurate than the tensor-core paths; prefill only).
// ---------------------------------------------------------------------------
template <int DH>
__global__ void __launch_bounds__(128)
    attention_general_kernel(const float* __restrict__ qkv, int64_t ld_qkv, int seq, int heads, int causal,
                             float scale, float* __restrict__ ctx, int64_t ld_ctx) {
  constexpr int NJ = (DH + 31) / 32;  // head-dim columns per lane (the last one masked if DH % 32)
  constexpr int RW = 8;         // query rows per warp
  constexpr int QB = 4 * RW;    // query rows per CTA
  constexpr int KP = DH + 4;    // padded K row (16-byte loads stay conflict-free)
  extern __shared__ float4 smg4[];
  float* sQ = reinterpret_cast<float*>(smg4);  // [QB][DH]
  float* sK = sQ + QB * DH;                    // [32][KP]
  float* sV = sK + 32 * KP;                    // [32][DH]
  pdl_trigger();
  pdl_wait();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q0 = blockIdx.x * QB, h = blockIdx.y, b = blockIdx.z;
  const int dmodel = heads * DH;
  const float* base = qkv + (int64_t)b * seq * ld_qkv;
  for (int i = threadIdx.x; i < QB * DH / 4; i += 128) {
    const int r = i / (DH / 4), d4 = i - r * (DH / 4);
    reinterpret_cast<float4*>(sQ)[i] =
        q0 + r < seq ? *reinterpret_cast<const float4*>(base + (int64_t)(q0 + r) * ld_qkv + h * DH + 4 * d4)
                     : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  float m[RW], l[RW], o[RW][NJ];
#pragma unroll
  for (int r = 0; r < RW; ++r) {
    m[r] = -INFINITY;
    l[r] = 0.0f;
#pragma unroll
    for (int j = 0; j < NJ; ++j) o[r][j] = 0.0f;
  }
  const int qlast = min(seq, q0 + QB) - 1;
  const int kend = causal ? qlast + 1 : seq;
  const float c = __fmul_rn(scale, 1.4426950408889634f);
  const float4* qrow = reinterpret_cast<const float4*>(sQ + warp * RW * DH);
  for (int k0 = 0; k0 < kend; k0 += 32) {
    __syncthreads();  // previous block's K / V fully consumed (and sQ written, first pass)
    for (int i = threadIdx.x; i < 32 * DH / 4; i += 128) {
      const int r = i / (DH / 4), d4 = i - r * (DH / 4);
      const bool ok = k0 + r < seq;
      const float* row = base + (int64_t)(k0 + r) * ld_qkv + h * DH + 4 * d4;
      *reinterpret_cast<float4*>(sK + r * KP + 4 * d4) =
          ok ? *reinterpret_cast<const float4*>(row + dmodel) : make_float4(0.f, 0.f, 0.f, 0.f);
      *reinterpret_cast<float4*>(sV + r * DH + 4 * d4) =
          ok ? *reinterpret_cast<const float4*>(row + 2 * dmodel) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    __syncthreads();
    const int key = k0 + lane;
    float sc[RW];
#pragma unroll
    for (int r = 0; r < RW; ++r) sc[r] = 0.0f;
    const float4* krow = reinterpret_cast<const float4*>(sK + lane * KP);
#pragma unroll 4
    for (int d4 = 0; d4 < DH / 4; ++d4) {
      const float4 kv = krow[d4];
#pragma unroll
      for (int r = 0; r < RW; ++r) {
        const float4 qv = qrow[r * (DH / 4) + d4];
        sc[r] = __fmaf_rn(qv.x, kv.x, sc[r]);
        sc[r] = __fmaf_rn(qv.y, kv.y, sc[r]);
        sc[r] = __fmaf_rn(qv.z, kv.z, sc[r]);
        sc[r] = __fmaf_rn(qv.w, kv.w, sc[r]);
      }
    }
    float p[RW];
#pragma unroll
    for (int r = 0; r < RW; ++r) {
      const int q = q0 + warp * RW + r;
      const bool masked = key >= seq || (causal && key > q);
      const float v = masked ? -INFINITY : sc[r];
      float bm = v;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, off));
      const float mn = fmaxf(m[r], bm);
      // rows with every key so far masked keep m = -inf: nothing to rescale
      const float corr = mn == -INFINITY ? 1.0f : ex2_approx_f(__fmul_rn(__fsub_rn(m[r], mn), c));
      p[r] = mn == -INFINITY ? 0.0f : ex2_approx_f(__fmul_rn(__fsub_rn(v, mn), c));
      float ps = p[r];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) ps = __fadd_rn(ps, __shfl_xor_sync(0xffffffffu, ps, off));
      l[r] = __fmaf_rn(l[r], corr, ps);
      m[r] = mn;
#pragma unroll
      for (int j = 0; j < NJ; ++j) o[r][j] = __fmul_rn(o[r][j], corr);
    }
    const int nk = min(32, kend - k0);
    for (int kk = 0; kk < nk; ++kk) {
      float pk[RW];
#pragma unroll
      for (int r = 0; r < RW; ++r) pk[r] = __shfl_sync(0xffffffffu, p[r], kk);
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        if (DH % 32 != 0 && lane + 32 * j >= DH) continue;
        const float vv = sV[kk * DH + lane + 32 * j];
#pragma unroll
        for (int r = 0; r < RW; ++r) o[r][j] = __fmaf_rn(pk[r], vv, o[r][j]);
      }
    }
  }
#pragma unroll
  for (int r = 0; r < RW; ++r) {
    const int q = q0 + warp * RW + r;
    if (q >= seq) continue;
    const float inv = __frcp_rn(l[r]);
    float* dst = ctx + ((int64_t)b * seq + q) * ld_ctx + h * DH;
#pragma unroll
    for (int j = 0; j < NJ; ++j)
      if (DH % 32 == 0 || lane + 32 * j < DH) dst[lane + 32 * j] = __fmul_rn(o[r][j], inv);
  }
}

template <int DH>
static cudaError_t launch_att_general(const float* qkv, int64_t ld_qkv, int batch, int seq, int heads, int causal,
                                      float scale, float* ctx, int64_t ld_ctx, cudaStream_t st) {
  const size_t smem = sizeof(float) * (32 * DH + 32 * (DH + 4) + 32 * DH);
  static ZqDeviceOnce attr_once;
  attr_once([&](int) {
    cudaFuncSetAttribute(attention_general_kernel<DH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  });
  return launch_kernel(attention_general_kernel<DH>, dim3((unsigned)((seq + 31) / 32), (unsigned)heads, (unsigned)batch),
                       dim3(128), smem, st, 1, qkv, ld_qkv, seq, heads, causal, scale, ctx, ld_ctx);
}

// Long sequences (seq > 128, head_dim 64): flash-attention style online softmax
// over 128-key blocks.  Work item = (sequence, head, 128-query block), heaviest
// causal blocks first; persistent CTAs.  TMEM: S [0,128), P hi [128,256),
// P lo [256,384), O [384,448).  Per key block: K (and on the first block Q) land
// by TMA, lo(K) / V^T are split in smem, S = Q K^T (3xTF32), the row max / sum
// are carried online (O in TMEM is rescaled by exp(m_old - m_new) before the
// block's P.V accumulates into it), and the next block's V / K loads are issued
// as soon as their smem is consumed.  O / l is written at the end.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256, 1)
    attention_long_kernel(const __grid_constant__ CUtensorMap tm, int seq, int heads, int dmodel,
                          int causal, float scale, float* __restrict__ ctx, int64_t ld_ctx, int nbh,
                          int nq) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* sQh = sm;
  uint8_t* sQl = sm + kRegion;
  uint8_t* sKh = sm + 2 * kRegion;
  uint8_t* sKl = sm + 3 * kRegion;
  uint8_t* sV = sm + 4 * kRegion;
  uint8_t* sVh = sm + 5 * kRegion;
  uint8_t* sVl = sm + 6 * kRegion;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 7 * kRegion);  // Q, K, V, S, O
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 5);
  float* red = reinterpret_cast<float*>(bar + 6);  // [2][128]

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nitems = nbh * nq;
  if (tid == 0) {
    if (smem_u32(sm) & 1023) __trap();
    prefetch_tmap(&tm);
    for (int i = 0; i < 5; ++i) mbar_init(&bar[i], 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  const uint32_t tS = tmem, tPh = tmem + 128, tPl = tmem + 256, tO = tmem + 384;
  const int quarter = warp & 3, half = warp >> 2;
  const int row = quarter * 32 + lane;
  uint32_t phQ = 0, phK = 0, phV = 0, phS = 0, phO = 0;

  // item -> (b, h, qb): the heaviest causal query blocks first
  auto decode = [&](int item, int& b, int& h, int& qb) {
    qb = nq - 1 - item / nbh;
    const int bh = item % nbh;
    b = bh / heads;
    h = bh % heads;
  };
  auto nkeys = [&](int qb) { return causal ? qb + 1 : nq; };
  auto load_q = [&](int b, int h, int qb) {
    mbar_arrive_expect_tx(&bar[0], 2 * 128 * 128);
#pragma unroll
    for (int j = 0; j < 2; ++j)
      tma_load_2d(sQh + j * (kRegion / 2), &tm, &bar[0], h * kAttD + 32 * j, b * seq + qb * 128);
  };
  auto load_k = [&](int b, int h, int kb) {
    mbar_arrive_expect_tx(&bar[1], 2 * 128 * 128);
#pragma unroll
    for (int j = 0; j < 2; ++j)
      tma_load_2d(sKh + j * (kRegion / 2), &tm, &bar[1], dmodel + h * kAttD + 32 * j, b * seq + kb * 128);
  };
  auto load_v = [&](int b, int h, int kb) {
    mbar_arrive_expect_tx(&bar[2], 2 * 128 * 128);
#pragma unroll
    for (int j = 0; j < 2; ++j)
      tma_load_2d(sV + j * (kRegion / 2), &tm, &bar[2], 2 * dmodel + h * kAttD + 32 * j, b * seq + kb * 128);
  };

  pdl_trigger();
  pdl_wait();
  if (tid == 0 && (int)blockIdx.x < nitems) {
    int b, h, qb;
    decode(blockIdx.x, b, h, qb);
    load_q(b, h, qb);
    load_k(b, h, 0);
    load_v(b, h, 0);
  }
  for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
    int b, h, qb;
    decode(item, b, h, qb);
    const int nk = nkeys(qb);
    const int q0 = qb * 128;
    int nb = 0, nh = 0, nqb = 0;
    const int nitem = item + gridDim.x;
    if (nitem < nitems) decode(nitem, nb, nh, nqb);
    float m_run = -INFINITY, l_run = 0.0f;
    for (int kb = 0; kb < nk; ++kb) {
      const bool last = kb == nk - 1;
      // ---- lo(K) (and lo(Q) on the first block) while P.V of the previous
      //      block may still run on the tensor pipe ----
      if (kb == 0) {
        mbar_wait(&bar[0], phQ);
        phQ ^= 1;
      }
      mbar_wait(&bar[1], phK);
      phK ^= 1;
      for (int i = tid; i < (kb == 0 ? 2 : 1) * (kRegion / 16); i += 256) {
        const int part = (kb == 0) ? i / (kRegion / 16) : 1;
        const int off = (i % (kRegion / 16)) * 16;
        const float4 x = *reinterpret_cast<const float4*>(sm + 2 * part * kRegion + off);
        float4 hi, lo;
        split_tf32(x.x, hi.x, lo.x);
        split_tf32(x.y, hi.y, lo.y);
        split_tf32(x.z, hi.z, lo.z);
        split_tf32(x.w, hi.w, lo.w);
        *reinterpret_cast<float4*>(sm + (2 * part + 1) * kRegion + off) = lo;
      }
      fence_proxy_async_smem();
      tc_fence_before();
      __syncthreads();
      tc_fence_after();
      // ---- S = Q K^T (queued behind the previous P.V) ----
      if (warp == 0) {
        const uint32_t idesc = make_idesc_tf32(128, 128, 0);
        const uint64_t dQh = make_sw128_desc(smem_u32(sQh)), dQl = make_sw128_desc(smem_u32(sQl));
        const uint64_t dKh = make_sw128_desc(smem_u32(sKh)), dKl = make_sw128_desc(smem_u32(sKl));
#pragma unroll
        for (int t3 = 0; t3 < 3; ++t3)
#pragma unroll
          for (int ks = 0; ks < kAttD / 8; ++ks) {
            const int kbt = 32 * ks;
            const uint64_t aoff = (uint64_t)(((kbt >> 7) * kAttT * 128 + (kbt & 127)) >> 4);
            mma_tf32_elect(tS, (t3 == 2 ? dQl : dQh) + aoff, (t3 == 1 ? dKl : dKh) + aoff, idesc,
                           (t3 | ks) != 0);
          }
        mma_commit_elect(&bar[3]);
      }
      // ---- V^T of this block once the previous P.V no longer reads it ----
      if (kb > 0) {
        mbar_wait(&bar[4], phO);
        phO ^= 1;
        tc_fence_after();
      }
      mbar_wait(&bar[2], phV);
      phV ^= 1;
      {
        const int j = (warp & 1) * 32 + lane;
        const uint8_t* vcol = sV + (j >> 5) * (kRegion / 2) + (j & 3) * 4;
        const int jc = (j & 31) >> 2;
#pragma unroll 2
        for (int q = warp >> 1; q < kAttT / 4; q += 4) {
          float v[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int t = 4 * q + e;
            v[e] = *reinterpret_cast<const float*>(vcol + t * 128 + ((jc ^ (t & 7)) << 4));
          }
          float4 hi, lo;
          split_tf32(v[0], hi.x, lo.x);
          split_tf32(v[1], hi.y, lo.y);
          split_tf32(v[2], hi.z, lo.z);
          split_tf32(v[3], hi.w, lo.w);
          hi = make_float4(v[0], v[1], v[2], v[3]);
          const uint32_t o = (q >> 3) * (kAttD * 128) + j * 128 + (((q & 7) ^ (j & 7)) << 4);
          *reinterpret_cast<float4*>(sVh + o) = hi;
          *reinterpret_cast<float4*>(sVl + o) = lo;
        }
      }
      fence_proxy_async_smem();
      tc_fence_before();
      __syncthreads();
      tc_fence_after();
      if (tid == 0) {  // V raw is consumed: next block's (or next item's first) V
        if (!last) load_v(b, h, kb + 1);
        else if (nitem < nitems) load_v(nb, nh, 0);
      }
      mbar_wait(&bar[3], phS);
      phS ^= 1;
      tc_fence_after();
      if (tid == 0) {  // K (and after the last block, Q) are consumed
        if (!last) {
          load_k(b, h, kb + 1);
        } else if (nitem < nitems) {
          load_q(nb, nh, nqb);
          load_k(nb, nh, 0);
        }
      }
      // ---- online softmax ----
      float sv[64];
      {
        uint32_t r0[32], r1[32];
        const uint32_t ta = tS + ((uint32_t)(quarter * 32) << 16) + half * 64;
        tmem_ld_32x32b_x32(ta, r0);
        tmem_ld_32x32b_x32(ta + 32, r1);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          sv[j] = __uint_as_float(r0[j]);
          sv[32 + j] = __uint_as_float(r1[j]);
        }
      }
      float mx = -INFINITY;
      const int qrow = q0 + row;
#pragma unroll
      for (int j = 0; j < 64; ++j) {
        const int key = kb * 128 + half * 64 + j;
        float v = __fmul_rn(sv[j], scale);
        if (key >= seq || (causal && key > qrow)) v = -INFINITY;
        sv[j] = v;
        mx = fmaxf(mx, v);
      }
      red[half * 128 + row] = mx;
      __syncthreads();
      const float m_new = fmaxf(m_run, fmaxf(red[row], red[128 + row]));
      const float m_use = m_new == -INFINITY ? 0.0f : m_new;  // fully masked so far
      const float corr = ex2_approx_f(__fmul_rn(__fsub_rn(m_run, m_use), 1.4426950408889634f));
      float sum = 0.0f;
#pragma unroll
      for (int j = 0; j < 64; ++j) {
        const float e = ex2_approx_f(__fmul_rn(__fsub_rn(sv[j], m_use), 1.4426950408889634f));
        sv[j] = e;
        sum = __fadd_rn(sum, e);
      }
      __syncthreads();
      red[half * 128 + row] = sum;
      __syncthreads();
      l_run = __fadd_rn(__fmul_rn(l_run, corr), __fadd_rn(red[row], red[128 + row]));
      m_run = m_new;
#pragma unroll
      for (int c2 = 0; c2 < 2; ++c2) {
        float hi[32], lo[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) split_tf32(sv[32 * c2 + j], hi[j], lo[j]);
        const uint32_t ta = ((uint32_t)(quarter * 32) << 16) + half * 64 + 32 * c2;
        tmem_st_32x32b_x32(tPh + ta, hi);
        tmem_st_32x32b_x32(tPl + ta, lo);
      }
      if (kb > 0) {  // rescale the running O (this warp's 32 columns)
        uint32_t r0[32];
        const uint32_t ta = tO + ((uint32_t)(quarter * 32) << 16) + half * 32;
        tmem_ld_32x32b_x32(ta, r0);
        tmem_ld_wait();
        float o[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) o[j] = __fmul_rn(__uint_as_float(r0[j]), corr);
        tmem_st_32x32b_x32(ta, o);
      }
      tmem_st_wait();
      tc_fence_before();
      __syncthreads();
      tc_fence_after();
      // ---- O += P V ----
      if (warp == 0) {
        const uint32_t idesc = make_idesc_tf32(128, kAttD, 0);
        const uint64_t dVh = make_sw128_desc(smem_u32(sVh)), dVl = make_sw128_desc(smem_u32(sVl));
#pragma unroll
        for (int t3 = 0; t3 < 3; ++t3)
#pragma unroll
          for (int ks = 0; ks < kAttT / 8; ++ks) {
            const int kbt = 32 * ks;
            const uint64_t boff = (uint64_t)(((kbt >> 7) * kAttD * 128 + (kbt & 127)) >> 4);
            mma_tf32_ts_elect(tO, (t3 == 2 ? tPl : tPh) + 8 * ks, (t3 == 1 ? dVl : dVh) + boff, idesc,
                              (kb | t3 | ks) != 0);
          }
        mma_commit_elect(&bar[4]);
      }
    }
    // ---- epilogue: ctx = O / l ----
    mbar_wait(&bar[4], phO);
    phO ^= 1;
    tc_fence_after();
    {
      uint32_t r0[32];
      tmem_ld_32x32b_x32(tO + ((uint32_t)(quarter * 32) << 16) + half * 32, r0);
      tmem_ld_wait();
      const float inv_l = __frcp_rn(l_run);
      if (q0 + row < seq) {
        float* dst = ctx + ((int64_t)b * seq + q0 + row) * ld_ctx + h * kAttD + half * 32;
#pragma unroll
        for (int j = 0; j < 32; j += 4)
          *reinterpret_cast<float4*>(dst + j) = make_float4(
              __fmul_rn(__uint_as_float(r0[j]), inv_l), __fmul_rn(__uint_as_float(r0[j + 1]), inv_l),
              __fmul_rn(__uint_as_float(r0[j + 2]), inv_l), __fmul_rn(__uint_as_float(r0[j + 3]), inv_l));
      }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  }
  if (warp == 0) tmem_dealloc(tmem, 512);
}

// ---------------------------------------------------------------------------
// Fused QKV projection + attention (encoder, seq <= 128, head_dim 64).
// One CTA per (sequence, head) unit computes that unit's 128 x 192 slice of the
// W8A8 QKV linear (tokens b*seq.., weight rows {Q, K, V} x [64h, 64h+64)) with
// tcgen05 kind::i8 into TMEM, dequantizes it from TMEM exactly as the GEMM
// epilogue does (((f32(acc) * s_tok) * s_w) + b, pkg/src/lowbit/igemm.py:131-139 —
// the values zq_linear writes) straight into attention_f16_kernel's hi/lo split;
// the attention then runs as in that kernel.  The [T, 3d] f32 QKV activation never
// leaves the SM: ctx is bit-identical to zq_linear + zq_attention_f32
// (tests/test_qkv_attention_gpu.py).
//   warps 0-7: GEMM epilogue + split, attention (attention_f16_kernel's code)
//   warp 8   : TMA producer of the GEMM operands (3-stage ring)
//   warp 9   : GEMM MMA issuer
//   warp 10  : attention MMA issuer (S = Q K^T, O = P V)
//   smem: ring (3 x [A 128 x 128 B | B 192 x 128 B], 120 KB) | K hi | K lo |
//         2 x (V^T hi | V^T lo) | barriers
//   TMEM (512 cols): attention's [0, 256) + the GEMM accumulator [256, 448)
// Pipeline: the operands of unit u+1 stream in while unit u's attention runs and
// its MMAs start as soon as unit u's accumulator has been read (accfree).
// ---------------------------------------------------------------------------
constexpr int kQaStages = 3;
constexpr int kQaStageA = 128 * 128, kQaStageB = 3 * kAttD * 128;
constexpr int kQaStage = kQaStageA + kQaStageB;  // 40 KB
constexpr int kQaX = kQaStages * kQaStage;       // 120 KB
constexpr int kQaSc = 2 * 2 * 3 * kAttD * 4;      // [unit parity][scale | bias][Q | K | V][64] f32
// CW compute warps (8 or 16): TMEM lane quarter warp % 4, column part warp / 4
template <int CW>
struct QaCfg {
  static constexpr int NCQ = CW / 4;          // column parts per row
  static constexpr int KPT = 128 / NCQ;       // S columns (keys) per thread
  static constexpr int DPT = kAttD / NCQ;     // Q / K / V / O columns per thread
  static constexpr int THREADS = (CW + 3) * 32;
  static constexpr int SMEM = kQaX + 6 * kH16 + kQaSc + 128 + 16 + CW * 3 * 4 + 2 * NCQ * 128 * 4;
};
constexpr uint32_t kQaAcc = 256;

__device__ __forceinline__ void tmem_ld_32x32b_x16(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_st_32x32b_x8(uint32_t taddr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
      : "memory");
}
// n (a multiple of 8) consecutive 32-bit TMEM columns of this thread's lane
template <int N>
__device__ __forceinline__ void tmem_ld_cols(uint32_t taddr, uint32_t* r) {
#pragma unroll
  for (int c = 0; c < N; c += 16) tmem_ld_32x32b_x16(taddr + c, r + c);
}
template <int N>
__device__ __forceinline__ void tmem_st_cols(uint32_t taddr, const uint32_t* v) {
#pragma unroll
  for (int c = 0; c < N; c += 8) tmem_st_32x32b_x8(taddr + c, v + c);
}

__device__ __forceinline__ void bulk_load_1d(void* smem_dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(smem_dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

template <int CW>
__device__ __forceinline__ void compute_bar() { asm volatile("bar.sync 1, %0;" ::"n"(CW * 32) : "memory"); }
// Long waits of the producer / MMA warps: back off between polls so the waiting
// lane does not take issue slots from the compute warps on its scheduler.
__device__ __forceinline__ void mbar_wait_idle(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar), done;
  for (;;) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
        "selp.u32 %0, 1, 0, P1;\n"
        "}\n"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
    if (done) return;
    __nanosleep(128);
  }
}

template <int CW>
__global__ void __launch_bounds__(QaCfg<CW>::THREADS, 1)
    qkv_attention_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW,
                         const float* __restrict__ ts, const float* __restrict__ rs, const float* __restrict__ bias,
                         int M, int seq, int heads, int dmodel, int causal, float scale, float* __restrict__ ctx,
                         int64_t ld_ctx, int nheads_total, unsigned long long* __restrict__ trace,
                         const __grid_constant__ CUtensorMap tmc, int tma_store, int trigger_late) {
  using Cfg = QaCfg<CW>;
  constexpr int NCQ = Cfg::NCQ, KPT = Cfg::KPT, DPT = Cfg::DPT;
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* sX = sm;
  uint8_t* sKh = sm + kQaX;
  uint8_t* sKl = sKh + kH16;
  uint8_t* sVT = sKl + kH16;  // [2 buffers][hi | lo]
  float* sSc = reinterpret_cast<float*>(sVT + 4 * kH16);  // per-unit weight scales and bias
  uint64_t* bars = reinterpret_cast<uint64_t*>(sVT + 4 * kH16 + kQaSc);
  uint64_t* gfull = bars;       // [3] operand stage landed
  uint64_t* gempty = bars + 3;  // [3] operand stage consumed by the MMAs
  uint64_t* accf = bars + 6;    // GEMM accumulator complete
  uint64_t* accfree = bars + 7; // accumulator read by the epilogue
  uint64_t* barS = bars + 8;
  uint64_t* barO = bars + 9;
  uint64_t* scf = bars + 10;    // [2] unit parity: scales and bias landed
  uint64_t* scfree = bars + 12; // [2] unit parity: scales and bias read by epi_split
  uint64_t* qkr = bars + 14;    // Q, K, V^T of the next unit split (S may be issued)
  uint64_t* prdy = bars + 15;   // P written (P V may be issued)
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 16);
  uint32_t* rmax = reinterpret_cast<uint32_t*>(bars + 18);  // [CW warps][3]
  float* redm = reinterpret_cast<float*>(rmax + CW * 3);    // [NCQ][128] row partial maxima
  float* reds = redm + NCQ * 128;                           // [NCQ][128] row partial sums

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nkb = dmodel / 128;
  if (tid == 0) {
    if (smem_u32(sm) & 1023) __trap();
    prefetch_tmap(&tmX);
    prefetch_tmap(&tmW);
    for (int i = 0; i < 16; ++i) mbar_init(&bars[i], 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  unsigned long long* tr = (trace && tid == 0) ? trace + (size_t)blockIdx.x * 64 : nullptr;
  if (tr) tr[0] = gtime();
  if (!(trigger_late & 1)) pdl_trigger();

  if (warp == CW) {  // ===== GEMM operand producer =====
    if (lane == 0) {
      // the unit's 192 weight-row scales and biases -> buffer u & 1 (free once
      // epi_split(u - 2) has read it)
      auto load_scales = [&](int h, int u) {
        if (u >= 2) mbar_wait_idle(&scfree[u & 1], ((u >> 1) - 1) & 1);
        float* dst = sSc + (u & 1) * (2 * 3 * kAttD);
        mbar_arrive_expect_tx(&scf[u & 1], (bias ? 2 : 1) * 3 * kAttD * 4);
#pragma unroll
        for (int part = 0; part < 3; ++part) {
          bulk_load_1d(dst + part * kAttD, rs + part * dmodel + h * kAttD, kAttD * 4, &scf[u & 1]);
          if (bias) bulk_load_1d(dst + 3 * kAttD + part * kAttD, bias + part * dmodel + h * kAttD, kAttD * 4,
                                 &scf[u & 1]);
        }
      };
      auto load_w = [&](uint8_t* st, int kb, int h, uint64_t* bar) {
#pragma unroll
        for (int part = 0; part < 3; ++part)
          tma_load_2d(st + kQaStageA + part * (kAttD * 128), &tmW, bar, kb * 128, part * dmodel + h * kAttD);
      };
      // weights and scales do not depend on the previous kernel: unit 0's first
      // stages of B go out before griddepcontrol.wait, A (the activations) after it
      const int npre = nkb < kQaStages ? nkb : kQaStages;
      if ((int)blockIdx.x < nheads_total) {
        const int h0 = (int)blockIdx.x % heads;
        load_scales(h0, 0);
        for (int kb = 0; kb < npre; ++kb) {
          mbar_arrive_expect_tx(&gfull[kb], kQaStage);
          load_w(sX + kb * kQaStage, kb, h0, &gfull[kb]);
        }
      }
      pdl_wait();
      if (tr) tr[1] = gtime();
      int kc = 0, u = 0;
      for (int hd = blockIdx.x; hd < nheads_total; hd += gridDim.x, ++u) {
        const int b = hd / heads, h = hd % heads;
        if ((trigger_late & 2) && u >= 1) mbar_wait(accfree, (u - 1) & 1);  // debug: no operand prefetch
        if (u > 0) load_scales(h, u);
        for (int kb = 0; kb < nkb; ++kb, ++kc) {
          const int s = kc % kQaStages;
          uint8_t* st = sX + s * kQaStage;
          if (u == 0 && kb < npre) {  // B already in flight
            tma_load_2d(st, &tmX, &gfull[s], kb * 128, b * seq);
            continue;
          }
          if (kc >= kQaStages) mbar_wait_idle(&gempty[s], ((kc / kQaStages) - 1) & 1);
          if (trace && kb == 0 && kc / nkb < 4) trace[(size_t)blockIdx.x * 64 + 60 + kc / nkb] = gtime();
          mbar_arrive_expect_tx(&gfull[s], kQaStage);
          tma_load_2d(st, &tmX, &gfull[s], kb * 128, b * seq);
          load_w(st, kb, h, &gfull[s]);
        }
      }
    }
    return;
  }
  if (warp == CW + 1) {  // ===== GEMM MMA issuer =====
    if (lane == 0) {
      constexpr uint32_t idesc = make_idesc_i8(128, 3 * kAttD);
      int kc = 0, u = 0;
      for (int hd = blockIdx.x; hd < nheads_total; hd += gridDim.x, ++u) {
        if (u > 0) mbar_wait_idle(accfree, (u - 1) & 1);  // the previous unit's accumulator has been read
        tc_fence_after();
        for (int kb = 0; kb < nkb; ++kb, ++kc) {
          const int s = kc % kQaStages;
          mbar_wait(&gfull[s], (kc / kQaStages) & 1);
          tc_fence_after();
          if (trace && kb == nkb - 1 && u < 4) trace[(size_t)blockIdx.x * 64 + 56 + u] = gtime();
          if (trace && kb == 0 && u < 4) trace[(size_t)blockIdx.x * 64 + 52 + u] = gtime();
          const uint32_t a_addr = smem_u32(sX + s * kQaStage);
          const uint32_t b_addr = a_addr + kQaStageA;
#pragma unroll
          for (int k = 0; k < 4; ++k)
            mma_i8(tmem + kQaAcc, make_sw128_desc(a_addr + k * 32), make_sw128_desc(b_addr + k * 32), idesc,
                   (kb | k) != 0);
          mma_commit(&gempty[s]);
        }
        mma_commit(accf);
      }
    }
    return;
  }

  if (warp == CW + 2) {  // ===== attention MMA issuer: S = Q K^T, O = P V (3-term f16 splits) =====
    int it = 0;
    for (int hd = blockIdx.x; hd < nheads_total; hd += gridDim.x, ++it) {
      mbar_wait_idle(qkr, it & 1);                         // Q, K, V^T of unit it split
      if (it > 0) mbar_wait_idle(barO, (it - 1) & 1);      // P of unit it - 1 consumed
      tc_fence_after();
      {
        const uint32_t idesc = make_idesc_f16(128, 128);
        const uint64_t dKh = make_sw128_desc(smem_u32(sKh)), dKl = make_sw128_desc(smem_u32(sKl));
#pragma unroll
        for (int t3 = 0; t3 < 3; ++t3)
#pragma unroll
          for (int ks = 0; ks < kAttD / 16; ++ks)
            mma_f16_ts_elect(tmem, tmem + kT16Q + (t3 == 2 ? 32 : 0) + 8 * ks, (t3 == 1 ? dKl : dKh) + 2 * ks,
                             idesc, (t3 | ks) != 0);
        mma_commit_elect(barS);
      }
      mbar_wait_idle(prdy, it & 1);                        // P of unit it written
      tc_fence_after();
      {
        const uint32_t idesc = make_idesc_f16(128, kAttD);
        const uint8_t* vh = sVT + (it & 1) * (2 * kH16);
        const uint64_t dVh = make_sw128_desc(smem_u32(vh)), dVl = make_sw128_desc(smem_u32(vh + kH16));
#pragma unroll
        for (int t3 = 0; t3 < 3; ++t3)
#pragma unroll
          for (int ks = 0; ks < kAttT / 16; ++ks) {
            const uint64_t boff = (uint64_t)(((ks >> 2) * (64 * 128) + (ks & 3) * 32) >> 4);
            mma_f16_ts_elect(tmem + kT16O, tmem + (t3 == 2 ? 64 : 0) + 8 * ks, (t3 == 1 ? dVl : dVh) + boff, idesc,
                             (t3 | ks) != 0);
          }
        mma_commit_elect(barO);
      }
    }
    return;
  }

  // ===== warps 0 .. CW-1: GEMM epilogue + split, softmax, O =====
  pdl_wait();  // token scales come from the previous kernel
  const int quarter = warp & 3, cq = warp >> 2;  // TMEM lane quarter, column part
  const int row = quarter * 32 + lane;
  const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;

  // accumulator columns -> dequantized f32 (((f32(acc) * s_tok) * s_w) + b, the GEMM
  // epilogue's arithmetic); rows past the last token are 0, as the TMA fill of the
  // unfused path.
  auto dequant = [&](uint32_t* r, const float* sw, const float* sb, bool live, float s_tok) {
#pragma unroll
    for (int j = 0; j < DPT / 4; ++j) {
      const float4 w = *reinterpret_cast<const float4*>(sw + 4 * j);
      // two columns per FMUL2 (the bias add stays scalar: no f32x2 contraction)
      float d0, d1, d2, d3;
      f2unpack(f2mul(f2mul(f2pack(__int2float_rn((int)r[4 * j + 0]), __int2float_rn((int)r[4 * j + 1])), f2splat(s_tok)),
                     f2pack(w.x, w.y)), d0, d1);
      f2unpack(f2mul(f2mul(f2pack(__int2float_rn((int)r[4 * j + 2]), __int2float_rn((int)r[4 * j + 3])), f2splat(s_tok)),
                     f2pack(w.z, w.w)), d2, d3);
      r[4 * j + 0] = __float_as_uint(d0);
      r[4 * j + 1] = __float_as_uint(d1);
      r[4 * j + 2] = __float_as_uint(d2);
      r[4 * j + 3] = __float_as_uint(d3);
    }
    if (bias != nullptr) {
#pragma unroll
      for (int j = 0; j < DPT / 4; ++j) {
        const float4 bb = *reinterpret_cast<const float4*>(sb + 4 * j);
        r[4 * j + 0] = __float_as_uint(__fadd_rn(__uint_as_float(r[4 * j + 0]), bb.x));
        r[4 * j + 1] = __float_as_uint(__fadd_rn(__uint_as_float(r[4 * j + 1]), bb.y));
        r[4 * j + 2] = __float_as_uint(__fadd_rn(__uint_as_float(r[4 * j + 2]), bb.z));
        r[4 * j + 3] = __float_as_uint(__fadd_rn(__uint_as_float(r[4 * j + 3]), bb.w));
      }
    }
    if (!live) {
#pragma unroll
      for (int j = 0; j < DPT; ++j) r[j] = 0u;
    }
  };

  // accumulator of unit (hd, u) -> Q hi/lo in TMEM, K hi/lo and V^T hi/lo (buffer
  // vb) in smem, with attention_f16_kernel's per-tile power-of-two scales (the
  // tile maxima do not depend on which thread holds which element).  Thread
  // (row, cq) holds columns [DPT cq, DPT cq + DPT) of its row of Q, K and V; V^T is
  // written as token pairs exchanged between adjacent lanes.  The accumulator
  // goes back to the GEMM (accfree) as soon as it has been read.  s_tok: the token
  // scale of this thread's row of unit hd (0 past the last token), loaded ahead.
  auto epi_split = [&](int hd, int u, int vb, float s_tok, float& fq, float& fk, float& fv,
                       unsigned long long* stamp) {
    const bool live = (hd / heads) * seq + row < M;
    uint32_t qa[DPT], ka[DPT], va[DPT];
    mbar_wait(accf, u & 1);
    tc_fence_after();
    if (stamp) *stamp = gtime();
    unsigned long long* ss = (stamp && u == 1) ? tr + 40 : nullptr;
    tmem_ld_cols<DPT>(tmem + lane_base + kQaAcc + DPT * cq, qa);
    tmem_ld_cols<DPT>(tmem + lane_base + kQaAcc + kAttD + DPT * cq, ka);
    tmem_ld_cols<DPT>(tmem + lane_base + kQaAcc + 2 * kAttD + DPT * cq, va);
    if (tid == 0 && tma_store && u >= 2) bulk_wait_read0();  // O staging (V^T buffer vb) read out
    mbar_wait(&scf[u & 1], (u >> 1) & 1);
    tmem_ld_wait();
    if (ss) ss[0] = gtime();
    {
      const float* sw = sSc + (u & 1) * (2 * 3 * kAttD) + DPT * cq;
      dequant(qa, sw, sw + 3 * kAttD, live, s_tok);
      dequant(ka, sw + kAttD, sw + 4 * kAttD, live, s_tok);
      dequant(va, sw + 2 * kAttD, sw + 5 * kAttD, live, s_tok);
    }
    const float* q = reinterpret_cast<const float*>(qa);
    const float* k = reinterpret_cast<const float*>(ka);
    const float* v = reinterpret_cast<const float*>(va);
    uint32_t mq = 0, mk = 0, mv = 0;
#pragma unroll
    for (int i = 0; i < DPT; ++i) {
      mq = max(mq, qa[i] & 0x7fffffffu);
      mk = max(mk, ka[i] & 0x7fffffffu);
      mv = max(mv, va[i] & 0x7fffffffu);
    }
    mq = __reduce_max_sync(0xffffffffu, mq);
    mk = __reduce_max_sync(0xffffffffu, mk);
    mv = __reduce_max_sync(0xffffffffu, mv);
    if (ss) ss[1] = gtime();
    compute_bar<CW>();  // rmax of the previous split has been read by everyone
    if (lane == 0) rmax[warp * 3] = mq, rmax[warp * 3 + 1] = mk, rmax[warp * 3 + 2] = mv;
    tc_fence_before();
    compute_bar<CW>();  // also: every thread has read the accumulator and the scales
    if (tid == 0) {
      if (!(trigger_late & 4)) mbar_arrive(accfree);
      mbar_arrive(&scfree[u & 1]);
    }
    {
      const uint32_t a = lane < CW ? rmax[lane * 3] : 0u, bq = lane < CW ? rmax[lane * 3 + 1] : 0u,
                     cq3 = lane < CW ? rmax[lane * 3 + 2] : 0u;
      mq = __reduce_max_sync(0xffffffffu, a);
      mk = __reduce_max_sync(0xffffffffu, bq);
      mv = __reduce_max_sync(0xffffffffu, cq3);
    }
    fq = pow2_scale_for(mq), fk = pow2_scale_for(mk), fv = pow2_scale_for(mv);
    if (ss) ss[2] = gtime();
    {
      uint32_t hi[DPT / 2], lo[DPT / 2];
#pragma unroll
      for (int j = 0; j < DPT / 2; ++j)
        split_f16x2(__fmul_rn(q[2 * j], fq), __fmul_rn(q[2 * j + 1], fq), hi[j], lo[j]);
      tmem_st_cols<DPT / 2>(tmem + lane_base + kT16Q + (DPT / 2) * cq, hi);
      tmem_st_cols<DPT / 2>(tmem + lane_base + kT16Q + 32 + (DPT / 2) * cq, lo);
    }
    {
      uint32_t hi[DPT / 2], lo[DPT / 2];
#pragma unroll
      for (int j = 0; j < DPT / 2; ++j)
        split_f16x2(__fmul_rn(k[2 * j], fk), __fmul_rn(k[2 * j + 1], fk), hi[j], lo[j]);
#pragma unroll
      for (int c = 0; c < DPT / 8; ++c) {
        const uint32_t off = row * 128 + (((((DPT / 8) * cq + c) ^ (row & 7))) << 4);
        *reinterpret_cast<uint4*>(sKh + off) = make_uint4(hi[4 * c], hi[4 * c + 1], hi[4 * c + 2], hi[4 * c + 3]);
        *reinterpret_cast<uint4*>(sKl + off) = make_uint4(lo[4 * c], lo[4 * c + 1], lo[4 * c + 2], lo[4 * c + 3]);
      }
    }
    {
      if (ss) ss[3] = gtime();
      // V^T [64 dims][128 tokens] f16, 2 atoms of [64 x 128 B]: token t of dim d at
      // atom t / 64, row d, 16-byte chunk ((t % 64) / 8) ^ (d % 8), element t % 8.
      // Of this thread's DPT dims, the even lane of a token pair writes dim kk and
      // the odd lane dim DPT/2 + (kk ^ 4) (their swizzled chunks differ: no bank
      // conflict between the two halves).  An element travels as one word, f16 hi |
      // f16 lo << 16 (split_f16x2 of the dim pair, then byte permutes).
      uint8_t* vh = sVT + vb * (2 * kH16);
      uint8_t* vl = vh + kH16;
      const bool odd = lane & 1;
      const int t0 = row & ~1;
      const uint32_t tbase = (uint32_t)(t0 >> 6) * (64 * 128) + (uint32_t)(t0 & 7) * 2;
      const int tch = (t0 & 63) >> 3;
#pragma unroll
      for (int kk = 0; kk < DPT / 2; ++kk) {
        const int dm = kk, dp = DPT / 2 + (kk ^ 4);
        uint32_t hi2, lo2;  // (hi, lo) of dims dm (low halves) and dp (high halves)
        split_f16x2(__fmul_rn(v[dm], fv), __fmul_rn(v[dp], fv), hi2, lo2);
        const uint32_t e_dm = __byte_perm(hi2, lo2, 0x5410), e_dp = __byte_perm(hi2, lo2, 0x7632);
        const uint32_t recv = __shfl_xor_sync(0xffffffffu, odd ? e_dm : e_dp, 1);
        const uint32_t mine = odd ? e_dp : e_dm;
        const uint32_t ev = odd ? recv : mine, od = odd ? mine : recv;  // tokens t0, t0 + 1
        const int d = DPT * cq + (odd ? dp : dm);
        const uint32_t off = tbase + (uint32_t)d * 128 + (uint32_t)((tch ^ (d & 7)) << 4);
        *reinterpret_cast<uint32_t*>(vh + off) = (ev & 0xffffu) | (od << 16);
        *reinterpret_cast<uint32_t*>(vl + off) = (ev >> 16) | (od & 0xffff0000u);
      }
    }
    if (ss) ss[4] = gtime();
    tmem_st_wait();
    fence_proxy_async_smem();
    tc_fence_before();
    compute_bar<CW>();
    tc_fence_after();
    if (tid == 0) {
      if (trigger_late & 4) mbar_arrive(accfree);  // debug: GEMM after the whole split
      mbar_arrive(qkr);  // S of this unit may be issued
    }
    if (ss) ss[5] = gtime();
  };

  auto token_scale = [&](int hd) {
    const int grow = (hd / heads) * seq + row;
    return hd < nheads_total && grow < M ? __ldg(ts + grow) : 0.0f;
  };
  float fq = 1.0f, fk = 1.0f, fv = 1.0f;
  // it = -1: the first unit's projection and split only; it >= 0: unit hd's attention,
  // with unit nxt's projection and split under its P V.  One loop body: a single copy
  // of epi_split in the instruction stream (the prologue warms it).
  for (int it = -1;; ++it) {
    const bool cur = it >= 0;
    const int hd = (int)blockIdx.x + it * (int)gridDim.x;
    const int nxt = hd + (int)gridDim.x;
    if (cur ? hd >= nheads_total : nxt >= nheads_total) break;
    const uint32_t ph = it & 1;
    const int b = hd / heads, h = hd % heads;
    unsigned long long* ti = (tr && cur && it < 6) ? tr + 8 + it * 8 : nullptr;
    if (ti) ti[7] = gtime();
    const float cfq = fq, cfk = fk, cfv = fv;  // this head's scales (split(nxt) overwrites)
    const float s_tok_nxt = token_scale(nxt);  // in flight during the softmax
    if (ti) ti[0] = gtime();
    float oscale = 0.0f;
    if (cur) {
      mbar_wait(barS, ph);
      tc_fence_after();
      if (ti) ti[1] = gtime();
      // ---- softmax: S' from TMEM; P' = 2^15 exp(.) as f16 hi / lo back into TMEM ----
      float s[KPT];
      {
        uint32_t r0[KPT];
        tmem_ld_cols<KPT>(tmem + lane_base + KPT * cq, r0);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < KPT; ++j) s[j] = __uint_as_float(r0[j]);
      }
      float mx = -INFINITY;
      if (seq == kAttT && !causal) {
#pragma unroll
        for (int j = 0; j < KPT; ++j) mx = fmaxf(mx, s[j]);
      } else {
#pragma unroll
        for (int j = 0; j < KPT; ++j) {
          const int key = KPT * cq + j;
          if (key >= seq || (causal && key > row)) s[j] = -INFINITY;  // mask (transformer.py:433-434)
          mx = fmaxf(mx, s[j]);
        }
      }
      redm[cq * 128 + row] = mx;
      compute_bar<CW>();
#pragma unroll
      for (int c = 0; c < NCQ; ++c) mx = fmaxf(mx, redm[c * 128 + row]);
      // exp(inv (s - max)) with s = S' / (fq fk): c = inv log2(e) / (fq fk), exact powers of two
      const float c = __fmul_rn(__fmul_rn(__fmul_rn(scale, 1.4426950408889634f), pow2_inv(cfq)), pow2_inv(cfk));
      const float mxc = __fsub_rn(__fmul_rn(mx, c), 15.0f);  // P' = 2^15 exp(.): +15 in the exponent
      // row sum in attention_f16_kernel's order: per 32-key quarter, four
      // interleaved partials ((p0 + p1) + (p2 + p3)); quarters ((q0 + q1) + (q2 + q3))
      float qs[KPT / 32];
#pragma unroll
      for (int qq = 0; qq < KPT / 32; ++qq) {
        float sp[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float e = ex2_approx_f(__fmaf_rn(s[32 * qq + j], c, -mxc));
          s[32 * qq + j] = e;
          sp[j & 3] = __fadd_rn(sp[j & 3], e);
        }
        qs[qq] = __fadd_rn(__fadd_rn(sp[0], sp[1]), __fadd_rn(sp[2], sp[3]));
      }
      reds[cq * 128 + row] = KPT / 32 == 2 ? __fadd_rn(qs[0], qs[KPT / 32 - 1]) : qs[0];
      compute_bar<CW>();
      float sum;
      if (NCQ == 2)
        sum = __fadd_rn(reds[row], reds[128 + row]);
      else
        sum = __fadd_rn(__fadd_rn(reds[row], reds[128 + row]), __fadd_rn(reds[256 + row], reds[384 + row]));
      // O = (P' V') / (fv sum'), sum' = 2^15 sum
      oscale = __fmul_rn(__frcp_rn(sum), pow2_inv(cfv));
      {
        uint32_t hi[KPT / 2], lo[KPT / 2];
#pragma unroll
        for (int j = 0; j < KPT / 2; ++j) split_f16x2(s[2 * j], s[2 * j + 1], hi[j], lo[j]);
        tmem_st_cols<KPT / 2>(tmem + lane_base + (KPT / 2) * cq, hi);
        tmem_st_cols<KPT / 2>(tmem + lane_base + 64 + (KPT / 2) * cq, lo);
      }
      tmem_st_wait();
      tc_fence_before();
      compute_bar<CW>();
      tc_fence_after();
      if (ti) ti[2] = gtime();
      if (tid == 0) mbar_arrive(prdy);  // O' = P' V' is issued by the attention MMA warp
    }
    // ---- the next unit's projection epilogue and split run while the tensor
    //      core computes P V (the GEMM of the unit after streams meanwhile) ----
    if (nxt < nheads_total) {
      epi_split(nxt, it + 1, (it + 1) & 1, s_tok_nxt, fq, fk, fv, ti ? ti + 3 : (tr && !cur) ? tr + 2 : nullptr);
      if (ti) ti[4] = gtime();
      if (tr && !cur) tr[3] = gtime();
    }
    if (!cur) continue;
    mbar_wait(barO, ph);
    tc_fence_after();
    if (ti) ti[5] = gtime();
    {
      uint32_t r0[DPT];
      tmem_ld_cols<DPT>(tmem + lane_base + kT16O + DPT * cq, r0);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < DPT; ++j) r0[j] = __float_as_uint(__fmul_rn(__uint_as_float(r0[j]), oscale));
      if (tma_store) {  // stage in this unit's V^T buffer (P V is done with it), SW128 f32 boxes
        const int col = DPT * cq;  // of the head's 64
        uint8_t* st = sVT + (it & 1) * (2 * kH16) + (col >> 5) * kH16 + row * 128;
#pragma unroll
        for (int c = 0; c < DPT / 4; ++c)
          *reinterpret_cast<uint4*>(st + (((((col & 31) >> 2) + c) ^ (row & 7)) << 4)) =
              make_uint4(r0[4 * c], r0[4 * c + 1], r0[4 * c + 2], r0[4 * c + 3]);
      } else if (row < seq) {
        float* dst = ctx + ((int64_t)b * seq + row) * ld_ctx + h * kAttD + DPT * cq;
#pragma unroll
        for (int j = 0; j < DPT; j += 4)
          *reinterpret_cast<float4*>(dst + j) =
              make_float4(__uint_as_float(r0[j]), __uint_as_float(r0[j + 1]), __uint_as_float(r0[j + 2]),
                          __uint_as_float(r0[j + 3]));
      }
    }
    if (tma_store) fence_proxy_async_smem();
    tc_fence_before();
    compute_bar<CW>();  // O read out: the next P V may overwrite it
    tc_fence_after();
    if (tma_store && tid == 0) {
      const uint8_t* st = sVT + (it & 1) * (2 * kH16);
      tma_store_2d(&tmc, st, h * kAttD, b * seq);
      tma_store_2d(&tmc, st + kH16, h * kAttD + 32, b * seq);
      bulk_commit();
    }
    if (ti) ti[6] = gtime();
  }
  if (tma_store && tid == 0) bulk_wait0();
  if (trigger_late & 1) pdl_trigger();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

// ---------------------------------------------------------------------------
// Split-role variant of the fused kernel (16 compute warps): warps 8-15 dequantize
// and split unit u + 1 while warps 0-7 run unit u's softmax and O, so the two
// CUDA-core phases overlap instead of taking turns on the same warps.  Scales per
// unit travel through smem (sfr), the V^T buffer is handed back by the attention
// warps once O has been staged out of it (vtfree).  Same arithmetic and order as
// qkv_attention_kernel: ctx is bit-identical.
// ---------------------------------------------------------------------------
constexpr int kQsThreads = 640;
constexpr int kQsSmem = kQaX + 6 * kH16 + kQaSc + 168 + 8 * 3 * 4 + 4 * 128 * 4 + 32;

__global__ void __launch_bounds__(kQsThreads, 1)
    qkv_attention_split_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW,
                         const float* __restrict__ ts, const float* __restrict__ rs, const float* __restrict__ bias,
                         int M, int seq, int heads, int dmodel, int causal, float scale, float* __restrict__ ctx,
                         int64_t ld_ctx, int nheads_total, unsigned long long* __restrict__ trace,
                         const __grid_constant__ CUtensorMap tmc, int tma_store, int trigger_late) {
  constexpr int KPT = 64, DPT = 32;  // 8 attention + 8 convert warps, 2 column halves per row
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* sX = sm;
  uint8_t* sKh = sm + kQaX;
  uint8_t* sKl = sKh + kH16;
  uint8_t* sVT = sKl + kH16;  // [2 buffers][hi | lo]
  float* sSc = reinterpret_cast<float*>(sVT + 4 * kH16);  // per-unit weight scales and bias
  uint64_t* bars = reinterpret_cast<uint64_t*>(sVT + 4 * kH16 + kQaSc);
  uint64_t* gfull = bars;       // [3] operand stage landed
  uint64_t* gempty = bars + 3;  // [3] operand stage consumed by the MMAs
  uint64_t* accf = bars + 6;    // GEMM accumulator complete
  uint64_t* accfree = bars + 7; // accumulator read by the epilogue
  uint64_t* barS = bars + 8;
  uint64_t* barO = bars + 9;
  uint64_t* scf = bars + 10;    // [2] unit parity: scales and bias landed
  uint64_t* scfree = bars + 12; // [2] unit parity: scales and bias read by epi_split
  uint64_t* qkr = bars + 14;    // Q, K, V^T of the next unit split (S may be issued)
  uint64_t* prdy = bars + 15;   // P written (P V may be issued)
  // per unit parity (a single barrier could complete twice before the convert
  // warps look: the attention warps may finish units u - 2 and u - 1 first)
  uint64_t* vtfree = bars + 16; // [2] O of unit u staged out of V^T buffer u & 1
  uint64_t* sfr = bars + 18;    // [2] unit parity: the unit's power-of-two scales written
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 20);
  uint32_t* rmax = reinterpret_cast<uint32_t*>(bars + 21);  // [8 convert warps][3]
  float* redm = reinterpret_cast<float*>(rmax + 8 * 3);     // [2][128] row partial maxima
  float* reds = redm + 2 * 128;                             // [2][128] row partial sums
  float* sfs = reds + 2 * 128;                              // [2][4] (fq, fk, fv) per unit parity

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nkb = dmodel / 128;
  if (tid == 0) {
    if (smem_u32(sm) & 1023) __trap();
    prefetch_tmap(&tmX);
    prefetch_tmap(&tmW);
    for (int i = 0; i < 20; ++i) mbar_init(&bars[i], 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  unsigned long long* tr = (trace && tid == 0) ? trace + (size_t)blockIdx.x * 64 : nullptr;
  if (tr) tr[0] = gtime();
  // PDL: dependents may launch only once every warp has resized its registers (a
  // dependent CTA landing on this SM could otherwise take the registers the TMA /
  // MMA warpgroup released before the convert warps claim them: deadlock)
  auto resized = [&]() {
    asm volatile("bar.sync 3, %0;" ::"n"(kQsThreads) : "memory");
    if (!(trigger_late & 1)) pdl_trigger();
  };
  // registers: the 640 threads launch at 96 each (61440, the CTA's pool); the TMA /
  // MMA warpgroup gives 48 of its 96 to the convert warps (dequant + split hold 3 x
  // 32 values): 4 x 48 + 8 x 96 + 8 x 120 = 20 x 96.  setmaxnreg.inc only draws on
  // what the CTA's own dec released.  Each role's code sits inside the branch that
  // resizes its warpgroup.
  if (warp >= 16) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 48;" ::: "memory");
    resized();

  if (warp == 16) {  // ===== GEMM operand producer =====
    if (lane == 0) {
      // the unit's 192 weight-row scales and biases -> buffer u & 1 (free once
      // epi_split(u - 2) has read it)
      auto load_scales = [&](int h, int u) {
        if (u >= 2) mbar_wait_idle(&scfree[u & 1], ((u >> 1) - 1) & 1);
        float* dst = sSc + (u & 1) * (2 * 3 * kAttD);
        mbar_arrive_expect_tx(&scf[u & 1], (bias ? 2 : 1) * 3 * kAttD * 4);
#pragma unroll
        for (int part = 0; part < 3; ++part) {
          bulk_load_1d(dst + part * kAttD, rs + part * dmodel + h * kAttD, kAttD * 4, &scf[u & 1]);
          if (bias) bulk_load_1d(dst + 3 * kAttD + part * kAttD, bias + part * dmodel + h * kAttD, kAttD * 4,
                                 &scf[u & 1]);
        }
      };
      auto load_w = [&](uint8_t* st, int kb, int h, uint64_t* bar) {
#pragma unroll
        for (int part = 0; part < 3; ++part)
          tma_load_2d(st + kQaStageA + part * (kAttD * 128), &tmW, bar, kb * 128, part * dmodel + h * kAttD);
      };
      // weights and scales do not depend on the previous kernel: unit 0's first
      // stages of B go out before griddepcontrol.wait, A (the activations) after it
      const int npre = nkb < kQaStages ? nkb : kQaStages;
      if ((int)blockIdx.x < nheads_total) {
        const int h0 = (int)blockIdx.x % heads;
        load_scales(h0, 0);
        for (int kb = 0; kb < npre; ++kb) {
          mbar_arrive_expect_tx(&gfull[kb], kQaStage);
          load_w(sX + kb * kQaStage, kb, h0, &gfull[kb]);
        }
      }
      pdl_wait();
      if (tr) tr[1] = gtime();
      int kc = 0, u = 0;
      for (int hd = blockIdx.x; hd < nheads_total; hd += gridDim.x, ++u) {
        const int b = hd / heads, h = hd % heads;
        if ((trigger_late & 2) && u >= 1) mbar_wait(accfree, (u - 1) & 1);  // debug: no operand prefetch
        if (u > 0) load_scales(h, u);
        for (int kb = 0; kb < nkb; ++kb, ++kc) {
          const int s = kc % kQaStages;
          uint8_t* st = sX + s * kQaStage;
          if (u == 0 && kb < npre) {  // B already in flight
            tma_load_2d(st, &tmX, &gfull[s], kb * 128, b * seq);
            continue;
          }
          if (kc >= kQaStages) mbar_wait_idle(&gempty[s], ((kc / kQaStages) - 1) & 1);
          if (trace && kb == 0 && kc / nkb < 4) trace[(size_t)blockIdx.x * 64 + 60 + kc / nkb] = gtime();
          mbar_arrive_expect_tx(&gfull[s], kQaStage);
          tma_load_2d(st, &tmX, &gfull[s], kb * 128, b * seq);
          load_w(st, kb, h, &gfull[s]);
        }
      }
    }
    return;
  }
  if (warp == 17) {  // ===== GEMM MMA issuer =====
    if (lane == 0) {
      constexpr uint32_t idesc = make_idesc_i8(128, 3 * kAttD);
      int kc = 0, u = 0;
      for (int hd = blockIdx.x; hd < nheads_total; hd += gridDim.x, ++u) {
        if (u > 0) mbar_wait_idle(accfree, (u - 1) & 1);  // the previous unit's accumulator has been read
        tc_fence_after();
        for (int kb = 0; kb < nkb; ++kb, ++kc) {
          const int s = kc % kQaStages;
          mbar_wait(&gfull[s], (kc / kQaStages) & 1);
          tc_fence_after();
          if (trace && kb == nkb - 1 && u < 4) trace[(size_t)blockIdx.x * 64 + 56 + u] = gtime();
          if (trace && kb == 0 && u < 4) trace[(size_t)blockIdx.x * 64 + 52 + u] = gtime();
          const uint32_t a_addr = smem_u32(sX + s * kQaStage);
          const uint32_t b_addr = a_addr + kQaStageA;
#pragma unroll
          for (int k = 0; k < 4; ++k)
            mma_i8(tmem + kQaAcc, make_sw128_desc(a_addr + k * 32), make_sw128_desc(b_addr + k * 32), idesc,
                   (kb | k) != 0);
          mma_commit(&gempty[s]);
        }
        mma_commit(accf);
      }
    }
    return;
  }

  if (warp == 18) {  // ===== attention MMA issuer: S = Q K^T, O = P V (3-term f16 splits) =====
    int it = 0;
    for (int hd = blockIdx.x; hd < nheads_total; hd += gridDim.x, ++it) {
      mbar_wait_idle(qkr, it & 1);                         // Q, K, V^T of unit it split
      if (it > 0) mbar_wait_idle(barO, (it - 1) & 1);      // P of unit it - 1 consumed
      tc_fence_after();
      {
        const uint32_t idesc = make_idesc_f16(128, 128);
        const uint64_t dKh = make_sw128_desc(smem_u32(sKh)), dKl = make_sw128_desc(smem_u32(sKl));
#pragma unroll
        for (int t3 = 0; t3 < 3; ++t3)
#pragma unroll
          for (int ks = 0; ks < kAttD / 16; ++ks)
            mma_f16_ts_elect(tmem, tmem + kT16Q + (t3 == 2 ? 32 : 0) + 8 * ks, (t3 == 1 ? dKl : dKh) + 2 * ks,
                             idesc, (t3 | ks) != 0);
        mma_commit_elect(barS);
      }
      mbar_wait_idle(prdy, it & 1);                        // P of unit it written
      tc_fence_after();
      {
        const uint32_t idesc = make_idesc_f16(128, kAttD);
        const uint8_t* vh = sVT + (it & 1) * (2 * kH16);
        const uint64_t dVh = make_sw128_desc(smem_u32(vh)), dVl = make_sw128_desc(smem_u32(vh + kH16));
#pragma unroll
        for (int t3 = 0; t3 < 3; ++t3)
#pragma unroll
          for (int ks = 0; ks < kAttT / 16; ++ks) {
            const uint64_t boff = (uint64_t)(((ks >> 2) * (64 * 128) + (ks & 3) * 32) >> 4);
            mma_f16_ts_elect(tmem + kT16O, tmem + (t3 == 2 ? 64 : 0) + 8 * ks, (t3 == 1 ? dVl : dVh) + boff, idesc,
                             (t3 | ks) != 0);
          }
        mma_commit_elect(barO);
      }
    }
    return;
  }

    return;  // warp 19
  }
  const int quarter = warp & 3, half = (warp >> 2) & 1;  // TMEM lane quarter, column half
  const int row = quarter * 32 + lane;
  const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
  auto token_scale = [&](int hd) {
    const int grow = (hd / heads) * seq + row;
    return hd < nheads_total && grow < M ? __ldg(ts + grow) : 0.0f;
  };

  if (warp >= 8) {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 120;" ::: "memory");
    resized();
    pdl_wait();  // token scales come from the previous kernel
    // ===== convert warps 8-15: accumulator of unit u -> Q hi/lo (TMEM), K hi/lo and
    //       V^T hi/lo (smem), the next split overlapping the attention warps' softmax =====
    const int gtid = tid - 256;  // 0 .. 255
    unsigned long long* trb = (trace && gtid == 0) ? trace + (size_t)blockIdx.x * 64 : nullptr;
    auto gbar = []() { asm volatile("bar.sync 2, 256;" ::: "memory"); };
    auto dequant = [&](uint32_t* r, const float* sw, const float* sb, bool live, float s_tok) {
#pragma unroll
      for (int j = 0; j < DPT / 4; ++j) {
        const float4 w = *reinterpret_cast<const float4*>(sw + 4 * j);
        // two columns per FMUL2 (the bias add stays scalar: no f32x2 contraction)
        float d0, d1, d2, d3;
        f2unpack(f2mul(f2mul(f2pack(__int2float_rn((int)r[4 * j + 0]), __int2float_rn((int)r[4 * j + 1])), f2splat(s_tok)),
                       f2pack(w.x, w.y)), d0, d1);
        f2unpack(f2mul(f2mul(f2pack(__int2float_rn((int)r[4 * j + 2]), __int2float_rn((int)r[4 * j + 3])), f2splat(s_tok)),
                       f2pack(w.z, w.w)), d2, d3);
        r[4 * j + 0] = __float_as_uint(d0);
        r[4 * j + 1] = __float_as_uint(d1);
        r[4 * j + 2] = __float_as_uint(d2);
        r[4 * j + 3] = __float_as_uint(d3);
      }
      if (bias != nullptr) {
#pragma unroll
        for (int j = 0; j < DPT / 4; ++j) {
          const float4 bb = *reinterpret_cast<const float4*>(sb + 4 * j);
          r[4 * j + 0] = __float_as_uint(__fadd_rn(__uint_as_float(r[4 * j + 0]), bb.x));
          r[4 * j + 1] = __float_as_uint(__fadd_rn(__uint_as_float(r[4 * j + 1]), bb.y));
          r[4 * j + 2] = __float_as_uint(__fadd_rn(__uint_as_float(r[4 * j + 2]), bb.z));
          r[4 * j + 3] = __float_as_uint(__fadd_rn(__uint_as_float(r[4 * j + 3]), bb.w));
        }
      }
      if (!live) {
#pragma unroll
        for (int j = 0; j < DPT; ++j) r[j] = 0u;
      }
    };
    int u = 0;
    float s_tok = token_scale(blockIdx.x);
    for (int hd = blockIdx.x; hd < nheads_total; hd += gridDim.x, ++u) {
      const int vb = u & 1;
      const bool live = (hd / heads) * seq + row < M;
      const float s_tok_next = token_scale(hd + (int)gridDim.x);
      unsigned long long* st_acc = trb ? (u == 0 ? trb + 2 : u <= 6 ? trb + 8 + (u - 1) * 8 + 3 : nullptr) : nullptr;
      uint32_t qa[DPT], ka[DPT], va[DPT];
      mbar_wait(accf, u & 1);
      tc_fence_after();
      if (st_acc) *st_acc = gtime();
      tmem_ld_cols<DPT>(tmem + lane_base + kQaAcc + DPT * half, qa);
      tmem_ld_cols<DPT>(tmem + lane_base + kQaAcc + kAttD + DPT * half, ka);
      tmem_ld_cols<DPT>(tmem + lane_base + kQaAcc + 2 * kAttD + DPT * half, va);
      mbar_wait(&scf[u & 1], (u >> 1) & 1);
      tmem_ld_wait();
      {
        const float* sw = sSc + (u & 1) * (2 * 3 * kAttD) + DPT * half;
        dequant(qa, sw, sw + 3 * kAttD, live, s_tok);
        dequant(ka, sw + kAttD, sw + 4 * kAttD, live, s_tok);
        dequant(va, sw + 2 * kAttD, sw + 5 * kAttD, live, s_tok);
      }
      uint32_t mq = 0, mk = 0, mv = 0;
#pragma unroll
      for (int i = 0; i < DPT; ++i) {
        mq = max(mq, qa[i] & 0x7fffffffu);
        mk = max(mk, ka[i] & 0x7fffffffu);
        mv = max(mv, va[i] & 0x7fffffffu);
      }
      mq = __reduce_max_sync(0xffffffffu, mq);
      mk = __reduce_max_sync(0xffffffffu, mk);
      mv = __reduce_max_sync(0xffffffffu, mv);
      gbar();  // rmax of the previous split has been read by everyone
      if (lane == 0) rmax[(warp - 8) * 3] = mq, rmax[(warp - 8) * 3 + 1] = mk, rmax[(warp - 8) * 3 + 2] = mv;
      tc_fence_before();
      gbar();  // also: every thread has read the accumulator and the scales
      if (gtid == 0) {
        if (!(trigger_late & 4)) mbar_arrive(accfree);
        mbar_arrive(&scfree[u & 1]);
      }
      {
        const uint32_t a = lane < 8 ? rmax[lane * 3] : 0u, bq = lane < 8 ? rmax[lane * 3 + 1] : 0u,
                       cq3 = lane < 8 ? rmax[lane * 3 + 2] : 0u;
        mq = __reduce_max_sync(0xffffffffu, a);
        mk = __reduce_max_sync(0xffffffffu, bq);
        mv = __reduce_max_sync(0xffffffffu, cq3);
      }
      const float fq = pow2_scale_for(mq), fk = pow2_scale_for(mk), fv = pow2_scale_for(mv);
      const float* q = reinterpret_cast<const float*>(qa);
      const float* k = reinterpret_cast<const float*>(ka);
      const float* v = reinterpret_cast<const float*>(va);
      if (u >= 1) {  // S of the previous unit has read Q and K
        mbar_wait(barS, (u - 1) & 1);
        tc_fence_after();
      }
      {
        uint32_t hi[DPT / 2], lo[DPT / 2];
#pragma unroll
        for (int j = 0; j < DPT / 2; ++j)
          split_f16x2(__fmul_rn(q[2 * j], fq), __fmul_rn(q[2 * j + 1], fq), hi[j], lo[j]);
        tmem_st_cols<DPT / 2>(tmem + lane_base + kT16Q + (DPT / 2) * half, hi);
        tmem_st_cols<DPT / 2>(tmem + lane_base + kT16Q + 32 + (DPT / 2) * half, lo);
      }
      {
        uint32_t hi[DPT / 2], lo[DPT / 2];
#pragma unroll
        for (int j = 0; j < DPT / 2; ++j)
          split_f16x2(__fmul_rn(k[2 * j], fk), __fmul_rn(k[2 * j + 1], fk), hi[j], lo[j]);
#pragma unroll
        for (int c = 0; c < DPT / 8; ++c) {
          const uint32_t off = row * 128 + (((((DPT / 8) * half + c) ^ (row & 7))) << 4);
          *reinterpret_cast<uint4*>(sKh + off) = make_uint4(hi[4 * c], hi[4 * c + 1], hi[4 * c + 2], hi[4 * c + 3]);
          *reinterpret_cast<uint4*>(sKl + off) = make_uint4(lo[4 * c], lo[4 * c + 1], lo[4 * c + 2], lo[4 * c + 3]);
        }
      }
      if (u >= 2) mbar_wait(&vtfree[vb], ((u >> 1) - 1) & 1);  // O of unit u - 2 has left V^T buffer vb
      {
        // V^T as in qkv_attention_kernel: token pairs across adjacent lanes, the even
        // lane writes dim kk, the odd lane DPT/2 + (kk ^ 4)
        uint8_t* vh = sVT + vb * (2 * kH16);
        uint8_t* vl = vh + kH16;
        const bool odd = lane & 1;
        const int t0 = row & ~1;
        const uint32_t tbase = (uint32_t)(t0 >> 6) * (64 * 128) + (uint32_t)(t0 & 7) * 2;
        const int tch = (t0 & 63) >> 3;
#pragma unroll
        for (int kk = 0; kk < DPT / 2; ++kk) {
          const int dm = kk, dp = DPT / 2 + (kk ^ 4);
          uint32_t hi2, lo2;
          split_f16x2(__fmul_rn(v[dm], fv), __fmul_rn(v[dp], fv), hi2, lo2);
          const uint32_t e_dm = __byte_perm(hi2, lo2, 0x5410), e_dp = __byte_perm(hi2, lo2, 0x7632);
          const uint32_t recv = __shfl_xor_sync(0xffffffffu, odd ? e_dm : e_dp, 1);
          const uint32_t mine = odd ? e_dp : e_dm;
          const uint32_t ev = odd ? recv : mine, od = odd ? mine : recv;
          const int d = DPT * half + (odd ? dp : dm);
          const uint32_t off = tbase + (uint32_t)d * 128 + (uint32_t)((tch ^ (d & 7)) << 4);
          *reinterpret_cast<uint32_t*>(vh + off) = (ev & 0xffffu) | (od << 16);
          *reinterpret_cast<uint32_t*>(vl + off) = (ev >> 16) | (od & 0xffff0000u);
        }
      }
      tmem_st_wait();
      fence_proxy_async_smem();
      tc_fence_before();
      gbar();
      tc_fence_after();
      if (gtid == 0) {
        if (trigger_late & 4) mbar_arrive(accfree);
        // the attention warps take this unit's scales from a slot per unit parity
        // (free: the attention warps read unit u - 2's before their O of u - 2,
        // which this split waited for through vtfree)
        sfs[4 * (u & 1)] = fq, sfs[4 * (u & 1) + 1] = fk, sfs[4 * (u & 1) + 2] = fv;
        mbar_arrive(&sfr[u & 1]);
        mbar_arrive(qkr);  // S of unit u may be issued
      }
      if (trb && u <= 6) {
        if (u == 0) trb[3] = gtime();
        else trb[8 + (u - 1) * 8 + 4] = gtime();
      }
      s_tok = s_tok_next;
    }
    return;
  }
  // ===== attention warps 0-7: softmax of unit it (P into TMEM), then its O =====
  asm volatile("setmaxnreg.inc.sync.aligned.u32 96;" ::: "memory");
  resized();
  pdl_wait();
  auto abar = []() { asm volatile("bar.sync 1, 256;" ::: "memory"); };
  int it = 0;
  for (int hd = blockIdx.x; hd < nheads_total; hd += gridDim.x, ++it) {
    const uint32_t ph = it & 1;
    const int b = hd / heads, h = hd % heads;
    unsigned long long* ti = (tr && it < 6) ? tr + 8 + it * 8 : nullptr;
    if (ti) ti[0] = gtime();
    mbar_wait(barS, ph);
    tc_fence_after();
    mbar_wait(&sfr[it & 1], (it >> 1) & 1);
    const float cfq = sfs[4 * (it & 1)], cfk = sfs[4 * (it & 1) + 1], cfv = sfs[4 * (it & 1) + 2];
    if (ti) ti[1] = gtime();
    // ---- softmax: S' from TMEM; P' = 2^15 exp(.) as f16 hi / lo back into TMEM ----
    float s[KPT];
    {
      uint32_t r0[KPT];
      tmem_ld_cols<KPT>(tmem + lane_base + KPT * half, r0);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < KPT; ++j) s[j] = __uint_as_float(r0[j]);
    }
    float mx = -INFINITY;
    if (seq == kAttT && !causal) {
#pragma unroll
      for (int j = 0; j < KPT; ++j) mx = fmaxf(mx, s[j]);
    } else {
#pragma unroll
      for (int j = 0; j < KPT; ++j) {
        const int key = KPT * half + j;
        if (key >= seq || (causal && key > row)) s[j] = -INFINITY;  // mask (transformer.py:433-434)
        mx = fmaxf(mx, s[j]);
      }
    }
    redm[half * 128 + row] = mx;
    abar();
    mx = fmaxf(redm[row], redm[128 + row]);
    const float c = __fmul_rn(__fmul_rn(__fmul_rn(scale, 1.4426950408889634f), pow2_inv(cfq)), pow2_inv(cfk));
    const float mxc = __fsub_rn(__fmul_rn(mx, c), 15.0f);
    float qs[2];
#pragma unroll
    for (int qq = 0; qq < 2; ++qq) {
      float sp[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const float e = ex2_approx_f(__fmaf_rn(s[32 * qq + j], c, -mxc));
        s[32 * qq + j] = e;
        sp[j & 3] = __fadd_rn(sp[j & 3], e);
      }
      qs[qq] = __fadd_rn(__fadd_rn(sp[0], sp[1]), __fadd_rn(sp[2], sp[3]));
    }
    reds[half * 128 + row] = __fadd_rn(qs[0], qs[1]);
    abar();
    const float sum = __fadd_rn(reds[row], reds[128 + row]);
    const float oscale = __fmul_rn(__frcp_rn(sum), pow2_inv(cfv));
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {  // P hi / lo in two 16-word halves (registers)
      uint32_t hi[16], lo[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) split_f16x2(s[32 * hh + 2 * j], s[32 * hh + 2 * j + 1], hi[j], lo[j]);
      tmem_st_cols<16>(tmem + lane_base + (KPT / 2) * half + 16 * hh, hi);
      tmem_st_cols<16>(tmem + lane_base + 64 + (KPT / 2) * half + 16 * hh, lo);
    }
    tmem_st_wait();
    tc_fence_before();
    abar();
    tc_fence_after();
    if (ti) ti[2] = gtime();
    if (tid == 0) mbar_arrive(prdy);  // O' = P' V' is issued by the attention MMA warp
    mbar_wait(barO, ph);
    tc_fence_after();
    if (ti) ti[5] = gtime();
    {
      uint32_t r0[DPT];
      tmem_ld_cols<DPT>(tmem + lane_base + kT16O + DPT * half, r0);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < DPT; ++j) r0[j] = __float_as_uint(__fmul_rn(__uint_as_float(r0[j]), oscale));
      if (tma_store) {  // stage in this unit's V^T buffer (P V is done with it), SW128 f32 boxes
        uint8_t* st = sVT + (it & 1) * (2 * kH16) + half * kH16 + row * 128;
#pragma unroll
        for (int cc = 0; cc < 8; ++cc)
          *reinterpret_cast<uint4*>(st + ((cc ^ (row & 7)) << 4)) =
              make_uint4(r0[4 * cc], r0[4 * cc + 1], r0[4 * cc + 2], r0[4 * cc + 3]);
      } else if (row < seq) {
        float* dst = ctx + ((int64_t)b * seq + row) * ld_ctx + h * kAttD + DPT * half;
#pragma unroll
        for (int j = 0; j < DPT; j += 4)
          *reinterpret_cast<float4*>(dst + j) =
              make_float4(__uint_as_float(r0[j]), __uint_as_float(r0[j + 1]), __uint_as_float(r0[j + 2]),
                          __uint_as_float(r0[j + 3]));
      }
    }
    if (tma_store) fence_proxy_async_smem();
    tc_fence_before();
    abar();  // O read out: the next P V may overwrite it
    tc_fence_after();
    if (tid == 0) {
      if (tma_store) {
        const uint8_t* st = sVT + (it & 1) * (2 * kH16);
        tma_store_2d(&tmc, st, h * kAttD, b * seq);
        tma_store_2d(&tmc, st + kH16, h * kAttD + 32, b * seq);
        bulk_commit();
        bulk_wait_read0();  // the staging (V^T buffer it & 1) has been read
      }
      mbar_arrive(&vtfree[it & 1]);
    }
    if (ti) ti[6] = gtime();
  }
  if (tma_store && tid == 0) bulk_wait0();
  if (trigger_late & 1) pdl_trigger();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

int make_tmap_f32(CUtensorMap* tm, const void* base, int64_t rows, int64_t cols, int64_t ld_bytes,
                  int box_cols, int box_rows, CUtensorMapSwizzle sw);
int make_tmap_2d(CUtensorMap* tm, CUtensorMapDataType dt, const void* base, int64_t rows, int64_t cols,
                 int64_t ld_bytes, int box_cols, int box_rows, CUtensorMapSwizzle sw,
                 CUtensorMapL2promotion promo);

}  // namespace zq

using namespace zq;

static unsigned long long* g_att_trace = nullptr;
extern "C" int zq_attention_debug(int mode) {  // kept for ABI stability; see zq_attention_set_trace
  return mode == 0 ? ZQ_OK : ZQ_ERR_UNSUPPORTED;
}
extern "C" int zq_attention_set_trace(unsigned long long* buf) {
  g_att_trace = buf;
  return ZQ_OK;
}

extern "C" int zq_attention_f32(const float* qkv, int64_t ld_qkv, int batch, int seq, int heads,
                                int head_dim, int causal, float scale, float* ctx, int64_t ld_ctx,
                                void* stream) {
  ZQ_CHECK_ARG(batch >= 1 && seq >= 1 && heads >= 1, ZQ_ERR_SHAPE, "bad attention shape");
  ZQ_CHECK_ARG(ld_qkv % 4 == 0 && ld_ctx % 4 == 0 && (reinterpret_cast<uintptr_t>(qkv) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(ctx) & 15) == 0,
               ZQ_ERR_UNSUPPORTED, "attention operands must be 16-byte aligned");
  if (head_dim != kAttD) {  // CUDA-core flash attention for the other head sizes
    ZQ_CHECK_ARG(head_dim % 16 == 0 && head_dim <= 256, ZQ_ERR_UNSUPPORTED,
                 "attention supports head_dim 64 (tensor cores) or a multiple of 16 up to 256");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    cudaError_t e2;
    switch (head_dim) {
      case 16: e2 = launch_att_general<16>(qkv, ld_qkv, batch, seq, heads, causal, scale, ctx, ld_ctx, st); break;
      case 32: e2 = launch_att_general<32>(qkv, ld_qkv, batch, seq, heads, causal, scale, ctx, ld_ctx, st); break;
      case 48: e2 = launch_att_general<48>(qkv, ld_qkv, batch, seq, heads, causal, scale, ctx, ld_ctx, st); break;
      case 80: e2 = launch_att_general<80>(qkv, ld_qkv, batch, seq, heads, causal, scale, ctx, ld_ctx, st); break;
      case 112: e2 = launch_att_general<112>(qkv, ld_qkv, batch, seq, heads, causal, scale, ctx, ld_ctx, st); break;
      case 96: e2 = launch_att_general<96>(qkv, ld_qkv, batch, seq, heads, causal, scale, ctx, ld_ctx, st); break;
      case 128: e2 = launch_att_general<128>(qkv, ld_qkv, batch, seq, heads, causal, scale, ctx, ld_ctx, st); break;
      case 160: e2 = launch_att_general<160>(qkv, ld_qkv, batch, seq, heads, causal, scale, ctx, ld_ctx, st); break;
      case 192: e2 = launch_att_general<192>(qkv, ld_qkv, batch, seq, heads, causal, scale, ctx, ld_ctx, st); break;
      case 224: e2 = launch_att_general<224>(qkv, ld_qkv, batch, seq, heads, causal, scale, ctx, ld_ctx, st); break;
      case 256: e2 = launch_att_general<256>(qkv, ld_qkv, batch, seq, heads, causal, scale, ctx, ld_ctx, st); break;
      default:
        set_error("attention: head_dim %d has no instantiation", head_dim);
        return ZQ_ERR_UNSUPPORTED;
    }
    if (e2 != cudaSuccess) {
      set_error("attention launch: %s", cudaGetErrorString(e2));
      return ZQ_ERR_CUDA;
    }
    return ZQ_OK;
  }
  ZQ_CHECK_ARG(ld_qkv % 4 == 0 && ld_ctx % 4 == 0 && (reinterpret_cast<uintptr_t>(qkv) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(ctx) & 15) == 0,
               ZQ_ERR_UNSUPPORTED, "attention operands must be 16-byte aligned");
  CUtensorMap tm;
  const int rc = make_tmap_f32(&tm, qkv, (int64_t)batch * seq, 3LL * heads * head_dim, ld_qkv * 4,
                               32, kAttT, CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc != ZQ_OK) return rc;
  static ZqDeviceOnce attr_once;
  attr_once([&](int) {
    cudaFuncSetAttribute(attention_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kAttSmem);
    cudaFuncSetAttribute(attention_long_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kAttSmem);
    cudaFuncSetAttribute(attention_f16_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kAtt16Smem);
    cudaFuncSetAttribute(attention_f16_long_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kAtt16Smem);
  });
  const int nsm = zq_num_sms();
  const int total = batch * heads;
  cudaError_t e;
  if (seq <= kAttT) {
    const int grid = total < nsm ? total : nsm;
    // seq == 128: whole 128-row boxes belong to one sequence, so O leaves by bulk TMA stores
    CUtensorMap tmc;
    int tma_store = 0;
    if (seq == kAttT && (ld_ctx * 4) % 16 == 0) {
      tma_store = make_tmap_f32(&tmc, ctx, (int64_t)batch * seq, (int64_t)heads * head_dim, ld_ctx * 4, 32, kAttT,
                                CU_TENSOR_MAP_SWIZZLE_128B) == ZQ_OK;
    }
    if (!tma_store) memset(&tmc, 0, sizeof(tmc));
    static int use_tf32 = -1;
    if (use_tf32 < 0) {
      const char* ev = getenv("ZQ_ATT_TF32");
      use_tf32 = ev ? atoi(ev) : 0;
    }
    if (use_tf32)
      e = launch_kernel(attention_kernel, dim3(grid), dim3(256), kAttSmem, reinterpret_cast<cudaStream_t>(stream),
                        1, tm, seq, heads, heads * head_dim, causal, scale, ctx, ld_ctx, total, g_att_trace, tmc,
                        tma_store);
    else
      e = launch_kernel(attention_f16_kernel, dim3(grid), dim3(256), kAtt16Smem,
                        reinterpret_cast<cudaStream_t>(stream), 1, tm, seq, heads, heads * head_dim, causal, scale,
                        ctx, ld_ctx, total, g_att_trace, tmc, tma_store);
  } else {
    const int nq = (seq + kAttT - 1) / kAttT;
    const int items = total * nq;
    const int grid = items < nsm ? items : nsm;
    static int long_tf32 = -1;  // ZQ_ATT_LONG_TF32=1: the 3xTF32 long-sequence kernel
    if (long_tf32 < 0) {
      const char* ev = getenv("ZQ_ATT_LONG_TF32");
      long_tf32 = ev ? atoi(ev) : 0;
    }
    if (long_tf32)
      e = launch_kernel(attention_long_kernel, dim3(grid), dim3(256), kAttSmem,
                        reinterpret_cast<cudaStream_t>(stream), 1, tm, seq, heads, heads * head_dim, causal,
                        scale, ctx, ld_ctx, total, nq);
    else
      e = launch_kernel(attention_f16_long_kernel, dim3(grid), dim3(256), kAtt16Smem,
                        reinterpret_cast<cudaStream_t>(stream), 1, tm, seq, heads, heads * head_dim, causal,
                        scale, ctx, ld_ctx, total, nq);
  }
  if (e != cudaSuccess) {
    set_error("attention launch: %s", cudaGetErrorString(e));
    return ZQ_ERR_CUDA;
  }
  return ZQ_OK;
}

static int qa_trigger_late() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("ZQ_QA_LATE");
    v = e ? atoi(e) : 0;
  }
  return v;
}

// Fused W8A8 QKV projection + attention (encoder, dynamic token-wise activations):
// ctx == zq_attention_f32(zq_linear(xq, w_qkv) as f32) bit for bit, without the
// [T, 3d] f32 QKV round trip.  ZQ_ERR_UNSUPPORTED outside head_dim 64, seq <= 128,
// d a multiple of 128 (the caller runs the two kernels).
extern "C" int zq_qkv_attention(const int8_t* xq, int64_t ld_x, const float* token_scales, const int8_t* w_qkv,
                                int64_t ld_w, const float* w_row_scales, const float* bias, int batch, int seq,
                                int heads, int head_dim, int causal, float scale, float* ctx, int64_t ld_ctx,
                                void* stream) {
  ZQ_CHECK_ARG(batch >= 1 && seq >= 1 && heads >= 1 && head_dim >= 1, ZQ_ERR_SHAPE, "bad attention shape");
  ZQ_CHECK_ARG(xq && token_scales && w_qkv && w_row_scales && ctx, ZQ_ERR_USAGE, "null operand");
  const int dmodel = heads * head_dim;
  ZQ_CHECK_ARG(head_dim == kAttD && seq <= kAttT && dmodel % 128 == 0, ZQ_ERR_UNSUPPORTED,
               "fused QKV attention needs head_dim 64, seq <= 128 and d a multiple of 128");
  auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  ZQ_CHECK_ARG(ld_x % 16 == 0 && ld_w % 16 == 0 && ld_ctx % 4 == 0 && ld_x >= dmodel && ld_w >= dmodel &&
                   ld_ctx >= dmodel && al16(xq) && al16(w_qkv) && al16(w_row_scales) && al16(ctx) &&
                   (bias == nullptr || al16(bias)),
               ZQ_ERR_UNSUPPORTED, "fused QKV attention operands must be 16-byte aligned");
  const int64_t M = (int64_t)batch * seq;
  CUtensorMap tmX, tmW;
  int rc = make_tmap_2d(&tmX, CU_TENSOR_MAP_DATA_TYPE_UINT8, xq, M, dmodel, ld_x, 128, 128,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
  if (rc == ZQ_OK)
    rc = make_tmap_2d(&tmW, CU_TENSOR_MAP_DATA_TYPE_UINT8, w_qkv, 3LL * dmodel, dmodel, ld_w, 128, kAttD,
                      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
  if (rc != ZQ_OK) return rc;
  static ZqDeviceOnce attr_once;
  attr_once([&](int) {
    cudaFuncSetAttribute(qkv_attention_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, QaCfg<8>::SMEM);
    cudaFuncSetAttribute(qkv_attention_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, QaCfg<16>::SMEM);
    cudaFuncSetAttribute(qkv_attention_split_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kQsSmem);
  });
  // variant (ZQ_QA_CW): 16 (default) / 8 compute warps taking turns on split and
  // softmax, or 0 = split roles (8 convert + 8 attention warps, setmaxnreg): in the
  // BERT graph 22.2 / 24.4 / 21.9 us per layer — the split roles gain little (the two
  // groups compete for the same schedulers), so the simpler kernel is the default
  static int cw = -1;
  if (cw < 0) {
    const char* ev = getenv("ZQ_QA_CW");
    cw = ev ? atoi(ev) : 16;
    if (cw != 8 && cw != 0) cw = 16;
  }
  // seq == 128: whole 128-row boxes belong to one sequence, so O leaves by bulk TMA stores
  CUtensorMap tmc;
  int tma_store = 0;
  if (seq == kAttT && (ld_ctx * 4) % 16 == 0)
    tma_store = make_tmap_f32(&tmc, ctx, M, dmodel, ld_ctx * 4, 32, kAttT, CU_TENSOR_MAP_SWIZZLE_128B) == ZQ_OK;
  if (!tma_store) memset(&tmc, 0, sizeof(tmc));
  const int total = batch * heads;
  const int nsm = zq_num_sms();
  const int grid = total < nsm ? total : nsm;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e =
      cw == 0 ? launch_kernel(qkv_attention_split_kernel, dim3(grid), dim3(kQsThreads), kQsSmem, st, 1, tmX, tmW,
                              token_scales, w_row_scales, bias, (int)M, seq, heads, dmodel, causal, scale, ctx, ld_ctx,
                              total, g_att_trace, tmc, tma_store, qa_trigger_late())
      : cw == 8 ? launch_kernel(qkv_attention_kernel<8>, dim3(grid), dim3(QaCfg<8>::THREADS), QaCfg<8>::SMEM, st, 1, tmX,
                              tmW, token_scales, w_row_scales, bias, (int)M, seq, heads, dmodel, causal, scale, ctx,
                              ld_ctx, total, g_att_trace, tmc, tma_store, qa_trigger_late())
              : launch_kernel(qkv_attention_kernel<16>, dim3(grid), dim3(QaCfg<16>::THREADS), QaCfg<16>::SMEM, st, 1,
                              tmX, tmW, token_scales, w_row_scales, bias, (int)M, seq, heads, dmodel, causal, scale,
                              ctx, ld_ctx, total, g_att_trace, tmc, tma_store, qa_trigger_late());
  if (e != cudaSuccess) {
    set_error("fused QKV attention launch: %s", cudaGetErrorString(e));
    return ZQ_ERR_CUDA;
  }
  return ZQ_OK;
}
