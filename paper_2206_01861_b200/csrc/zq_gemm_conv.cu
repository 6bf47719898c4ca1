// CTA-pair tcgen05 GEMMs whose weight operand is converted in shared memory
// before the MMA reads it (the weight stays packed in HBM):
//
//   CONV_W4_I8   W4A8: INT4 weights -> int8, kind::i8, exact int32 accumulators,
//                the exact ZeroQuant epilogue ((f32(acc) * s_tok) * s_w) + b
//                (igemm.py:66-112 with the INT4 FFN of the W4/8 scheme,
//                quant.py:138-141).  Bit-identical to the 1-CTA W4 kernel.
//   CONV_W8_F16  weight-only (FullAct, igemm.py:127-130): int8 -> f16 (exact),
//   CONV_W4_F16  activations as NT = 1 or 2 f16 terms (hi [+ lo]) of the
//                row scaled by a power of two, kind::f16 with f32 accumulators;
//                out = ((acc * 2^-e_row) * s_w) + b.  A tolerance mode next to
//                the bit-exact sequential CUDA-core kernel (zq_linear_full):
//                NT = 1 is the paper's A16 deployment (fp16 activations),
//                NT = 2 carries 22 significant bits of each activation.
//
// Pair layout (cta_group::2) as in zq_gemm2_kernel: a cluster of 2 CTAs owns a
// 256 x BN tile; CTA r holds A rows [128r, 128r+128) and B rows
// [r*BN/2, (r+1)*BN/2).  Warp roles:
//   warp 0      TMA producer: A term tiles (SWIZZLE_128B, completing on the
//               leader's full barrier) and the raw weight rows (unswizzled,
//               completing on this CTA's raw barrier)
//   warp 1      TMEM allocator + (leader) MMA issuer
//   warps 2..9  epilogue (tcgen05.ld -> scale -> swizzled smem -> TMA store)
//   warps 10-13 converters: raw weight rows -> the K-major SWIZZLE_128B tile the
//               MMA reads (row r, 16-byte chunk j at r*128 + ((j ^ (r&7)) << 4)),
//               then a release arrive on the leader's full barrier.
// Every K-block is 128 bytes of A per row: 128 int8 or 64 f16 elements.
#include <cuda.h>
#include <cuda_fp16.h>
#include <cudaTypedefs.h>
#include <string.h>

#include <algorithm>
#include <cmath>

#include "zq_gemm.cuh"

namespace zq {

enum ConvKind { CONV_W4_I8 = 0, CONV_W8_F16 = 1, CONV_W4_F16 = 2 };

template <int BN, int CONV, int NT>
struct ConvCfg {
  static constexpr bool F16 = CONV != CONV_W4_I8;
  static constexpr int KB = F16 ? 64 : 128;                      // K elements per k-block
  static constexpr int A_BYTES = BLOCK_M * 128;                  // one A term tile
  static constexpr int B_BYTES = (BN / 2) * 128;                 // this CTA's converted B half
  static constexpr int RAW_ROW = CONV == CONV_W4_F16 ? 32 : 64;  // packed weight bytes per row per k-block
  static constexpr int RAW_BYTES = (BN / 2) * RAW_ROW;
  static constexpr int STAGE_BYTES = NT * A_BYTES + B_BYTES + RAW_BYTES;
  static constexpr int EPI_NB = NT > 1 ? 1 : 2;                  // staging buffers per epilogue warp
  static constexpr int EPI_BYTES = kNumEpiWarps * EPI_NB * 32 * 32 * 4;
  static constexpr int RING = 232448 - EPI_BYTES - 1024 - 256;
  static constexpr int STAGES = RING / STAGE_BYTES > 8 ? 8 : RING / STAGE_BYTES;
  static constexpr int TMEM_COLS = 2 * BN <= 256 ? 256 : 512;
  static constexpr int NUM_THREADS = (2 + kNumEpiWarps + 4) * 32;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + EPI_BYTES + 1024 + 256;
  static_assert(STAGES >= 2, "ring too small");
  static_assert(B_BYTES % 1024 == 0 && RAW_BYTES % 1024 == 0, "tiles must keep 1024-byte alignment");
};

// kind::f16 instruction descriptor: f32 accumulate, f16 A/B, both K-major.
__host__ __device__ constexpr uint32_t make_idesc_f16_kmajor(int M, int N) {
  return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_f16_cg2(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// 4 int8 -> 4 f16 (exact): 0x64XX is the f16 1024 + XX; XX = q + 128.
__device__ __forceinline__ void i8x4_to_f16(uint32_t w, uint32_t& lo, uint32_t& hi) {
  const uint32_t u = w ^ 0x80808080u;
  const uint32_t a = __byte_perm(u, 0x64646464u, 0x4140);
  const uint32_t b = __byte_perm(u, 0x64646464u, 0x4342);
  const __half2 k = __half2half2(__ushort_as_half((unsigned short)0x6480));  // 1152
  __half2 ha = __hsub2(*reinterpret_cast<const __half2*>(&a), k);
  __half2 hb = __hsub2(*reinterpret_cast<const __half2*>(&b), k);
  lo = *reinterpret_cast<uint32_t*>(&ha);
  hi = *reinterpret_cast<uint32_t*>(&hb);
}

// 8 int4 (nibble j = element j, two's complement) -> 8 f16 (exact): nibble ^ 8
// = q + 8, placed under 0x64 (1024 + q + 8), minus 1032.
__device__ __forceinline__ void i4x8_to_f16(uint32_t w, uint32_t (&o)[4]) {
  const uint32_t u = w ^ 0x88888888u;
  const uint32_t ev = u & 0x0F0F0F0Fu, od = (u >> 4) & 0x0F0F0F0Fu;
  const uint32_t p0 = __byte_perm(ev, od, 0x5140), p1 = __byte_perm(ev, od, 0x7362);
  const __half2 k = __half2half2(__ushort_as_half((unsigned short)0x6408));  // 1032
  const uint32_t q[4] = {__byte_perm(p0, 0x64646464u, 0x4140), __byte_perm(p0, 0x64646464u, 0x4342),
                         __byte_perm(p1, 0x64646464u, 0x4140), __byte_perm(p1, 0x64646464u, 0x4342)};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    __half2 h = __hsub2(*reinterpret_cast<const __half2*>(&q[i]), k);
    o[i] = *reinterpret_cast<uint32_t*>(&h);
  }
}

// 8 int4 -> 8 int8 (sign-extended bytes in element order).
__device__ __forceinline__ void i4x8_to_i8(uint32_t x, uint32_t& w0, uint32_t& w1) {
  uint32_t ev = x & 0x0F0F0F0Fu, od = (x >> 4) & 0x0F0F0F0Fu;
  ev |= (ev & 0x08080808u) * 0x1Eu;
  od |= (od & 0x08080808u) * 0x1Eu;
  w0 = __byte_perm(ev, od, 0x5140);
  w1 = __byte_perm(ev, od, 0x7362);
}

template <int BN, int KIND, int CONV, int NT>
__global__ void __launch_bounds__(ConvCfg<BN, CONV, NT>::NUM_THREADS, 1)
    zq_gemm2c_kernel(const __grid_constant__ CUtensorMap tmA0, const __grid_constant__ CUtensorMap tmA1,
                     const __grid_constant__ CUtensorMap tmB, const __grid_constant__ CUtensorMap tmC,
                     const GemmParams p) {
  using Cfg = ConvCfg<BN, CONV, NT>;
  constexpr int STAGES = Cfg::STAGES;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;                                       // STAGES x NT x [128 x 128 B]
  uint8_t* sB = smem + STAGES * NT * Cfg::A_BYTES;          // STAGES x [BN/2 x 128 B]
  uint8_t* sR = sB + STAGES * Cfg::B_BYTES;                 // STAGES x [BN/2 x RAW_ROW]
  uint8_t* sC = sR + STAGES * Cfg::RAW_BYTES;               // epilogue staging
  uint64_t* bars = reinterpret_cast<uint64_t*>(sC + Cfg::EPI_BYTES);
  uint64_t* full_bar = bars;                  // leader: producers + converters of both CTAs
  uint64_t* empty_bar = bars + STAGES;        // each: MMA commit (multicast)
  uint64_t* raw_bar = bars + 2 * STAGES;      // each: raw weight TMA bytes
  uint64_t* tfull_bar = bars + 3 * STAGES;    // each: accumulator ready (2)
  uint64_t* tempty_bar = bars + 3 * STAGES + 2;  // leader: epilogue warps of both CTAs (2)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * STAGES + 4);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank() & 1;
  const bool leader = rank == 0;
  const int unit0 = blockIdx.x >> 1, nunits_grid = gridDim.x >> 1;
  const int num_m_tiles = p.num_tiles / p.num_n_tiles;
  const int num_units = p.num_tiles;
  const int nkb = p.num_k_blocks;

  if (warp == 0 && lane == 0) {
    if (smem_u32(smem) & 1023) __trap();
    prefetch_tmap(&tmA0);
    if (NT > 1) prefetch_tmap(&tmA1);
    prefetch_tmap(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 2 + 2 * 4);
      mbar_init(&empty_bar[s], 1);
      mbar_init(&raw_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], 2 * kNumEpiWarps);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_cg2(tmem_slot, Cfg::TMEM_COLS);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  pdl_trigger();
  if (warp == 0) {
    // ===================== TMA producer (both CTAs) =====================
    int stage = 0, phase = 0;
    const int pre = unit0 < num_units ? (nkb < STAGES ? nkb : STAGES) : 0;
    if (lane == 0 && pre) {
      // the first unit's raw weight rows go out before the grid dependency resolves
      int mt, nt;
      tile_coords(unit0, num_m_tiles, p.num_n_tiles, p.group_m, mt, nt);
      for (int kb = 0; kb < pre; ++kb) {
        mbar_arrive_expect_tx(&raw_bar[kb], Cfg::RAW_BYTES);
        tma_load_2d(sR + kb * Cfg::RAW_BYTES, &tmB, &raw_bar[kb], kb * Cfg::RAW_ROW, nt * BN + rank * (BN / 2));
      }
    }
    pdl_wait();
    for (int u = unit0; u < num_units; u += nunits_grid) {
      int mt, nt;
      tile_coords(u, num_m_tiles, p.num_n_tiles, p.group_m, mt, nt);
      const int m0 = mt * (2 * BLOCK_M) + rank * BLOCK_M;
      const int n0 = nt * BN + rank * (BN / 2);
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&empty_bar[stage], phase ^ 1);
        if (lane == 0) {
          const uint32_t fb = leader_addr(&full_bar[stage]);
          if (leader)
            mbar_arrive_expect_tx(&full_bar[stage], 2 * NT * Cfg::A_BYTES);
          else
            mbar_arrive_cluster(fb);
          tma_load_2d_cg2(sA + (stage * NT) * Cfg::A_BYTES, &tmA0, fb, kb * Cfg::KB, m0);
          if (NT > 1) tma_load_2d_cg2(sA + (stage * NT + 1) * Cfg::A_BYTES, &tmA1, fb, kb * Cfg::KB, m0);
          if (!(u == unit0 && kb < pre)) {
            mbar_arrive_expect_tx(&raw_bar[stage], Cfg::RAW_BYTES);
            tma_load_2d(sR + stage * Cfg::RAW_BYTES, &tmB, &raw_bar[stage], kb * Cfg::RAW_ROW, n0);
          }
        }
        __syncwarp();
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (leader only) =====================
    if (leader) {
      constexpr uint32_t idesc = Cfg::F16 ? make_idesc_f16_kmajor(2 * BLOCK_M, BN) : make_idesc_i8(2 * BLOCK_M, BN);
      int stage = 0, phase = 0, acc = 0, acc_phase = 0;
      for (int u = unit0; u < num_units; u += nunits_grid) {
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          if (lane == 0) {
            const uint32_t b_addr = smem_u32(sB + stage * Cfg::B_BYTES);
#pragma unroll
            for (int t = 0; t < NT; ++t) {
              const uint32_t a_addr = smem_u32(sA + (stage * NT + t) * Cfg::A_BYTES);
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                const uint64_t ad = make_sw128_desc(a_addr + k * 32), bd = make_sw128_desc(b_addr + k * 32);
                if (Cfg::F16)
                  mma_f16_cg2(d_tmem, ad, bd, idesc, (kb | k | t) != 0);
                else
                  mma_i8_cg2(d_tmem, ad, bd, idesc, (kb | k) != 0);
              }
            }
            mma_commit_mc2(&empty_bar[stage], 0x3);
          }
          __syncwarp();
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (lane == 0) mma_commit_mc2(&tfull_bar[acc], 0x3);
        __syncwarp();
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else if (warp < 2 + kNumEpiWarps) {
    // ===================== epilogue (both CTAs, own 128 rows) =====================
    pdl_wait();
    const int quarter = warp & 3;
    const int half = (warp - 2) >> 2;
    constexpr int COLS = BN / 2;
    uint8_t* stage_c = sC + (warp - 2) * (Cfg::EPI_NB * 32 * 32 * 4);
    int sbuf = 0;
    if (p.tma_out && lane == 0) prefetch_tmap(&tmC);
    int acc = 0, acc_phase = 0;
    for (int u = unit0; u < num_units; u += nunits_grid) {
      int mt, nt;
      tile_coords(u, num_m_tiles, p.num_n_tiles, p.group_m, mt, nt);
      const int m0 = mt * (2 * BLOCK_M) + rank * BLOCK_M;
      const int n0 = nt * BN + half * COLS;
      const int row0 = m0 + quarter * 32;
      const int row = row0 + lane;
      float s_row = p.static_scale;
      if (KIND != OUT_S32 && p.token_scales != nullptr && row < p.M) s_row = __ldg(p.token_scales + row);
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const uint32_t t_row = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * BN + half * COLS;
#pragma unroll 1
      for (int c = 0; c < COLS; c += 32) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(t_row + c, r);
        tmem_ld_wait();
        if (c + 32 == COLS) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(leader_addr(&tempty_bar[acc]));
        }
        const int col0 = n0 + c;
        if (row0 >= p.M || col0 >= p.N) continue;
        if (p.tma_out) {
          uint8_t* sb = stage_c + sbuf * (32 * 32 * 4);
          if (lane == 0) {
            if (Cfg::EPI_NB == 2)
              bulk_wait_read1();
            else
              bulk_wait_read0();
          }
          __syncwarp();
          epi_chunk_smem<KIND, Cfg::F16>(r, s_row, p.row_scales, p.bias, col0, p.N, sb, lane);
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&tmC, sb, col0, row0);
            bulk_commit();
          }
          if (Cfg::EPI_NB == 2) sbuf ^= 1;
        } else if (row < p.M) {
          epi_chunk_slow<KIND, Cfg::F16>(r, s_row, p.row_scales, p.bias, p.out, (int64_t)row * p.ld_out, col0, p.N);
        }
      }
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
    if (lane == 0) bulk_wait0();
  } else {
    // ===================== converters (both CTAs) =====================
    const int ct = threadIdx.x - (2 + kNumEpiWarps) * 32;  // 0..127
    constexpr int CH = Cfg::RAW_ROW / 16;                   // 16-byte raw chunks per row
    int stage = 0, phase = 0;
    for (int u = unit0; u < num_units; u += nunits_grid) {
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&empty_bar[stage], phase ^ 1);
        mbar_wait(&raw_bar[stage], phase);
        const uint8_t* src = sR + stage * Cfg::RAW_BYTES;
        uint8_t* dst = sB + stage * Cfg::B_BYTES;
#pragma unroll 2
        for (int idx = ct; idx < (BN / 2) * CH; idx += 128) {
          const int r = idx / CH, c = idx % CH;
          const uint4 v = *reinterpret_cast<const uint4*>(src + r * Cfg::RAW_ROW + c * 16);
          uint8_t* drow = dst + r * 128;
          const int sw = r & 7;
          if (CONV == CONV_W8_F16) {
            uint32_t o[8];
            i8x4_to_f16(v.x, o[0], o[1]);
            i8x4_to_f16(v.y, o[2], o[3]);
            i8x4_to_f16(v.z, o[4], o[5]);
            i8x4_to_f16(v.w, o[6], o[7]);
            *reinterpret_cast<uint4*>(drow + (((2 * c) ^ sw) << 4)) = make_uint4(o[0], o[1], o[2], o[3]);
            *reinterpret_cast<uint4*>(drow + (((2 * c + 1) ^ sw) << 4)) = make_uint4(o[4], o[5], o[6], o[7]);
          } else if (CONV == CONV_W4_F16) {
            const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              uint32_t o[4];
              i4x8_to_f16(wv[i], o);
              *reinterpret_cast<uint4*>(drow + (((4 * c + i) ^ sw) << 4)) = make_uint4(o[0], o[1], o[2], o[3]);
            }
          } else {
            uint32_t o[8];
            i4x8_to_i8(v.x, o[0], o[1]);
            i4x8_to_i8(v.y, o[2], o[3]);
            i4x8_to_i8(v.z, o[4], o[5]);
            i4x8_to_i8(v.w, o[6], o[7]);
            *reinterpret_cast<uint4*>(drow + (((2 * c) ^ sw) << 4)) = make_uint4(o[0], o[1], o[2], o[3]);
            *reinterpret_cast<uint4*>(drow + (((2 * c + 1) ^ sw) << 4)) = make_uint4(o[4], o[5], o[6], o[7]);
          }
        }
        // generic-proxy smem writes -> visible to the async proxy (tcgen05 reads this
        // CTA's tile directly or, for the peer, through the pair), then one arrive
        // on the leader's barrier.  An explicit .release.cluster arrive compiles to
        // MEMBAR.ALL.GPU (~1 us per stage under load: 619 TF/s at NeoX QKV); the
        // proxy fence's MEMBAR.ALL.CTA already completes the writes to this CTA's
        // own shared memory before the arrive is issued.
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(leader_addr(&full_bar[stage]));
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 1) tmem_dealloc_cg2(tmem_base, Cfg::TMEM_COLS);
}

// ---------------------------------------------------------------------------
// Activation split for the weight-only path: per row, e = 141 - exponent(max|x|)
// puts the row max in [2^14, 2^15) (an exact power-of-two scaling, so no f16
// overflow whatever the activation range); hi = f16(x * 2^e), lo = f16(x * 2^e
// - hi); row_inv = 2^-e is folded back in the epilogue.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) act_split16_kernel(const float* __restrict__ x, int64_t ld_x, int64_t M,
                                                          int64_t K, int terms, __half* __restrict__ hi,
                                                          __half* __restrict__ lo, int64_t ld_h,
                                                          float* __restrict__ row_inv,
                                                          int32_t* __restrict__ flag) {
  __shared__ uint32_t red[32];
  pdl_wait();
  pdl_trigger();
  const bool vec = ((ld_x & 3) == 0) && ((reinterpret_cast<uintptr_t>(x) & 15) == 0) && ((K & 3) == 0) &&
                   ((ld_h & 3) == 0) && ((reinterpret_cast<uintptr_t>(hi) & 7) == 0) &&
                   (lo == nullptr || (reinterpret_cast<uintptr_t>(lo) & 7) == 0);
  for (int64_t row = blockIdx.x; row < M; row += gridDim.x) {
    const float* xr = x + row * ld_x;
    uint32_t m = 0;
    if (vec) {
      for (int64_t j = threadIdx.x * 4; j < K; j += 1024) {
        const float4 v = *reinterpret_cast<const float4*>(xr + j);
        m = max(m, max(max(abs_bits(v.x), abs_bits(v.y)), max(abs_bits(v.z), abs_bits(v.w))));
      }
    } else {
      for (int64_t j = threadIdx.x; j < K; j += 256) m = max(m, abs_bits(xr[j]));
    }
    const uint32_t mb = __float_as_uint(block_max_nonneg(__uint_as_float(m), red));
    if (mb >= 0x7f800000u && flag != nullptr && threadIdx.x == 0) atomicExch(flag, 1);
    int E = (int)(mb >> 23);
    if (E > 254) E = 254;
    int e = 141 - E;  // max * 2^e in [2^14, 2^15) for normal max
    if (e > 127) e = 127;
    const float sc = __uint_as_float((uint32_t)(e + 127) << 23);
    if (threadIdx.x == 0) row_inv[row] = ldexpf(1.0f, -e);
    __half* hr = hi + row * ld_h;
    __half* lr = lo ? lo + row * ld_h : nullptr;
    if (vec) {
      for (int64_t j = threadIdx.x * 4; j < K; j += 1024) {
        const float4 v = *reinterpret_cast<const float4*>(xr + j);
        const float s[4] = {__fmul_rn(v.x, sc), __fmul_rn(v.y, sc), __fmul_rn(v.z, sc), __fmul_rn(v.w, sc)};
        __half2 h0 = __floats2half2_rn(s[0], s[1]), h1 = __floats2half2_rn(s[2], s[3]);
        uint2 hv;
        hv.x = *reinterpret_cast<uint32_t*>(&h0);
        hv.y = *reinterpret_cast<uint32_t*>(&h1);
        *reinterpret_cast<uint2*>(hr + j) = hv;
        if (lr) {
          const float2 f0 = __half22float2(h0), f1 = __half22float2(h1);
          __half2 l0 = __floats2half2_rn(__fsub_rn(s[0], f0.x), __fsub_rn(s[1], f0.y));
          __half2 l1 = __floats2half2_rn(__fsub_rn(s[2], f1.x), __fsub_rn(s[3], f1.y));
          uint2 lv;
          lv.x = *reinterpret_cast<uint32_t*>(&l0);
          lv.y = *reinterpret_cast<uint32_t*>(&l1);
          *reinterpret_cast<uint2*>(lr + j) = lv;
        }
      }
    } else {
      for (int64_t j = threadIdx.x; j < K; j += 256) {
        const float s = __fmul_rn(xr[j], sc);
        const __half h = __float2half_rn(s);
        hr[j] = h;
        if (lr) lr[j] = __float2half_rn(__fsub_rn(s, __half2float(h)));
      }
    }
  }
  (void)terms;
}

// ---------------------------------------------------------------------------
// host
// ---------------------------------------------------------------------------
template <int BN, int KIND, int CONV, int NT>
static int launch_conv_t(const CUtensorMap& ta0, const CUtensorMap& ta1, const CUtensorMap& tb,
                         const CUtensorMap& tc, const GemmParams& p, cudaStream_t st) {
  using Cfg = ConvCfg<BN, CONV, NT>;
  static ZqDeviceOnce attr_once;
  attr_once([&](int) {
    cudaFuncSetAttribute(zq_gemm2c_kernel<BN, KIND, CONV, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         Cfg::SMEM_BYTES);
  });
  const int pairs = zq_num_sms() / 2;
  const int units = p.num_tiles < pairs ? p.num_tiles : pairs;
  const cudaError_t e = launch_kernel(zq_gemm2c_kernel<BN, KIND, CONV, NT>, dim3(2 * units),
                                      dim3(Cfg::NUM_THREADS), Cfg::SMEM_BYTES, st, 2, ta0, ta1, tb, tc, p);
  if (e != cudaSuccess) {
    set_error("tcgen05 converted-weight pair gemm launch: %s", cudaGetErrorString(e));
    return ZQ_ERR_CUDA;
  }
  return ZQ_OK;
}

// Output tensor map (32 x 32 boxes, clipped at M / N) when the output, scales
// and bias are 16-byte aligned; otherwise the epilogue stores element-wise.
static void make_out_map(GemmParams& p, int kind, CUtensorMap* tc) {
  memset(tc, 0, sizeof(*tc));
  const int esz = (kind == OUT_F16 || kind == OUT_BF16) ? 2 : 4;
  p.tma_out = ((reinterpret_cast<uintptr_t>(p.out) & 15) == 0) && ((p.ld_out * esz) % 16 == 0) &&
              (p.row_scales == nullptr || (reinterpret_cast<uintptr_t>(p.row_scales) & 15) == 0) &&
              (p.bias == nullptr || (reinterpret_cast<uintptr_t>(p.bias) & 15) == 0);
  if (!p.tma_out) return;
  const CUtensorMapDataType dt = kind == OUT_S32   ? CU_TENSOR_MAP_DATA_TYPE_INT32
                                 : kind == OUT_F32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                 : kind == OUT_F16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16
                                                   : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  if (make_tmap_2d(tc, dt, p.out, p.M, p.N, p.ld_out * esz, 32, 32,
                   esz == 4 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                   CU_TENSOR_MAP_L2_PROMOTION_NONE) != ZQ_OK) {
    p.tma_out = 0;
    cudaGetLastError();
  }
}

#define ZQ_CONV_KINDS(BN_, CONV_, NT_)                                                           \
  switch (kind) {                                                                                \
    case OUT_S32: return launch_conv_t<BN_, OUT_S32, CONV_, NT_>(ta0, ta1, tb, tc, p, st);        \
    case OUT_F32: return launch_conv_t<BN_, OUT_F32, CONV_, NT_>(ta0, ta1, tb, tc, p, st);        \
    case OUT_F16: return launch_conv_t<BN_, OUT_F16, CONV_, NT_>(ta0, ta1, tb, tc, p, st);        \
    default: return launch_conv_t<BN_, OUT_BF16, CONV_, NT_>(ta0, ta1, tb, tc, p, st);            \
  }

// W4A8 CTA-pair GEMM (called from zq_gemm.cu's dispatcher): `p` carries the
// scales / bias / output; the A map is the int8 activation map (128 x 128 B
// boxes), `wq` the packed INT4 rows (ld_w / 2 bytes each).
int gemm2c_w4i8(const int8_t* xq, int64_t ld_x, const void* wq, int64_t ld_w, int64_t M, int64_t N, int64_t K,
                int kind, int bn, GemmParams p, cudaStream_t st) {
  CUtensorMap ta0, tb, tc;
  int rc = make_tmap_2d(&ta0, CU_TENSOR_MAP_DATA_TYPE_UINT8, xq, M, K, ld_x, 128, BLOCK_M,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
  if (rc) return rc;
  rc = make_tmap_2d(&tb, CU_TENSOR_MAP_DATA_TYPE_UINT8, wq, N, ld_w / 2, ld_w / 2, 64, bn / 2,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
  if (rc) return rc;
  const CUtensorMap& ta1 = ta0;
  p.M = (int)M;
  p.N = (int)N;
  p.K = (int)K;
  make_out_map(p, kind, &tc);
  p.num_n_tiles = (int)((N + bn - 1) / bn);
  p.num_tiles = (int)((M + 255) / 256) * p.num_n_tiles;
  p.num_k_blocks = (int)((K + 127) / 128);
  p.group_m = K >= 2048 ? 8 : 1;
  if (bn == 256) ZQ_CONV_KINDS(256, CONV_W4_I8, 1)
  ZQ_CONV_KINDS(128, CONV_W4_I8, 1)
}

}  // namespace zq

using namespace zq;

extern "C" {

int zq_act_split16(const float* x, int64_t ld_x, int64_t M, int64_t K, int terms, void* hi, void* lo,
                   int64_t ld_h, float* row_inv, int32_t* nonfinite_flag, void* stream) {
  ZQ_CHECK_ARG(terms == 1 || terms == 2, ZQ_ERR_USAGE, "terms must be 1 or 2, got %d", terms);
  ZQ_CHECK_ARG(M >= 1 && K >= 1 && ld_x >= K && ld_h >= K, ZQ_ERR_SHAPE, "bad split shape");
  ZQ_CHECK_ARG(terms == 1 || lo != nullptr, ZQ_ERR_USAGE, "two-term split needs a lo buffer");
  int grid = (int)std::min<int64_t>(M, (int64_t)zq_num_sms() * 8);
  const cudaError_t e =
      launch_kernel(act_split16_kernel, dim3(grid), dim3(256), 0, reinterpret_cast<cudaStream_t>(stream), 1, x, ld_x,
                    M, K, terms, reinterpret_cast<__half*>(hi), terms == 2 ? reinterpret_cast<__half*>(lo) : nullptr,
                    ld_h, row_inv, nonfinite_flag);
  if (e != cudaSuccess) {
    set_error("act split launch: %s", cudaGetErrorString(e));
    return ZQ_ERR_CUDA;
  }
  return ZQ_OK;
}

int zq_linear_wo(const void* a_hi, const void* a_lo, int64_t ld_a, const float* row_inv, const void* wq,
                 int64_t ld_w, int w_bits, const float* w_row_scales, const float* bias, int64_t M, int64_t N,
                 int64_t K, void* out, int64_t ld_out, int out_type, void* stream) {
  ZQ_CHECK_ARG(w_bits == 8 || w_bits == 4, ZQ_ERR_USAGE, "unsupported weight bit width %d", w_bits);
  ZQ_CHECK_ARG(out_type >= ZQ_OUT_F32 && out_type <= ZQ_OUT_BF16, ZQ_ERR_USAGE, "bad output type %d", out_type);
  ZQ_CHECK_ARG(M >= 1 && N >= 1 && K >= 1 && ld_a >= K && ld_w >= K && ld_out >= N, ZQ_ERR_SHAPE,
               "bad weight-only linear shape");
  ZQ_CHECK_ARG((ld_a * 2) % 16 == 0 && (reinterpret_cast<uintptr_t>(a_hi) & 15) == 0 &&
                   (a_lo == nullptr || (reinterpret_cast<uintptr_t>(a_lo) & 15) == 0),
               ZQ_ERR_USAGE, "activation terms need 16-byte aligned rows");
  ZQ_CHECK_ARG(ld_w % 32 == 0 && (reinterpret_cast<uintptr_t>(wq) & 15) == 0, ZQ_ERR_USAGE,
               "weight rows must be 32-element aligned");
  ZQ_CHECK_ARG(w_row_scales != nullptr && row_inv != nullptr, ZQ_ERR_USAGE, "scales required");
  const int NT = a_lo ? 2 : 1;
  const int kind = out_type + 1;  // ZQ_OUT_F32/F16/BF16 -> OUT_F32/F16/BF16
  CUtensorMap ta0, ta1, tb, tc;
  int rc = make_tmap_2d(&ta0, CU_TENSOR_MAP_DATA_TYPE_UINT16, a_hi, M, K, ld_a * 2, 64, BLOCK_M,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
  if (rc) return rc;
  ta1 = ta0;
  if (NT == 2) {
    rc = make_tmap_2d(&ta1, CU_TENSOR_MAP_DATA_TYPE_UINT16, a_lo, M, K, ld_a * 2, 64, BLOCK_M,
                      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
    if (rc) return rc;
  }
  if (w_bits == 8)
    rc = make_tmap_2d(&tb, CU_TENSOR_MAP_DATA_TYPE_UINT8, wq, N, K, ld_w, 64, 128, CU_TENSOR_MAP_SWIZZLE_NONE,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
  else
    rc = make_tmap_2d(&tb, CU_TENSOR_MAP_DATA_TYPE_UINT8, wq, N, (K + 1) / 2, ld_w / 2, 32, 128,
                      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
  if (rc) return rc;
  GemmParams p;
  memset(&p, 0, sizeof(p));
  p.M = (int)M;
  p.N = (int)N;
  p.K = (int)K;
  p.out = out;
  p.ld_out = ld_out;
  p.token_scales = row_inv;
  p.static_scale = 1.0f;
  p.row_scales = w_row_scales;
  p.bias = bias;
  make_out_map(p, kind, &tc);
  p.num_n_tiles = (int)((N + 255) / 256);
  p.num_tiles = (int)((M + 255) / 256) * p.num_n_tiles;
  p.num_k_blocks = (int)((K + 63) / 64);
  p.group_m = 8;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (w_bits == 8) {
    if (NT == 1) ZQ_CONV_KINDS(256, CONV_W8_F16, 1)
    ZQ_CONV_KINDS(256, CONV_W8_F16, 2)
  }
  if (NT == 1) ZQ_CONV_KINDS(256, CONV_W4_F16, 1)
  ZQ_CONV_KINDS(256, CONV_W4_F16, 2)
}

}  // extern "C"
