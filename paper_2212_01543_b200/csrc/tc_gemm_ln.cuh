// Residual projection with the following LayerNorm fused into the tcgen05
// GEMM epilogue (the north star's "residual+LayerNorm epilogue"):
//
//     x[M, d] += A[M, K] . W[d, K]^T + bias          (infer.py:204-205, :210-212)
//     y[M, d]  = LN(x) * g + b   (bf16, optionally    (kernels.py:42-57)
//                gathered to rows out_row[r])
//
// A LayerNorm needs whole rows, and a d = 512 row spans two 256-column
// accumulator tiles. The d / 256 CTAs that own one 128-row block form a
// thread-block cluster along N (NC = d / 256 in {1, 2, 4}); each computes its
// 128 x 256 tile exactly as tc_gemm_kernel does (TMA ring, one elected MMA
// lane, two TMEM accumulators), then the epilogue
//   pass 1  acc + bias + x -> x (fp32, coalesced through a per-warp smem
//           transpose as in tc_gemm_kernel); per-row partial mean / M2 over the
//           warp's 128 columns (Chan merge of 32-column chunks, lane-group
//           shuffles); the TMEM accumulator is released right after;
//   swap    each warp stages its 32 row partials in shared memory, and one
//           lane copies them into every other cluster CTA's shared memory
//           (DSMEM, st.shared::cluster) and arrives on every CTA's mbarrier
//           (release.cluster; one arrival per warp), then waits on its own
//           (acquire.cluster);
//   pass 2  merges the 2 NC partials of each row in a fixed order, re-reads
//           the updated rows (just written: L2 hits) and writes
//           y = (x - mean) rstd g + b as bf16.
// No LayerNorm launch and no DRAM re-read of x. Stats buffers and their
// barriers alternate by tile parity, so a CTA one tile ahead never overwrites
// statistics its peer has not read (and never arrives on a phase in flight).
#pragma once
#include "common.cuh"
#include "sm100_ptx.cuh"
#include "tc_gemm.cuh"

namespace hrt {

constexpr int TL_BN = 256;

template <int NC, int STAGES>
struct TlSmem {
  static constexpr int A_BYTES = TC_BM * TC_BK * 2;
  static constexpr int B_BYTES = TL_BN * TC_BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STG_OFFSET = STAGES * STAGE_BYTES;   // per-warp 32 x 32 fp32 transpose buffers
  static constexpr int STG_BYTES = TC_EPI_WARPS * 32 * TC_STG_LD * 4;
  static constexpr int ST_OFFSET = STG_OFFSET + STG_BYTES;  // row statistics [2][2 NC][128] float2
  static constexpr int ST_BYTES = 2 * 2 * NC * TC_BM * 8;
  static constexpr int BAR_OFFSET = ST_OFFSET + ST_BYTES;
  static constexpr int TOTAL = BAR_OFFSET + 256 + 1024;
};

__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t"
      ".reg .pred P1;\n\t"
      "LAB_WAITC:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONEC;\n\t"
      "bra LAB_WAITC;\n\t"
      "DONEC:\n\t"
      "}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// running (count, mean, M2) += a block of n values with mean bm and M2 bq (Chan et al.)
__device__ __forceinline__ void chan_merge(float& n, float& mean, float& m2, float bn, float bm, float bq) {
  const float nt = n + bn;
  const float delta = bm - mean;
  mean += delta * (bn / nt);
  m2 += bq + delta * delta * (n * bn / nt);
  n = nt;
}

struct ResLnArgs {
  float* x;          // [M][d] fp32 residual stream (read-modify-write)
  int ldx;
  const float* bias;  // [d]
  const float* g;     // LayerNorm gain / bias [d]
  const float* b;
  bf16* y;            // [*][d] normalised rows (bf16 GEMM operand)
  int ldy;
  const int* out_row;  // nullable: y row of x row r (< 0: not written)
};

template <int NC, int STAGES>
__global__ void __launch_bounds__(TC_THREADS, 1)
    tc_gemm_resln_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M,
                         int K, const int* __restrict__ M_dev, ResLnArgs ep) {
  using L = TlSmem<NC, STAGES>;
  constexpr int D = NC * TL_BN;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float2* stats = reinterpret_cast<float2*>(smem + L::ST_OFFSET);  // [buf][2 NC][128]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::BAR_OFFSET);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;  // [2]
  uint64_t* tempty = tfull + 2;      // [2]
  uint64_t* lnbar = tempty + 2;      // [2] row-statistics exchange, by tile parity
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(lnbar + 2);

  pdl_trigger();
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int num_kb = K / TC_BK;
  const int crank = NC > 1 ? (int)cluster_ctarank() : 0;
  const int cid = blockIdx.x / NC, ncl = gridDim.x / NC;
  const int n0 = crank * TL_BN;
  constexpr uint32_t TMEM_COLS = 512;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], TC_EPI_WARPS);
      mbar_init(&lnbar[a], NC * TC_EPI_WARPS);  // one arrival per epilogue warp of every cluster CTA
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, TMEM_COLS);
  tc_fence_before();
  if constexpr (NC > 1)
    cluster_sync_all();  // every peer's barriers are initialised before any remote arrive
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  // the first STAGES weight tiles do not depend on the previous kernel
  int pre = 0;
  if (warp == 0 && lane == 0) {
    pre = min(STAGES, num_kb);
    const uint64_t pol = policy_evict_last();
    for (int s2 = 0; s2 < pre; ++s2) {
      mbar_arrive_expect_tx(&full[s2], L::STAGE_BYTES);
      tma_load_2d_hint(smem + s2 * L::STAGE_BYTES + L::A_BYTES, &tmB, &full[s2], s2 * TC_BK, n0, pol);
    }
  }
  pdl_wait();
  if (M_dev != nullptr) M = *M_dev;
  const int num_units = (M + TC_BM - 1) / TC_BM;  // 128-row blocks; every cluster CTA walks the same ones

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol_w = policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      for (int u = cid; u < num_units; u += ncl) {
        const int m0 = u * TC_BM;
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * L::STAGE_BYTES;
          if (u == cid && kb < pre) {
            tma_load_2d(sa, &tmA, &full[stage], kb * TC_BK, m0);
          } else {
            mbar_arrive_expect_tx(&full[stage], L::STAGE_BYTES);
            tma_load_2d(sa, &tmA, &full[stage], kb * TC_BK, m0);
            tma_load_2d_hint(sa + L::A_BYTES, &tmB, &full[stage], kb * TC_BK, n0, pol_w);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      if (cid >= num_units) {  // no rows after all: the armed stages still expect their A tiles
        for (int s2 = 0; s2 < pre; ++s2) tma_load_2d(smem + s2 * L::STAGE_BYTES, &tmA, &full[s2], s2 * TC_BK, 0);
        for (int s2 = 0; s2 < pre; ++s2) mbar_wait(&full[s2], 0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_bf16_f32(TC_BM, TL_BN);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int u = cid; u < num_units; u += ncl, ++it) {
        const int acc = it & 1;
        mbar_wait(&tempty[acc], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * TL_BN;
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * L::STAGE_BYTES);
          const uint32_t sb = sa + L::A_BYTES;
#pragma unroll
          for (int k = 0; k < TC_BK / 16; ++k)
            tc_mma_f16(d_tmem, sdesc_kmajor_sw128(sa + k * 32), sdesc_kmajor_sw128(sb + k * 32), idesc,
                       (kb | k) != 0);
          tc_commit(&empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        tc_commit(&tfull[acc]);
      }
    }
  } else {
    // ===== epilogue: 8 warps, warp (quarter q, half h) owns rows 32 q .. 32 q + 31, columns 128 h .. +127.
    // Each 32 x 32 accumulator chunk is transposed through a per-warp smem buffer (as in
    // tc_gemm_kernel) so every global access is a coalesced 4-row x 128-byte group: lane
    // (g = lane / 8, c = lane % 8) holds rows g + 4 i (i < 8), columns 4 c .. 4 c + 3.
    const int ew = warp - 2;
    const int quarter = warp & 3;
    const int half = ew >> 2;
    const int cbeg = half * (TL_BN / 2);
    const int pidx = crank * 2 + half;  // this warp's partial slot
    const int lg = lane >> 3, lc = lane & 7;
    float* stg = reinterpret_cast<float*>(smem + L::STG_OFFSET) + ew * (32 * TC_STG_LD);
    int it = 0;
    for (int u = cid; u < num_units; u += ncl, ++it) {
      const int acc = it & 1, buf = it & 1;
      const int rbase = u * TC_BM + quarter * 32;
      // residual rows of the first chunk are requested before the accumulator is ready;
      // every later chunk's are requested one chunk ahead (DRAM latency off the critical path)
      float4 xo[8];
      auto load_x = [&](int cc, float4 (&dst)[8]) {
        const int colx = n0 + cc + lc * 4;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int row = rbase + lg + 4 * i;
          dst[i] = row < M ? *reinterpret_cast<const float4*>(ep.x + (size_t)row * ep.ldx + colx)
                           : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      };
      load_x(cbeg, xo);
      mbar_wait(&tfull[acc], (it >> 1) & 1);
      tc_fence_after();
      const uint32_t tbase = tmem_base + acc * TL_BN + (static_cast<uint32_t>(quarter * 32) << 16);
      // ---- pass 1: x += acc + bias (coalesced), per-row partial (mean, M2) of this warp's 128 columns ----
      float cn[8], cmean[8], cm2[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) cn[i] = cmean[i] = cm2[i] = 0.f;
#pragma unroll 1
      for (int c = cbeg; c < cbeg + TL_BN / 2; c += 32) {
        float v[32];
        tmem_ld32(tbase + c, v);
        const uint32_t sbase = smem_u32(stg);
#pragma unroll
        for (int i = 0; i < 8; ++i)
          asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(
                           sbase + 4u * (lane * TC_STG_LD + 4 * (i ^ (lane & 7)))),
                       "f"(v[4 * i]), "f"(v[4 * i + 1]), "f"(v[4 * i + 2]), "f"(v[4 * i + 3])
                       : "memory");
        __syncwarp();
        float4 a[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int r = i * 4 + lg;
          asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                       : "=f"(a[i].x), "=f"(a[i].y), "=f"(a[i].z), "=f"(a[i].w)
                       : "r"(sbase + 4u * (r * TC_STG_LD + 4 * (lc ^ (r & 7))))
                       : "memory");
        }
        __syncwarp();
        const int col = n0 + c + lc * 4;
        const float4 bb = __ldg(reinterpret_cast<const float4*>(ep.bias + col));
        float4 xnext[8];
        if (c + 32 < cbeg + TL_BN / 2) load_x(c + 32, xnext);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int row = rbase + lg + 4 * i;
          float4 xn = xo[i];
          xn.x += a[i].x + bb.x;
          xn.y += a[i].y + bb.y;
          xn.z += a[i].z + bb.z;
          xn.w += a[i].w + bb.w;
          if (row < M) *reinterpret_cast<float4*>(ep.x + (size_t)row * ep.ldx + col) = xn;
          // chunk statistics of row (32 columns over the 8 lanes of this lane group)
          float sm = (xn.x + xn.y) + (xn.z + xn.w);
          sm += __shfl_xor_sync(0xffffffffu, sm, 1);
          sm += __shfl_xor_sync(0xffffffffu, sm, 2);
          sm += __shfl_xor_sync(0xffffffffu, sm, 4);
          const float bm = sm * (1.f / 32.f);
          const float e0 = xn.x - bm, e1 = xn.y - bm, e2 = xn.z - bm, e3 = xn.w - bm;
          float q = (e0 * e0 + e1 * e1) + (e2 * e2 + e3 * e3);
          q += __shfl_xor_sync(0xffffffffu, q, 1);
          q += __shfl_xor_sync(0xffffffffu, q, 2);
          q += __shfl_xor_sync(0xffffffffu, q, 4);
          chan_merge(cn[i], cmean[i], cm2[i], 32.f, bm, q);
        }
        if (c + 32 < cbeg + TL_BN / 2) {
#pragma unroll
          for (int i = 0; i < 8; ++i) xo[i] = xnext[i];
        }
      }
      // ---- exchange row partials across the cluster ----
      // lanes (g, 0) stage the warp's 32 row partials in local smem; lane 0 copies them
      // to every other cluster CTA (DSMEM) and arrives once per CTA (release.cluster)
      float2* sb = stats + (size_t)buf * (2 * NC * TC_BM);
      float2* mine = sb + pidx * TC_BM + quarter * 32;
      if (lc == 0) {
#pragma unroll
        for (int i = 0; i < 8; ++i) mine[lg + 4 * i] = make_float2(cmean[i], cm2[i]);
      }
      __syncwarp();
      const uint32_t barl = smem_u32(&lnbar[buf]);
      if (lane == 0) {
        const uint32_t src = smem_u32(mine);
#pragma unroll
        for (int r = 0; r < NC; ++r) {
          if (r == crank) continue;
          const uint32_t dst = mapa_shared(src, (uint32_t)r);
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            float4 v4;
            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                         : "=f"(v4.x), "=f"(v4.y), "=f"(v4.z), "=f"(v4.w)
                         : "r"(src + 16u * j));
            asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(dst + 16u * j), "f"(v4.x),
                         "f"(v4.y), "f"(v4.z), "f"(v4.w)
                         : "memory");
          }
        }
        // own barrier first (see header: no peer can reach this parity's next phase before it completes)
        mbar_arrive_cluster(mapa_shared(barl, (uint32_t)crank));
#pragma unroll
        for (int r = 0; r < NC; ++r)
          if (r != crank) mbar_arrive_cluster(mapa_shared(barl, (uint32_t)r));
      }
      // the accumulator is no longer needed: release it to the MMA warp now
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&tempty[acc]);
        mbar_wait_cluster(&lnbar[buf], (it >> 1) & 1);
      }
      __syncwarp();
      float mean[8], rstd[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float tn = 0.f, tmean = 0.f, tm2 = 0.f;
#pragma unroll
        for (int p = 0; p < 2 * NC; ++p) {
          const float2 st = sb[p * TC_BM + quarter * 32 + lg + 4 * i];
          chan_merge(tn, tmean, tm2, (float)(TL_BN / 2), st.x, st.y);
        }
        mean[i] = tmean;
        rstd[i] = 1.0f / sqrtf(tm2 / (float)D + 1e-5f);
      }
      // ---- pass 2: y = LN(x) for this warp's columns (x re-read from L2, coalesced) ----
      int orow[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int row = rbase + lg + 4 * i;
        orow[i] = row < M ? (ep.out_row ? ep.out_row[row] : row) : -1;
      }
      float4 xv[8];
      auto load_xn = [&](int cc, float4 (&dst)[8]) {
        const int colx = n0 + cc + lc * 4;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int row = rbase + lg + 4 * i;
          dst[i] = orow[i] >= 0 ? __ldcg(reinterpret_cast<const float4*>(ep.x + (size_t)row * ep.ldx + colx))
                                : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      };
      load_xn(cbeg, xv);
#pragma unroll 1
      for (int c = cbeg; c < cbeg + TL_BN / 2; c += 32) {
        const int col = n0 + c + lc * 4;
        const float4 gg = __ldg(reinterpret_cast<const float4*>(ep.g + col));
        const float4 bb = __ldg(reinterpret_cast<const float4*>(ep.b + col));
        float4 xnx[8];
        if (c + 32 < cbeg + TL_BN / 2) load_xn(c + 32, xnx);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if (orow[i] < 0) continue;
          __nv_bfloat162 lo = __floats2bfloat162_rn((xv[i].x - mean[i]) * rstd[i] * gg.x + bb.x,
                                                    (xv[i].y - mean[i]) * rstd[i] * gg.y + bb.y);
          __nv_bfloat162 hi = __floats2bfloat162_rn((xv[i].z - mean[i]) * rstd[i] * gg.z + bb.z,
                                                    (xv[i].w - mean[i]) * rstd[i] * gg.w + bb.w);
          uint2 o;
          o.x = *reinterpret_cast<uint32_t*>(&lo);
          o.y = *reinterpret_cast<uint32_t*>(&hi);
          *reinterpret_cast<uint2*>(ep.y + (size_t)orow[i] * ep.ldy + col) = o;
        }
        if (c + 32 < cbeg + TL_BN / 2) {
#pragma unroll
          for (int i = 0; i < 8; ++i) xv[i] = xnx[i];
        }
      }
    }
  }
  tc_fence_before();
  if constexpr (NC > 1)
    cluster_sync_all();  // no CTA leaves while a peer may still write its statistics / barriers
  else
    __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, TMEM_COLS);
  }
}

}  // namespace hrt
