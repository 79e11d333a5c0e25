// tcgen05 / TMEM / TMA GEMM for sm_100a:   C[M, N] = A[M, K] . B[N, K]^T
//
// A (activations) and B (weights, stored N x K "K-major", i.e. the transpose
// of the reference's (d_in, d_out) row-major W, model.py:152-165) are bf16;
// the accumulator is fp32 in TMEM. One CTA computes a 128 x BN tile:
//   warp 0     TMA producer (one elected lane), STAGES-deep smem ring
//   warp 1     TMEM allocator + MMA issuer (one elected lane)
//   warps 2-5  epilogue: tcgen05.ld 32 rows x 32 cols per warp per chunk,
//              then a fused epilogue functor (bias / ReLU / residual / vocab
//              softmax statistics) writes straight to global memory.
#pragma once
#include "sm100_ptx.cuh"

namespace hrt {

constexpr int TC_BM = 128;
constexpr int TC_BK = 64;  // 64 bf16 = 128 B rows -> SWIZZLE_128B
constexpr int TC_THREADS = 192;

template <int BN, int STAGES>
struct TcSmem {
  static constexpr int A_BYTES = TC_BM * TC_BK * 2;
  static constexpr int B_BYTES = BN * TC_BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int BAR_OFFSET = STAGES * STAGE_BYTES;
  static constexpr int TOTAL = BAR_OFFSET + 256 + 1024;  // barriers + alignment slack
};

template <int BN>
__host__ __device__ constexpr int tmem_cols_for() {
  return BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256;
}

// Epilogue functor protocol (all methods const, called per epilogue thread):
//   struct State;                                   per-thread scratch
//   begin(State&, int row, int n0)                  row < M only
//   chunk(State&, int row, int col0, const float* v, int nvalid)
//   end(State&, int row, int n0)
template <int BN, int STAGES, class Epi>
__global__ void __launch_bounds__(TC_THREADS, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M, int N,
                   int K, const int* __restrict__ M_dev, Epi epi) {
  using L = TcSmem<BN, STAGES>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::BAR_OFFSET);
  uint64_t* empty = full + STAGES;
  uint64_t* tmem_full = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

  if (M_dev != nullptr) M = *M_dev;
  const int m0 = blockIdx.y * TC_BM;
  const int n0 = blockIdx.x * BN;
  if (m0 >= M) return;  // whole CTA uniform: nothing allocated yet

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int num_kb = K / TC_BK;
  constexpr uint32_t TMEM_COLS = tmem_cols_for<BN>();

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tmem_full, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ===== TMA producer =====
      const uint64_t pol_w = policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      for (int kb = 0; kb < num_kb; ++kb) {
        mbar_wait(&empty[stage], phase ^ 1);
        uint8_t* sa = smem + stage * L::STAGE_BYTES;
        uint8_t* sb = sa + L::A_BYTES;
        mbar_arrive_expect_tx(&full[stage], L::STAGE_BYTES);
        tma_load_2d(sa, &tmA, &full[stage], kb * TC_BK, m0);
        tma_load_2d_hint(sb, &tmB, &full[stage], kb * TC_BK, n0, pol_w);
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ===== MMA issuer =====
      constexpr uint32_t idesc = idesc_bf16_f32(TC_BM, BN);
      int stage = 0;
      uint32_t phase = 0;
      for (int kb = 0; kb < num_kb; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        const uint32_t sa = smem_u32(smem + stage * L::STAGE_BYTES);
        const uint32_t sb = sa + L::A_BYTES;
#pragma unroll
        for (int k = 0; k < TC_BK / 16; ++k) {
          // advance 16 bf16 = 32 B along K inside the 128 B swizzle atom
          tc_mma_f16(tmem_base, sdesc_kmajor_sw128(sa + k * 32), sdesc_kmajor_sw128(sb + k * 32), idesc,
                     (kb | k) != 0);
        }
        tc_commit(&empty[stage]);
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
      tc_commit(tmem_full);
    }
  } else {
    // ===== epilogue warps 2..5 =====
    const int quarter = warp & 3;  // TMEM lane quarter this warp may access
    const int row = m0 + quarter * 32 + lane;
    mbar_wait(tmem_full, 0);
    tc_fence_after();
    typename Epi::State st;
    const bool live = row < M;
    if (live) epi.begin(st, row, n0);
#pragma unroll 1
    for (int c = 0; c < BN; c += 32) {
      float v[32];
      tmem_ld32(tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + c, v);
      const int col0 = n0 + c;
      int nvalid = N - col0;
      nvalid = nvalid > 32 ? 32 : nvalid;
      if (live && nvalid > 0) epi.chunk(st, row, col0, v, nvalid);
    }
    if (live) epi.end(st, row, n0);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, TMEM_COLS);
  }
}

}  // namespace hrt
