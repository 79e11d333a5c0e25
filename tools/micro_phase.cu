// Per-phase cost breakdown of the persistent decode kernel's building blocks
// (R = 1, d = 512): barrier alone, + residual projection (Wo), + LN projection (Qc),
// + attention, + vocab.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/micro_phase tools/micro_phase.cu
#include <cstdio>
#include <vector>
#include <cstring>

#include "../paper_2212_01543_b200/csrc/decode_mega.cuh"

using namespace hrt;

// instrumented copy of phase D (LN2 + Qc) for block 0 / thread 0
__device__ __noinline__ void ph_d_instr(const MegaParams& p, int R, bf16* act, float* red, uint4* pf, long long* out) {
  const MegaLayer& W = p.L[0];
  const int d = p.d;
  long long t0 = clock64();
  if (!MgSplit(d, d).cta_has_work()) return;
  mg_stage_ln(p.x, R, d, W.ln2g, W.ln2b, act, d + MG_APAD);
  long long t1 = clock64();
  cp_async_wait_all();
  long long t2 = clock64();
  const MgSplit sp(d, d);
  const int tile = sp.tile(0);
  float c[1][4] = {{0.f, 0.f, 0.f, 0.f}};
  long long t3 = 0, t4 = 0;
  if (tile < sp.ntiles) {
    mg_tile<1, false>(W.wqc, d, tile * 16, d - tile * 16, 0, sp.cpw, act, d + MG_APAD, pf, p.npf, c);
    t3 = clock64();
    const int lane = threadIdx.x & 31, g = lane >> 2, t4_ = lane & 3;
    if (2 * t4_ < R) p.q[(size_t)(2 * t4_) * d + tile * 16 + g] = __float2bfloat16_rn(c[0][0] + __ldg(W.bqc + tile * 16 + g));
    t4 = clock64();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    out[0] = t1 - t0;
    out[1] = t2 - t1;
    out[2] = t3 - t2;
    out[3] = t4 - t3;
  }
}

__global__ void __launch_bounds__(MG_THREADS, 1) k_phase(const __grid_constant__ MegaParams p, int mode, int iters,
                                                         int R) {
  extern __shared__ __align__(16) unsigned char msm_raw[];
  uint4* pf = reinterpret_cast<uint4*>(msm_raw) + (size_t)(threadIdx.x >> 5) * p.npf * 64;
  bf16* act = reinterpret_cast<bf16*>(reinterpret_cast<uint4*>(msm_raw) + (size_t)MG_WARPS * p.npf * 64);
  float* red = reinterpret_cast<float*>(act + (size_t)MG_RMAX * (p.ff + MG_APAD));
  unsigned target = 0;
  const int d = p.d, ff = p.ff;
  const MegaLayer& W = p.L[0];
  for (int i = 0; i < iters; ++i) {
    if (mode == 1) mg_ph_residual<1>(p, p.ctx, d, W.wo, W.bo, R, act, red, pf);
    if (mode == 2) mg_ph_ln_proj<1, false>(p, W.ln2g, W.ln2b, W.wqc, W.bqc, d, p.q, R, act, red, pf);
    if (mode == 3) mg_ph_attn<true>(p, 0, 20, R, red);
    if (mode == 4) mg_ph_vocab<1>(p, R, act, red, pf);
    if (mode == 5) mg_ph_residual<1>(p, p.hid, ff, W.w2, W.b2, R, act, red, pf);
    if (mode == 6) mg_ph_qkv<1>(p, 0, 5, R, R, true, act, red, pf);
    if (mode == 7) mg_ph_ln_proj<1, true>(p, W.ln3g, W.ln3b, W.w1, W.b1, ff, p.hid, R, act, red, pf);
    if (mode == 8) ph_d_instr(p, R, act, red, pf, reinterpret_cast<long long*>(p.veos) + 8);
    mg_arrive(p.bar);
    if (mode == 1) mg_prefetch_proj(W.wo, d, d, pf, p.npf);
    if (mode == 2 || mode == 8) mg_prefetch_proj(W.wqc, d, d, pf, p.npf);
    if (mode == 4) mg_prefetch_vocab(p, pf);
    if (mode == 5) mg_prefetch_proj(W.w2, d, ff, pf, p.npf);
    if (mode == 6) mg_prefetch_proj(W.wqkv, 3 * d, d, pf, p.npf);
    if (mode == 7) mg_prefetch_proj(W.w1, ff, d, pf, p.npf);
    target += gridDim.x;
    mg_wait(p.bar, target);
  }
}

__global__ void fill_rand(bf16* p, size_t n, unsigned seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    unsigned h = (unsigned)i * 2654435761u ^ seed;
    h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
    p[i] = __float2bfloat16((float)(h & 0xffff) / 65536.f - 0.5f);
  }
}
int main(int argc, char** argv) {
  const bool rnd = argc > 1;
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int d = 512, ff = 2048, V = 32000, cap = 257;
  MegaParams p{};
  p.d = d;
  p.ff = ff;
  p.H = 8;
  p.V = V;
  p.Ld = 1;
  p.cap = cap;
  p.k = 2;
  p.rcap = 32;
  p.npf = 8;
  p.att_scale = 0.125f;
  p.scale = 22.6f;
  auto balloc = [&](size_t n) {
    bf16* q;
    cudaMalloc(&q, n * 2);
    cudaMemset(q, 0, n * 2);
    if (rnd) fill_rand<<<1024, 256>>>(q, n, 12345u);
    return q;
  };
  auto falloc = [](size_t n) {
    float* q;
    cudaMalloc(&q, n * 4);
    cudaMemset(q, 0, n * 4);
    return q;
  };
  MegaLayer L{};
  L.wqkv = balloc(3 * d * d);
  L.wo = balloc(d * d);
  L.wqc = balloc(d * d);
  L.woc = balloc(d * d);
  L.w1 = balloc(ff * d);
  L.w2 = balloc(d * ff);
  L.bqkv = falloc(3 * d);
  L.bo = falloc(d);
  L.bqc = falloc(d);
  L.boc = falloc(d);
  L.b1 = falloc(ff);
  L.b2 = falloc(d);
  float* ones = falloc(d);
  std::vector<float> h1(d, 1.f);
  cudaMemcpy(ones, h1.data(), d * 4, cudaMemcpyHostToDevice);
  L.ln1g = L.ln2g = L.ln3g = ones;
  L.ln1b = L.ln2b = L.ln3b = falloc(d);
  p.L[0] = L;
  p.lng = ones;
  p.lnb = L.ln1b;
  p.E = balloc((size_t)V * d);
  p.x = falloc(32 * d);
  p.q = balloc(32 * d);
  p.ctx = balloc(32 * d);
  p.hid = balloc(32 * ff);
  p.kc = balloc((size_t)32 * cap * d);
  p.vc = balloc((size_t)32 * cap * d);
  float4* vp;
  cudaMalloc(&vp, 32 * sms * 16);
  p.vpart = vp;
  p.veos = falloc(64);
  unsigned* bar;
  cudaMalloc(&bar, 64);
  p.bar = bar;
  auto ialloc = [](size_t n) {
    int* q;
    cudaMalloc(&q, n * 4);
    cudaMemset(q, 0, n * 4);
    return q;
  };
  p.st.feed = ialloc(32);
  p.st.done = ialloc(32);
  p.st.nsteps = ialloc(32);
  p.st.forced = ialloc(32);
  p.st.anchors = ialloc(32 * cap);
  int* caps = ialloc(32);
  std::vector<int> hc(32, 100);
  cudaMemcpy(caps, hc.data(), 32 * 4, cudaMemcpyHostToDevice);
  p.st.caps = caps;
  p.st.cap = cap;
  double* sc;
  cudaMalloc(&sc, 32 * 8);
  p.st.score = sc;
  StepCtl* ctl;
  cudaMalloc(&ctl, sizeof(StepCtl));
  cudaMemset(ctl, 0, sizeof(StepCtl));
  p.ctl = ctl;
  p.pe = falloc((size_t)300 * d);
  {
    std::vector<float> hv(32 * sms * 4);
    for (size_t i = 0; i < hv.size(); i += 4) { hv[i] = 1.f; hv[i + 1] = 2.f; hv[i + 2] = 1.f; int id = 100 + (int)(i / 4) % 50; memcpy(&hv[i + 3], &id, 4); }
    cudaMemcpy(vp, hv.data(), hv.size() * 4, cudaMemcpyHostToDevice);
  }
  const size_t smem = mega_smem_bytes(d, ff, p.npf);
  cudaFuncSetAttribute(k_phase, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const char* names[] = {"barrier only", "C Wo residual", "D LN2+Qc", "B self-attn t=20", "I vocab",
                         "H W2 residual", "A select+QKV", "G LN3+W1", "D instrumented"};
  for (int R : {1})
    for (int mode = 0; mode < 9; ++mode) {
      const int it = 500;
      float ms = 0;
      for (int rep = 0; rep < 2; ++rep) {
        cudaMemset(bar, 0, 64);
        cudaEventRecord(a);
        k_phase<<<sms, MG_THREADS, smem>>>(p, mode, it, R);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
      }
      printf("%s R=%d %-22s %.3f us/iter\n", rnd ? "rand" : "zero", R, names[mode], 1000 * ms / it);
    }
  {
    long long h[4];
    cudaMemcpy(h, reinterpret_cast<long long*>(p.veos) + 8, 32, cudaMemcpyDeviceToHost);
    printf("D cycles: LN stage %lld, cp wait %lld, tile %lld, epilogue %lld\n", h[0], h[1], h[2], h[3]);
  }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
