// Cluster exchange latency probe (the register-tiled solve's line step without loads/FMAs):
// cluster of C CTAs x 16 warps; per step every tile warp sends one double per lane to the
// owner of block (warp % NB) (st.async + mbarrier complete_tx), owners sum NC contributions
// and broadcast 32 doubles to every CTA (st.async), everyone waits for the broadcast.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, unsigned r) { uint32_t o; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r)); return o; }
__device__ __forceinline__ void sta(uint32_t d, double v, uint32_t b) { asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(d), "d"(v), "r"(b) : "memory"); }
__device__ __forceinline__ void minit(uint64_t* b, int c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c) : "memory"); }
__device__ __forceinline__ void marm(uint64_t* b, uint32_t tx) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(tx) : "memory"); }
__device__ __forceinline__ void mwait(uint64_t* b, uint32_t par) { asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n" ::"r"(su32(b)), "r"(par) : "memory"); }
__device__ __forceinline__ unsigned crank() { unsigned r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
__device__ __forceinline__ void csync() { asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory"); }
constexpr int C = 4, NB = 3;  // blocks owned per CTA (warps 13..15), 13 tile warps
__global__ void __cluster_dims__(C, 1, 1) k(long long* cyc, int steps) {
  __shared__ uint64_t bb[NB], wb[2];
  __shared__ double slots[NB][16][32], w[2][C * NB * 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, r = crank();
  const int ntile = 16 - NB;
  // tile warp -> block (owner CTA ob, local block b); contributions per block from all CTAs
  const int tb = warp % NB, tc = (warp + r) % C;  // spread targets
  const int per_block = ntile * C / (C * NB) + 0;  // not exact; computed below
  __shared__ int ncontrib[NB];
  if (threadIdx.x == 0) {
    for (int b = 0; b < NB; ++b) ncontrib[b] = 0;
    // count contributions to my blocks: every CTA c, warp w < ntile sends to ((w + c) % C, w % NB)
    for (int c = 0; c < C; ++c) for (int ww = 0; ww < ntile; ++ww) if ((ww + c) % C == r) ncontrib[ww % NB]++;
    for (int b = 0; b < NB; ++b) minit(&bb[b], 1);
    minit(&wb[0], 1); minit(&wb[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  csync();
  long long t0 = clock64();
  double acc = lane;
  for (int t = 0; t < steps; ++t) {
    const int par = t & 1;
    if (t > 0) mwait(&wb[par], ((t - 1) >> 1) & 1);
    if (threadIdx.x == 0) marm(&wb[par ^ 1], 8u * 32 * C * NB);
    if (warp >= ntile && lane == 0) marm(&bb[warp - ntile], 256u * ncontrib[warp - ntile]);
    if (warp < ntile) {
      const double v = acc + w[par][(warp * 32 + lane) % (C * NB * 32)];
      // slot index: sender (c, w) -> unique index among the contributors of that block
      const int idx = (r * ntile + warp) / (C * NB) % 16;
      sta(mapa(su32(&slots[tb][idx][lane]), tc), v, mapa(su32(&bb[tb]), tc));
    } else {
      const int b = warp - ntile;
      mwait(&bb[b], par);
      double s = 0.0;
      for (int q = 0; q < ncontrib[b] && q < 16; ++q) s += slots[b][q][lane];
      const double wv = s * 1e-3;
      for (int c = 0; c < C; ++c) sta(mapa(su32(&w[par ^ 1][(r * NB + b) * 32 + lane]), c), wv, mapa(su32(&wb[par ^ 1]), c));
    }
  }
  mwait(&wb[steps & 1], ((steps - 1) >> 1) & 1);
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = (t1 - t0) / steps;
  csync();
}
int main() {
  long long* cyc; cudaMalloc(&cyc, 64);
  for (int grid : {4, 128}) {
    k<<<grid, 512>>>(cyc, 2000);
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("grid %d: %lld cycles per exchange step (%s)\n", grid, c, cudaGetErrorString(cudaDeviceSynchronize()));
  }
}
