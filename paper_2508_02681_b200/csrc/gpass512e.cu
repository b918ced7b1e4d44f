// gpass512e.cu — elastic G pass at N3 = 512 (config 4: 512^3, c = 3, periodic z), persistent CTAs.
// z FFT -> s_hat = G_hat r_hat (3x3 real-symmetric block per bin, Eq 46/49, App. B) and the
// Parseval partial of gamma_1 -> inverse z FFT (Alg 2 l.4-7), in place on the half
// spectrum [load][c][kx][z][y].
#include <cuda_runtime.h>

#include "common.cuh"
#include "fft.cuh"
#include "kernels.cuh"
#include "dev_common.cuh"

namespace uno {

// Elastic G pass at N3 = 512 (config 4), persistent: the three 64 KB component tiles (8 y columns
// x 512 z each) fill the SM's shared memory (one CTA per SM), so load / compute / store can only
// overlap inside the CTA.  Each CTA walks tiles blockIdx.x, blockIdx.x + gridDim.x, ...; as soon as
// component q of the current tile has been stored, the cp.async copies of component q of the NEXT
// tile start into the same buffer (one commit group per component) and a third of the next tile's
// symbol rows is prefetched into L2 — they land while the inverse stages of the other components,
// the stores and the next tile's first forward stages run.
// 256 threads, two radix-8 butterflies per thread in every Stockham stage (512 = 8 . 8 . 8): the
// fused middle stage (last forward stage -> 3x3 symbol multiply -> first inverse stage, all on
// registers) holds 3 components x 8 bins x 2 items = 192 registers of data, which fits the
// 255-register budget of a 256-thread CTA without spills; with 512 threads and 128 registers the
// same stage spills, and the local-memory traffic (only ~28 KB of L1 is left next to 200 KB of
// shared memory) cost more than the pipelining gained (measured: 3.70 ms vs 3.45 ms one tile per
// CTA).  Same tile shape and per-tile gamma partials as gpass_z_kernel<512, 3>.
#ifndef UNO_G512E_PERSIST
#define UNO_G512E_PERSIST 1  // 0: A/B builds only (the one-tile-per-CTA gpass_z_kernel<512, 3>)
#endif
constexpr int kG512ePersistCTAs = 148;
namespace g5e {
constexpr int L = 512, NC = 3, T = 256, R = 8, NJ = L / R, NH = NJ * kTile / T;  // NH = 2 items per thread
static_assert(NH == 2 && pick_radix(512) == 8 && pick_radix(64) == 8 && pick_radix(8) == 8, "512 = 8.8.8");

struct Args {
  double2* spec;       // component 0 of this load
  const double* gtab;  // symbol entries [6][nspec]
  long long nspec;
  int N2, N3, M, ntile_y;
};
__device__ __forceinline__ long long tile_off(const Args& a, int tile) {
  const int kx = tile / a.ntile_y;
  return (long long)kx * a.N3 * a.N2 + (tile - kx * a.ntile_y) * 8;
}
// copies of component q of the tile at boff (one commit group) + symbol entries 2q, 2q + 1 -> L2
__device__ __forceinline__ void issue(const Args& a, double2* tile_q, int q, long long boff) {
  const int t = threadIdx.x;
  const double2* base = a.spec + q * a.nspec + boff;
#pragma unroll
  for (int i = 0; i < 8 * L / T; ++i) {
    const int e = t + i * T;
    cp_async16(&tile_q[tidx(e >> 3, e & 7)], base + (long long)(e >> 3) * a.N2 + (e & 7));
  }
  cp_commit();
#pragma unroll
  for (int i = 0; i < 2 * L / T; ++i) {
    const int r = t + i * T, ent = 2 * q + r / L, kz = r & (L - 1);
    asm volatile("prefetch.global.L2 [%0];\n" ::"l"(a.gtab + ent * a.nspec + boff + (long long)kz * a.N2));
  }
}
// One radix-8 Stockham stage of span NS over the 8 columns of one component tile, in place
// (fft.cuh fft_stage with two items per thread: j = t / 8 and t / 8 + 32).
template <int NS, bool INV>
__device__ __forceinline__ void stage(double2* s, const double2* __restrict__ tw) {
  const int t = threadIdx.x, c = t & 7, j0 = t >> 3;
  double2 v[NH][R];
#pragma unroll
  for (int h = 0; h < NH; ++h) {
    const int j = j0 + h * (T / 8), k = j % NS;
#pragma unroll
    for (int r = 0; r < R; ++r) v[h][r] = s[tidx(j + r * NJ, c)];
    if (NS > 1) {
#pragma unroll
      for (int r = 1; r < R; ++r) {
        double2 w = tw[r * k * (L / (NS * R))];
        if (INV) w.y = -w.y;
        v[h][r] = cmul(v[h][r], w);
      }
    }
    dft_reg<R, INV>(v[h]);
  }
  __syncthreads();
#pragma unroll
  for (int h = 0; h < NH; ++h) {
    const int j = j0 + h * (T / 8), k = j % NS, base = (j / NS) * NS * R + k;
#pragma unroll
    for (int r = 0; r < R; ++r) s[tidx(base + r * NS, c)] = v[h][r];
  }
  __syncthreads();
}

// One tile (fft.cuh fft_gconv with the hooks of the pipelined tile loop).  Not inlined: nothing of
// a tile's index arithmetic is hoisted out of the persistent loop and kept live across the middle
// stage.
__device__ __noinline__ double tile_pass(Args a, int tile, int next) {
  extern __shared__ double2 smem[];
  double2* tiles[NC];
#pragma unroll
  for (int q = 0; q < NC; ++q) tiles[q] = smem + q * 8 * L;
  const double2* tw = smem + NC * 8 * L;
  const int t = threadIdx.x, c = t & 7, j0 = t >> 3;
  const long long boff = tile_off(a, tile);
  const double w = parseval_w(tile / a.ntile_y, a.M);
#pragma unroll
  for (int q = 0; q < NC; ++q) {
    // component q's copy group has landed (groups are committed in component order)
    if (q == 0) cp_wait<2>();
    else if (q == 1) cp_wait<1>();
    else cp_wait<0>();
    __syncthreads();
    stage<1, false>(tiles[q], tw);
    stage<R, false>(tiles[q], tw);
  }
  // middle: last forward stage (span NJ) -> s_hat = G_hat r_hat on the bins j + r NJ -> first
  // inverse stage (span 1), on registers
  double part = 0.0;
  double2 v[NH][NC][R];
#pragma unroll
  for (int h = 0; h < NH; ++h) {
    const int j = j0 + h * (T / 8);
#pragma unroll
    for (int q = 0; q < NC; ++q) {
#pragma unroll
      for (int r = 0; r < R; ++r) v[h][q][r] = tiles[q][tidx(j + r * NJ, c)];
#pragma unroll
      for (int r = 1; r < R; ++r) v[h][q][r] = cmul(v[h][q][r], tw[r * j]);
      Dft<R>::run(v[h][q]);
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      double2 x[NC];
#pragma unroll
      for (int q = 0; q < NC; ++q) x[q] = v[h][q][r];
      part += gmul_vals<NC>(x, a.gtab, a.nspec, boff + (long long)(j + r * NJ) * a.N2 + c, w);
#pragma unroll
      for (int q = 0; q < NC; ++q) v[h][q][r] = x[q];
    }
#pragma unroll
    for (int q = 0; q < NC; ++q) dft_reg_inv_inline<R>(v[h][q]);
  }
  __syncthreads();
#pragma unroll
  for (int h = 0; h < NH; ++h) {
    const int j = j0 + h * (T / 8);
#pragma unroll
    for (int q = 0; q < NC; ++q)
#pragma unroll
      for (int r = 0; r < R; ++r) tiles[q][tidx(j * R + r, c)] = v[h][q][r];
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < NC; ++q) {
    stage<R, true>(tiles[q], tw);
    stage<R * R, true>(tiles[q], tw);
    double2* base = a.spec + q * a.nspec + boff;
#pragma unroll
    for (int i = 0; i < 8 * L / T; ++i) {
      const int e = t + i * T;
      base[(long long)(e >> 3) * a.N2 + (e & 7)] = tiles[q][tidx(e >> 3, e & 7)];
    }
    __syncthreads();  // every thread has read its part of tiles[q]: the buffer is free
    if (next >= 0) issue(a, tiles[q], q, tile_off(a, next));
    else cp_commit();
  }
  return part;
}
}  // namespace g5e

template <int MODE>
__global__ void __launch_bounds__(g5e::T, 1) gpass512e_kernel(Ctx cx) {
  using namespace g5e;
  const Geo& g = cx.g;
  const int load = blockIdx.y;
  if (MODE == CG && !cx.st[load].active) return;
  extern __shared__ double2 smem[];
  double2* tw = smem + NC * 8 * L;
  __shared__ double red_sh[32];
  for (int i = threadIdx.x; i < L; i += T) tw[i] = cx.tw.z[i];
  Args a;
  a.spec = cx.spec + (long long)load * g.c * g.nspec;
  a.gtab = cx.gtab;
  a.nspec = g.nspec;
  a.N2 = g.N2;
  a.N3 = g.N3;
  a.M = g.M;
  a.ntile_y = g.N2 >> 3;
  const int ntiles = g.H1 * a.ntile_y;
  int tile = blockIdx.x;
  if (tile < ntiles) {
    const long long b0 = tile_off(a, tile);
#pragma unroll
    for (int q = 0; q < NC; ++q) issue(a, smem + q * 8 * L, q, b0);
  }
  for (; tile < ntiles; tile += gridDim.x) {
    const int next = tile + gridDim.x;
    const double part = tile_pass(a, tile, next < ntiles ? next : -1);
    partial_write<false>(cx, RED_GAMMA, load, tile, part, red_sh);
  }
}

bool gpass512e_supported(const Geo& g) {
  return UNO_G512E_PERSIST && g.dim == 3 && !g.dirz && !g.zpad && g.c == 3 && g.N3 == 512 && g.N2 % 8 == 0;
}

int launch_gpass512e(const Ctx& cx, int mode, cudaStream_t s) {
  const Geo& g = cx.g;
  const int ntiles = g.H1 * (g.N2 / 8);
  const dim3 grid((unsigned)(ntiles < kG512ePersistCTAs ? ntiles : kG512ePersistCTAs), g.nrhs);
  constexpr int sm = (3 * 8 * 512 + 512) * (int)sizeof(double2);
  auto go = [&](auto k) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);  // per device: set on every launch
    k<<<grid, g5e::T, sm, s>>>(cx);
    return 1;
  };
  return mode == CG ? go(gpass512e_kernel<CG>) : go(gpass512e_kernel<STANDALONE>);
}

}  // namespace uno
