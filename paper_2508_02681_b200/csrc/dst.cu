// dst.cu — DST-I along z for the mixed boundary condition (periodic x, y; Dirichlet z).
//
// PAPER.md Table 1 row "Mixed" uses F^x o T_ST^y in 2D; for 3D with Dirichlet faces on
// z (BASELINE config 4 variant) the unitary transform is U = F_x (x) F_y (x) DST-I_z (SURVEY
// A13; DST variant SPEC S:249).  The z transform is the middle stage of the 5-pass schedule, on
// the complex half spectrum after the x R2C and y FFTs (the transforms commute), so the CG
// fusions of the periodic x passes (r -= alpha p, ||r||_inf; d = s + beta d, u += alpha d_old)
// carry over unchanged.  DST-I of length N-1 (N = N3) through a complex FFT of length 2N of the
// odd extension  y_0 = 0, y_j = x_j (1 <= j < N), y_N = 0, y_{2N-j} = -x_j:
//   sum_j x_j sin(pi j m / N) = (i/2) Y_m  (for complex x as well: S(a) + i S(b)).
// Unnormalised (the sine sum); N/2 of the round trip is folded into the tabulated symbol.
#include <cuda_runtime.h>

#include <type_traits>

#include "common.cuh"
#include "dev_common.cuh"
#include "fft.cuh"
#include "kernels.cuh"

namespace uno {

#ifndef UNO_DST_W4
#define UNO_DST_W4 1  // 4-column tiles for the 1024-point z DST (0: 8 columns, one CTA per SM; A/B only)
#endif
template <int L2>
__host__ __device__ constexpr int dst_smem_bytes() {
  return (8 * L2 + L2) * (int)sizeof(double2);
}

// ---------------------------------------------------------------------- z transform on the spectrum
// The z DST-I runs on the complex half spectrum [lc][kx][z][y] after the x R2C and y FFTs (the
// transforms commute, U is the same), as the middle stage of the 5-pass schedule:
//   x (+ r -= alpha p, ||r||) | y | DST_z . G . DST_z | y^-1 | x^-1 (+ d, u updates) | K.
// Two storages: the whole grid keeps the N3-1 interior node planes (node j at index j - 1, sine
// mode m at index m - 1, PAD = false); slab pencils keep N3 planes with plane 0 the fixed face
// (node / mode j at index j, index 0 = 0, PAD = true).  DST-I of a complex column through the
// length-2N3 odd extension: (i/2) Y_m = S(a) + i S(b).  The y extent is the grid's N2 (whole grid)
// or the rank's k_y chunk (pencil); 8 consecutive y columns per CTA.
// W: columns per CTA (8; 4 for the 1024-point transform of N3 = 512: two CTAs share an SM, so one's
// loads / stores overlap the other's FFT stages — 9.70 -> 8.24 ms for the DST . G . DST stage of the
// 512^3 elastic mixed grid, despite 168 bytes of spills at the 64-register cap).
#ifndef UNO_DST_T256
#define UNO_DST_T256 1  // 1024-point transform on 256 threads (1-2 butterflies each, no spills); 0: 512 threads (A/B)
#endif
template <int L2, int W>
__host__ __device__ constexpr int dst_threads() {
  return (L2 == 1024 && W == 4 && UNO_DST_T256) ? 256 : fft_threads_w(L2, W);
}
template <int L2, bool PAD, int MODE, int W = 8>
__global__ void __launch_bounds__(dst_threads<L2, W>(), (W == 4 || L2 <= 512) ? 2 : 1) spec_dst_kernel(Ctx cx, double2* __restrict__ P) {
  constexpr int T = dst_threads<L2, W>();
  constexpr int TT = T == fft_threads_w(L2, W) ? 0 : T;  // threads < butterflies: several per thread
  constexpr int N = L2 / 2;           // = N3
  constexpr int NP = PAD ? N : N - 1;  // stored planes
  constexpr int OFF = PAD ? 0 : 1;     // node / mode j lives at index j - OFF
  constexpr int B = W == 4 ? 4 : 1;    // loads in flight per thread (W = 4: one CTA per SM would
                                       // otherwise idle on them; at W = 8 batching measured slower)
  const Geo g = cx.g;
  const int load = blockIdx.y;
  if (MODE == CG && !cx.st[load].active) return;
  extern __shared__ double2 smem[];
  double2* tile = smem;
  double2* tw = smem + W * L2;
  const int t = threadIdx.x;
  const int Yc = g.N2, nyc = Yc / W;
  const int yq = blockIdx.x % nyc;
  const long long lk = blockIdx.x / nyc;  // (component, kx) row of this load
  const long long col0 = ((long long)load * g.c * g.H1 + lk) * NP * Yc + yq * W;
  for (int i = t; i < L2; i += T) tw[i] = cx.tw.z2[i];
  for (int e0 = t; e0 < W * (N - 1); e0 += B * T) {
    double2 v[B];
#pragma unroll
    for (int u = 0; u < B; ++u) {
      const int e = e0 + u * T;
      if (e < W * (N - 1)) {
        const double2* src = &P[col0 + (long long)(e / W + 1 - OFF) * Yc + (e & (W - 1))];
        v[u] = W == 4 ? __ldcg(src) : *src;
      }
    }
#pragma unroll
    for (int u = 0; u < B; ++u) {
      const int e = e0 + u * T;
      if (e < W * (N - 1)) {
        const int pz = e / W + 1, c = e & (W - 1);
        tile[tidx_w<W>(pz, c)] = v[u];
        tile[tidx_w<W>(L2 - pz, c)] = make_double2(-v[u].x, -v[u].y);
      }
    }
  }
  if (t < W) {
    tile[tidx_w<W>(0, t)] = make_double2(0.0, 0.0);
    tile[tidx_w<W>(N, t)] = make_double2(0.0, 0.0);
  }
  __syncthreads();
  fft_tile_w<L2, false, W, TT>(tile, tw);
  for (int e = t; e < W * NP; e += T) {
    const int i = e / W, c = e & (W - 1), m = i + OFF;
    const double2 Y = tile[tidx_w<W>(m, c)];
    const double2 o = m == 0 ? make_double2(0.0, 0.0) : make_double2(-0.5 * Y.y, 0.5 * Y.x);
    if (W == 4) __stcg(&P[col0 + (long long)i * Yc + c], o);
    else P[col0 + (long long)i * Yc + c] = o;
  }
}

// s_hat = G_hat r_hat on every bin of the spectrum (all c components of a bin together) and the
// Parseval partial of gamma (weights of the R2C kx planes), grid-stride over the bins.
constexpr int PG_NBLK = 148 * 4;
template <int NC, int MODE>
__global__ void __launch_bounds__(256) spec_gmul_kernel(Ctx cx, double2* __restrict__ P) {
  const Geo g = cx.g;
  const int load = blockIdx.y;
  if (MODE == CG && !cx.st[load].active) return;
  __shared__ double red_sh[32];
  const long long ns = g.nspec, zy = (long long)g.P3 * g.N2;
  double2* base = P + (long long)load * g.c * ns;
  double part = 0.0;
  for (long long b = (long long)blockIdx.x * blockDim.x + threadIdx.x; b < ns; b += (long long)gridDim.x * blockDim.x) {
    double2 x[NC];
#pragma unroll
    for (int q = 0; q < NC; ++q) x[q] = base[q * ns + b];
    part += gmul_vals<NC>(x, cx.gtab, ns, b, parseval_w((int)(b / zy), g.M));
#pragma unroll
    for (int q = 0; q < NC; ++q) base[q * ns + b] = x[q];
  }
  partial_write<false>(cx, RED_GAMMA, load, blockIdx.x, part, red_sh);
}

int pencil_gmul_nblk() { return PG_NBLK; }

template <class F>
static int dispatch_l2(int L, F&& f);

// DST_z . G . DST_z on the spectrum in place (Dirichlet z: whole-grid mixed BC or a slab pencil).
int launch_pencil_dst_green(const Ctx& cx, double2* spec, int mode, cudaStream_t s) {
  const Geo& g = cx.g;
  if (!(g.zpad || (g.dirz && g.dim == 3)) || g.N2 % 8 || (g.c != 1 && g.c != 3)) return -1;
  const bool pad = g.zpad != 0;
  const bool cg = mode == CG;
  return dispatch_l2(2 * g.N3, [&](auto Lc) {
    constexpr int L2 = decltype(Lc)::value;
    constexpr int W = (L2 >= 1024 && UNO_DST_W4) ? 4 : 8;
    const dim3 grid((unsigned)((long long)g.c * g.H1 * (g.N2 / W)), g.nrhs);
    constexpr int sm = (W * L2 + L2) * (int)sizeof(double2);
    auto dst = [&](auto k) {
      if (sm > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
      k<<<grid, dst_threads<L2, W>(), sm, s>>>(cx, spec);
    };
    auto run_dst = [&] {
      if (pad) cg ? dst(spec_dst_kernel<L2, true, CG, W>) : dst(spec_dst_kernel<L2, true, STANDALONE, W>);
      else cg ? dst(spec_dst_kernel<L2, false, CG, W>) : dst(spec_dst_kernel<L2, false, STANDALONE, W>);
    };
    run_dst();
    const dim3 gg(PG_NBLK, g.nrhs);
    if (g.c == 1) cg ? spec_gmul_kernel<1, CG><<<gg, 256, 0, s>>>(cx, spec) : spec_gmul_kernel<1, STANDALONE><<<gg, 256, 0, s>>>(cx, spec);
    else cg ? spec_gmul_kernel<3, CG><<<gg, 256, 0, s>>>(cx, spec) : spec_gmul_kernel<3, STANDALONE><<<gg, 256, 0, s>>>(cx, spec);
    run_dst();
    return 3;
  });
}

template <class F>
static int dispatch_l2(int L, F&& f) {
  switch (L) {
    case 16: return f(std::integral_constant<int, 16>{});
    case 32: return f(std::integral_constant<int, 32>{});
    case 64: return f(std::integral_constant<int, 64>{});
    case 128: return f(std::integral_constant<int, 128>{});
    case 256: return f(std::integral_constant<int, 256>{});
    case 512: return f(std::integral_constant<int, 512>{});
    case 1024: return f(std::integral_constant<int, 1024>{});
    default: return -1;
  }
}

}  // namespace uno
