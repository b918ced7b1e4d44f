// tiny.cu — the whole of PAPER.md Alg 2 in ONE CTA per load case for small 2D periodic
// thermal grids (config 0: 32 x 32; SURVEY §2.5 `tiny_pcg`).  At this size the graph-driven path
// is launch-latency bound (~9 dependent launches per iteration, ~25 us per iteration) while the
// whole CG state (r, d, u, p and the spectrum: ~60 KB at 32^2) fits in shared memory.  One
// persistent CTA iterates with block-wide barriers instead of kernel boundaries:
//   ||r||_inf (l.3, relative stop) -> s = T^H Q T r (l.4-6; 2D complex Stockham radix-2 FFT in
//   shared memory, the tabulated G_hat/n of the handle, Parseval gamma over all bins) -> beta,
//   d = s + beta d (l.7-8) -> p = A d (l.9; the Q1 element row of App. A1 as in the 2D K kernel)
//   -> alpha = gamma / d.p, r -= alpha p, u += alpha d (l.10-12),
// with the same device scalar logic (dev_common.cuh) as the multi-kernel loop, so reports,
// residual history and the recorded (gamma, alpha) are produced identically.
#include <cuda_runtime.h>

#include "common.cuh"
#include "dev_common.cuh"
#include "kernels.cuh"

namespace uno {

constexpr int TINY_T = 1024;

__device__ __forceinline__ double tiny_reduce_sum(double v, double* sh) {
  const double b = block_reduce<false>(v, sh);
  __shared__ double bc;
  if (threadIdx.x == 0) bc = b;
  __syncthreads();
  const double r = bc;
  __syncthreads();
  return r;
}
__device__ __forceinline__ double tiny_reduce_max(double v, double* sh) {
  const double b = block_reduce<true>(v, sh);
  __shared__ double bc;
  if (threadIdx.x == 0) bc = b;
  __syncthreads();
  const double r = bc;
  __syncthreads();
  return r;
}

// One radix-2 Stockham pass over every line of a 2D complex array: lines of length L along
// `stride` (1: rows of length N1; N1: columns of length N2), `nlines` of them at distance `lstep`.
// Ns = size of the sub-transforms already done.  tw[t] = exp(-2 pi i t / L) (conjugated for INV).
template <bool INV>
__device__ __forceinline__ void stockham_pass(const double2* __restrict__ in, double2* __restrict__ out,
                                              const double2* __restrict__ tw, int L, int stride, int nlines,
                                              int lstep, int Ns) {
  const int half = L / 2, nb = nlines * half;
  for (int e = threadIdx.x; e < nb; e += blockDim.x) {
    const int line = e / half, j = e - line * half;
    const int k = j & (Ns - 1);
    const long long base = (long long)line * lstep;
    double2 v0 = in[base + (long long)j * stride], v1 = in[base + (long long)(j + half) * stride];
    double2 w = tw[k * (L / (2 * Ns))];
    if (INV) w.y = -w.y;
    v1 = cmul(v1, w);
    const int od = (j / Ns) * 2 * Ns + k;
    out[base + (long long)od * stride] = cadd(v0, v1);
    out[base + (long long)(od + Ns) * stride] = csub(v0, v1);
  }
  __syncthreads();
}

// 2D transform of A (result returned: A or B, whichever holds it)
template <bool INV>
__device__ double2* tiny_fft2(double2* A, double2* B, const double2* twx, const double2* twy, int N1, int N2) {
  double2 *in = A, *out = B;
  for (int Ns = 1; Ns < N1; Ns *= 2) {  // rows (x)
    stockham_pass<INV>(in, out, twx, N1, 1, N2, N1, Ns);
    double2* t = in;
    in = out;
    out = t;
  }
  for (int Ns = 1; Ns < N2; Ns *= 2) {  // columns (y)
    stockham_pass<INV>(in, out, twy, N2, N1, N1, 1, Ns);
    double2* t = in;
    in = out;
    out = t;
  }
  return in;
}

__global__ void __launch_bounds__(TINY_T) tiny_pcg2d_kernel(Ctx cx) {
  const Geo g = cx.g;
  const int load = blockIdx.x;
  const int N1 = g.N1, N2 = g.N2, n = N1 * N2, M = N1 / 2;
  LoadState* st = cx.st + load;
  extern __shared__ double tsm[];
  double* r = tsm;
  double* d = r + n;
  double* u = d + n;
  double2* A = reinterpret_cast<double2*>(u + n);
  double2* B = A + n;
  double2* twx = B + n;
  double2* twy = twx + N1;
  unsigned char* ph = reinterpret_cast<unsigned char*>(twy + N2);
  __shared__ double red_sh[32];
  const int t = threadIdx.x, T = blockDim.x;
  const double k0 = cx.mat[0][0], k1 = cx.mat[1][0];
  // inputs: r = f (the RHS the host launch wrote into cx.r), u = 0, d = 0; twiddles exp(-2 pi i t / N)
  const double* f = cx.r + (long long)load * n;
  for (int i = t; i < n; i += T) {
    r[i] = f[i];
    u[i] = 0.0;
    d[i] = 0.0;
    ph[i] = cx.phase[i];
  }
  for (int i = t; i < N1; i += T) {
    double s, c;
    sincospi(-2.0 * i / N1, &s, &c);
    twx[i] = make_double2(c, s);
  }
  for (int i = t; i < N2; i += T) {
    double s, c;
    sincospi(-2.0 * i / N2, &s, &c);
    twy[i] = make_double2(c, s);
  }
  __syncthreads();
  const double* gt = cx.gtab;
  for (;;) {
    // ---- l.3: ||r||_inf and the stopping decision (scalar logic of the multi-kernel loop)
    double mx = 0.0;
    for (int i = t; i < n; i += T) mx = fmax(mx, fabs(r[i]));
    mx = tiny_reduce_max(mx, red_sh);
    if (t == 0) scalar_after_rnorm(st, mx, cx.hist, cx.hist_stride, load);
    __syncthreads();
    if (!st->active) break;
    // ---- l.4-6: s = T^H Q T r with the full complex 2D FFT; gamma_1 = r.s by Parseval
    for (int i = t; i < n; i += T) A[i] = make_double2(r[i], 0.0);
    __syncthreads();
    double2* R = tiny_fft2<false>(A, B, twx, twy, N1, N2);
    double gp = 0.0;
    for (int i = t; i < n; i += T) {
      const int kx = i % N1, ky = i / N1;
      // half-spectrum table [kx][ky] (kx <= N1/2); G(-k) = G(k) for the other half
      const int hx = kx <= M ? kx : N1 - kx, hy = kx <= M ? ky : (N2 - ky) & (N2 - 1);
      const double gv = gt[(long long)hx * N2 + hy];
      const double2 v = R[i];
      gp = fma(gv, fma(v.x, v.x, v.y * v.y), gp);
      R[i] = make_double2(gv * v.x, gv * v.y);
    }
    gp = tiny_reduce_sum(gp, red_sh);
    double2* S = tiny_fft2<true>(R, R == A ? B : A, twx, twy, N1, N2);
    if (t == 0) scalar_after_gamma(st, gp, cx.hist, cx.hist_stride, load);
    __syncthreads();
    if (!st->active) break;
    // ---- l.8: d = s + beta d
    const double beta = st->beta;
    for (int i = t; i < n; i += T) d[i] = fma(beta, d[i], S[i].x);
    __syncthreads();
    // ---- l.9-10: p = A d (into the free complex buffer) and d.p
    double* p = reinterpret_cast<double*>(S == A ? B : A);
    double dp = 0.0;
    for (int i = t; i < n; i += T) {
      const int x = i % N1, y = i / N1;
      const int xm = (x - 1 + N1) & (N1 - 1), xp = (x + 1) & (N1 - 1), ym = (y - 1 + N2) & (N2 - 1), yp = (y + 1) & (N2 - 1);
      auto D = [&](int xx, int yy) { return d[yy * N1 + xx]; };
      auto KAP = [&](int xx, int yy) { return ph[yy * N1 + xx] ? k1 : k0; };
      const double a00 = KAP(xm, ym), a01 = KAP(x, ym), a10 = KAP(xm, y), a11 = KAP(x, y);  // [oy][ox]
      const double dmm = D(xm, ym), d0m = D(x, ym), dpm = D(xp, ym);
      const double dm0 = D(xm, y), d00 = D(x, y), dp0 = D(xp, y);
      const double dmp = D(xm, yp), d0p = D(x, yp), dpp = D(xp, yp);
      const double S00 = (dmm + d0m) + (dm0 + d00), S01 = (d0m + dpm) + (d00 + dp0);
      const double S10 = (dm0 + d00) + (dmp + d0p), S11 = (d00 + dp0) + (d0p + dpp);
      const double Ksum = (a00 + a01) + (a10 + a11);
      const double KS = fma(a00, S00, fma(a01, S01, fma(a10, S10, a11 * S11)));
      double EE = (a01 + a11) * dp0;
      EE = fma(a00 + a10, dm0, EE);
      EE = fma(a10 + a11, d0p, EE);
      EE = fma(a00 + a01, d0m, EE);
      const double pv = (fma(6.0 * d00, Ksum, EE) - 2.0 * KS) * (1.0 / 6.0);
      p[i] = pv;
      dp = fma(d00, pv, dp);
    }
    dp = tiny_reduce_sum(dp, red_sh);
    if (t == 0) scalar_after_dp(st, dp, cx.hist, cx.hist_stride, load);
    __syncthreads();
    if (st->status != 0) break;
    // ---- l.11-12: r -= alpha p ; u += alpha d
    const double alpha = st->alpha;
    for (int i = t; i < n; i += T) {
      r[i] = fma(-alpha, p[i], r[i]);
      u[i] = fma(alpha, d[i], u[i]);
    }
    __syncthreads();
  }
  if (t == 0) st->pending_u = 0;  // u is complete (no deferred update)
  double* uo = cx.u + (long long)load * n;
  for (int i = t; i < n; i += T) uo[i] = u[i];
}

// ---------------------------------------------------------------------------- 32 x 32 fast path
// Config 0's grid: one thread per node (x = lane, y = warp), so r, d, u, p, the node's four element
// conductivities and its bin's symbol entry live in registers for the whole solve.  The 2D FFT is
// two warp-shuffle radix-2 passes (rows over the lanes; columns over the lanes after one padded
// shared-memory transpose): forward decimation in frequency leaves the bins in bit-reversed order,
// the symbol is applied there, and the inverse decimation-in-time pass (conjugate twiddles) takes
// them back to natural order (Eq 47-48; unnormalised, the 1/n is in the table as
// elsewhere).  Reductions are all-reduces (every warp combines the 32 warp partials in the same
// order), and every thread runs the scalar logic on its own copy of the load state, so an
// iteration has 7 barriers and no global-memory round trip.
constexpr int T32 = 1024, S32 = 33;  // transpose row stride (double2): conflict-free quarter warps

__device__ __forceinline__ double2 shfl_xor2(double2 v, int m) {
  return make_double2(__shfl_xor_sync(0xffffffffu, v.x, m), __shfl_xor_sync(0xffffffffu, v.y, m));
}
// forward DFT over the 32 lanes, decimation in frequency: lane x ends with X[brev5(x)]
__device__ __forceinline__ double2 warp_dif32(double2 v, const double2* tw, int lane) {
#pragma unroll
  for (int b = 16; b >= 1; b >>= 1) {
    const double2 pv = shfl_xor2(v, b);
    if (lane & b) v = cmul(csub(pv, v), tw[(lane & (b - 1)) * (16 / b)]);  // (a_j - a_{j+b}) W_{2b}^j
    else v = cadd(v, pv);
  }
  return v;
}
// inverse DFT (kernel e^{+2 pi i jk/32}) over the lanes from bit-reversed input, decimation in time
__device__ __forceinline__ double2 warp_dit32_inv(double2 v, const double2* tw, int lane) {
#pragma unroll
  for (int b = 1; b <= 16; b <<= 1) {
    const double2 pv = shfl_xor2(v, b);                    // every lane shuffles (full mask)
    const double2 tv = (lane & b) ? v : pv;                // the odd member of the pair
    const double2 ev = (lane & b) ? pv : v;                // the even member
    const double2 wt = cmul(tv, cconj(tw[(lane & (b - 1)) * (16 / b)]));
    v = (lane & b) ? csub(ev, wt) : cadd(ev, wt);
  }
  return v;
}
template <bool MAX>
__device__ __forceinline__ double allreduce32(double v, double* sh) {  // sh: 32 doubles, this reduction only
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    const double w = __shfl_xor_sync(0xffffffffu, v, o);
    v = MAX ? fmax(v, w) : v + w;
  }
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  double a = sh[0];
#pragma unroll
  for (int w = 1; w < 32; ++w) a = MAX ? fmax(a, sh[w]) : a + sh[w];
  return a;  // identical in every thread (same values, same order)
}

__global__ void __launch_bounds__(T32) tiny_pcg32_kernel(Ctx cx) {
  constexpr int N = 32, M = 16;
  const int load = blockIdx.x;
  const int t = threadIdx.x, x = t & 31, y = t >> 5;
  __shared__ double2 S[N * S32];
  __shared__ double Dsm[N * N];
  __shared__ double2 tw[16];
  __shared__ double red[3][32];
  LoadState st = cx.st[load];
  double* hist = t == 0 ? cx.hist : nullptr;
  if (t < 16) {
    double sn, cs;
    sincospi(-2.0 * t / N, &sn, &cs);
    tw[t] = make_double2(cs, sn);
  }
  // node state and constants
  double r = cx.r[(long long)load * N * N + t], d = 0.0, u = 0.0;
  const double k0 = cx.mat[0][0], k1 = cx.mat[1][0];
  const int xm = (x - 1) & 31, xp = (x + 1) & 31, ym = (y - 1) & 31, yp = (y + 1) & 31;
  auto KAP = [&](int xx, int yy) { return cx.phase[yy * N + xx] ? k1 : k0; };
  const double a00 = KAP(xm, ym), a01 = KAP(x, ym), a10 = KAP(xm, y), a11 = KAP(x, y);  // [oy][ox]
  const double Ksum = (a00 + a01) + (a10 + a11);
  // this thread's bin after the forward passes: column slot c = y of the warp doing the column
  // pass is the row frequency brev(c); the lane is the column frequency brev(lane)
  const int kx = __brev(y) >> 27, ky = __brev(x) >> 27;
  const int hx = kx <= M ? kx : N - kx, hy = kx <= M ? ky : (N - ky) & (N - 1);
  const double gv = cx.gtab[(long long)hx * N + hy];
  __syncthreads();
  for (;;) {
    // ---- l.3: ||r||_inf and the stopping decision
    const double rn = allreduce32<true>(fabs(r), red[0]);
    scalar_after_rnorm(&st, rn, hist, cx.hist_stride, load);
    if (!st.active) break;
    // ---- l.4-6: s = T^H Q T r; gamma_1 = r.s by Parseval (all n bins, weight 1)
    double2 v = warp_dif32(make_double2(r, 0.0), tw, x);  // row y, slot x
    S[y * S32 + x] = v;
    __syncthreads();
    v = warp_dif32(S[x * S32 + y], tw, x);                 // column slot y, row bin brev(x)
    double gp = gv * fma(v.x, v.x, v.y * v.y);
    v = make_double2(gv * v.x, gv * v.y);
    v = warp_dit32_inv(v, tw, x);                          // column slot y, row x
    __syncthreads();                                       // every transposed read done
    S[x * S32 + y] = v;
    __syncthreads();
    v = warp_dit32_inv(S[y * S32 + x], tw, x);             // row y, node x
    gp = allreduce32<false>(gp, red[1]);
    scalar_after_gamma(&st, gp, hist, cx.hist_stride, load);
    if (!st.active) break;
    // ---- l.8: d = s + beta d ; l.9-10: p = A d (Q1 row of App. A1), d.p
    d = fma(st.beta, d, v.x);
    Dsm[t] = d;
    __syncthreads();
    const double dmm = Dsm[ym * N + xm], d0m = Dsm[ym * N + x], dpm = Dsm[ym * N + xp];
    const double dm0 = Dsm[y * N + xm], dp0 = Dsm[y * N + xp];
    const double dmp = Dsm[yp * N + xm], d0p = Dsm[yp * N + x], dpp = Dsm[yp * N + xp];
    const double S00 = (dmm + d0m) + (dm0 + d), S01 = (d0m + dpm) + (d + dp0);
    const double S10 = (dm0 + d) + (dmp + d0p), S11 = (d + dp0) + (d0p + dpp);
    const double KS = fma(a00, S00, fma(a01, S01, fma(a10, S10, a11 * S11)));
    double EE = (a01 + a11) * dp0;
    EE = fma(a00 + a10, dm0, EE);
    EE = fma(a10 + a11, d0p, EE);
    EE = fma(a00 + a01, d0m, EE);
    const double p = (fma(6.0 * d, Ksum, EE) - 2.0 * KS) * (1.0 / 6.0);
    const double dp = allreduce32<false>(d * p, red[2]);
    scalar_after_dp(&st, dp, hist, cx.hist_stride, load);
    if (st.status != 0) break;
    // ---- l.11-12: r -= alpha p ; u += alpha d
    r = fma(-st.alpha, p, r);
    u = fma(st.alpha, d, u);
  }
  st.pending_u = 0;  // u is complete (no deferred update)
  cx.u[(long long)load * N * N + t] = u;
  if (t == 0) cx.st[load] = st;
}

int tiny_smem_bytes(const Geo& g) {
  const int n = g.N1 * g.N2;
  return 3 * n * 8 + 2 * n * 16 + (g.N1 + g.N2) * 16 + n;
}

// Alg 2 for every load, one CTA each; the handle's RHS must already be in cx.r.  -1: not a tiny grid.
int launch_tiny_pcg(const Ctx& cx, cudaStream_t s) {
  const Geo& g = cx.g;
  if (!tiny_supported(g)) return -1;
  if (g.N1 == 32 && g.N2 == 32) {  // config 0: the register-resident fast path
    tiny_pcg32_kernel<<<g.nrhs, T32, 0, s>>>(cx);
    return 1;
  }
  const int sm = tiny_smem_bytes(g);
  cudaFuncSetAttribute(tiny_pcg2d_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  tiny_pcg2d_kernel<<<g.nrhs, TINY_T, sm, s>>>(cx);
  return 1;
}

bool tiny_supported(const Geo& g) {
  return g.dim == 2 && g.c == 1 && !g.dmask && g.N1 * g.N2 <= 2048;
}

}  // namespace uno
