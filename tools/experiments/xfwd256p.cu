// MEASURED AND REJECTED (round 2): 296.9 us vs 267.9 us for the register-direct xfwd256_kernel at 256^3 x 3
// loads (parity green).  The 64 KB input ring leaves room for two 128-thread CTAs per SM; 8 warps cannot
// cover the FP64 latency of the FFT stages, while the register-direct kernel keeps 20 warps and ~160 KB of
// loads in flight per SM in registers.  Not part of libunocg.so; kept for the record (it compiled as
// paper_2508_02681_b200/csrc/xfwd256p.cu with launch_xfwd dispatching to launch_xfwd256p for N1 = 256).
// xfwd256p.cu — F1 for N1 = 256 (config 3, the headline) as a persistent kernel with a bulk-copy
// input ring: r -= alpha p (Alg 2 l.11), ||r||_inf partial (l.3), x-axis R2C FFT (l.4, Eq 47) of 8
// rows per unit, straight to the half spectrum [load][kx][z][y].
//
// Same arithmetic as xfwd256_kernel (kernels.cu: complex FFT of length 128 of z_j = r_2j + i r_2j+1
// as DFT8 over n2 -> twiddle -> padded transpose -> DFT16 over n1 split between two threads -> R2C
// post-processing), same 8-row blocks and ||r||_inf partial per block.  What changes is how the
// rows arrive: the 8 rows of a block are 16 KB contiguous in r (and in p), so one elected thread
// fetches them with cp.async.bulk into a two-stage shared-memory ring, two blocks ahead of the
// compute, completing on an mbarrier per stage — the register-direct kernel waits on its own
// global loads at 20 warps per SM (ncu: 41 % long scoreboard) and reloads 4 KB of twiddle tables
// per 8-row CTA; here the tables are loaded once per CTA and memory latency is covered by the ring.
#include <cuda_runtime.h>

#include "common.cuh"
#include "fft.cuh"
#include "kernels.cuh"
#include "dev_common.cuh"

namespace uno {

#ifndef UNO_XFWD256P
#define UNO_XFWD256P 1  // 0: the register-direct xfwd256_kernel (A/B builds)
#endif

namespace x2p {
constexpr int M = 128, T = 128, NSTG = 2;
constexpr int RS = 8 * 17;   // transpose buffer per row (8 x 16, padded)
constexpr int XS = 129;      // X row stride (odd in 16-byte units)
constexpr unsigned kRowsBytes = 8 * 256 * 8;  // 8 rows of N1 = 256 doubles
constexpr int kCtasPerSm = 2, kCtas = 148 * kCtasPerSm;
__device__ __forceinline__ int swz(int k) { return k ^ (((k >> 3) & 1) << 2); }

__device__ __forceinline__ unsigned sm_addr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned mb, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(mb), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned mb, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mb), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned mb, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "X2P_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@p bra X2P_DONE;\n"
      "bra X2P_WAIT;\n"
      "X2P_DONE:\n"
      "}\n" ::"r"(mb),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_load(unsigned dst, const void* src, unsigned bytes, unsigned mb) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(mb)
               : "memory");
}
}  // namespace x2p

template <int MODE>
__global__ void __launch_bounds__(x2p::T, x2p::kCtasPerSm) xfwd256p_kernel(Ctx cx, const double* __restrict__ src) {
  using namespace x2p;
  const Geo& g = cx.g;
  extern __shared__ __align__(128) double2 xsm[];
  double2* rin = xsm;                         // [NSTG][8 rows][128]
  double2* pin = rin + NSTG * 8 * M;          // [NSTG][8 rows][128]
  double2* tb = pin + NSTG * 8 * M;           // [8][RS]
  double2* xs = tb + 8 * RS;                  // [8][XS]
  double2* tw = xs + 8 * XS;                  // [M]
  double2* twp = tw + M;                      // [M + 1]
  double2* tw16 = twp + M + 1;                // [8]
  __shared__ double red_sh[32];
  __shared__ __align__(8) unsigned long long mbar[NSTG];
  __shared__ int act[kMaxRhs];
  __shared__ int nact_s;
  const int t = threadIdx.x;
  const int r = t >> 4, l16 = t & 15;
  if (t == 0) {
    int n = 0;
    for (int l = 0; l < g.nrhs; ++l)
      if (MODE == STANDALONE || cx.st[l].active) act[n++] = l;
    nact_s = n;
#pragma unroll
    for (int b = 0; b < NSTG; ++b) mbar_init(sm_addr(mbar) + 8 * b, 1);
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  }
  for (int i = t; i < M; i += T) tw[i] = cx.tw.x[((i & 15) * (i >> 4)) & (M - 1)];  // [k1][n1]
  for (int i = t; i <= M; i += T) twp[i] = cx.tw.xpost[i];
  if (t < 8) tw16[t] = cx.tw.x[8 * t];
  __syncthreads();
  const int nact = nact_s;
  if (nact == 0) return;
  const long long nblk = (long long)g.c * g.P3 * g.N2 / 8;  // 8-row blocks per load
  const long long total = nblk * nact;
  const long long first = blockIdx.x;
  const long long nunits = first < total ? (total - 1 - first) / gridDim.x + 1 : 0;
  // unit k of this CTA -> (load, block); loads fastest would interleave the CG scalars, so block fastest
  auto unit_of = [&](long long k, int& load, long long& bx) {
    const long long id = first + k * gridDim.x;
    const long long li = id / nblk;
    load = act[(int)li];
    bx = id - li * nblk;
  };
  auto issue = [&](long long k) {  // thread 0: rows of unit k -> stage k % NSTG
    int load;
    long long bx;
    unit_of(k, load, bx);
    const int stg = (int)(k % NSTG);
    const unsigned mb = sm_addr(mbar) + 8 * stg;
    const long long voff = (long long)load * g.c * g.n + bx * 8 * g.N1;
    const bool withp = MODE == CG && cx.st[load].iters > 0;
    mbar_expect_tx(mb, withp ? 2 * kRowsBytes : kRowsBytes);
    bulk_load(sm_addr(rin + stg * 8 * M), src + voff, kRowsBytes, mb);
    if (withp) bulk_load(sm_addr(pin + stg * 8 * M), cx.p + voff, kRowsBytes, mb);
  };
  if (t == 0)
    for (long long k = 0; k < NSTG && k < nunits; ++k) issue(k);
#pragma unroll 1
  for (long long k = 0; k < nunits; ++k) {
    int load;
    long long bx;
    unit_of(k, load, bx);
    const int stg = (int)(k % NSTG);
    const LoadState* st = cx.st + load;
    const long long row0 = bx * 8;  // row = (comp, z, y)
    const long long voff = (long long)load * g.c * g.n + (row0 + r) * g.N1;
    mbar_wait(sm_addr(mbar) + 8 * stg, (unsigned)((k / NSTG) & 1));
    const double2* rs = rin + stg * 8 * M + r * M;
    double2 v[8];
#pragma unroll
    for (int n2 = 0; n2 < 8; ++n2) v[n2] = rs[l16 + 16 * n2];
    double mx = 0.0;
    if (MODE == CG) {
      if (st->iters > 0) {  // r <- r - alpha p   (Alg 2 l.11)
        const double alpha = st->alpha;
        const double2* ps = pin + stg * 8 * M + r * M;
        double2* r2 = reinterpret_cast<double2*>(cx.r + voff);
#pragma unroll
        for (int n2 = 0; n2 < 8; ++n2) {
          const double2 pv = ps[l16 + 16 * n2];
          v[n2].x = fma(-alpha, pv.x, v[n2].x);
          v[n2].y = fma(-alpha, pv.y, v[n2].y);
          __stcg(r2 + l16 + 16 * n2, v[n2]);
        }
      }
#pragma unroll
      for (int n2 = 0; n2 < 8; ++n2) mx = fmax(mx, fmax(fabs(v[n2].x), fabs(v[n2].y)));
    }
    __syncthreads();  // every thread has read its part of the stage (and xs of the previous unit is consumed)
    if (t == 0 && k + NSTG < nunits) issue(k + NSTG);
    // stage 1 (thread = n1): DFT8 over n2 -> k1, twiddle w_128^{n1 k1} (table [k1][n1])
    dft_reg<8, false>(v);
#pragma unroll
    for (int k1 = 1; k1 < 8; ++k1) v[k1] = cmul(v[k1], tw[k1 * 16 + l16]);
#pragma unroll
    for (int k1 = 0; k1 < 8; ++k1) tb[r * RS + k1 * 17 + l16] = v[k1];
    __syncthreads();
    // stage 2 (thread = (k1, h)): half of DFT16 over n1 -> k2 = 2m + h ; X[k1 + 8 k2]
    {
      const int k1 = l16 >> 1, h = l16 & 1;
      double2 a[16], o[8];
#pragma unroll
      for (int n1 = 0; n1 < 16; ++n1) a[n1] = tb[r * RS + k1 * 17 + n1];
      dft_half<16, false>(a, h, tw16, o);
#pragma unroll
      for (int m = 0; m < 8; ++m) xs[r * XS + swz(k1 + 8 * (2 * m + h))] = o[m];
    }
    __syncthreads();
    // R2C post-processing: bins k and M - k of row c
    const int y0 = (int)(row0 % g.N2);
    const long long zc = row0 / g.N2;
    const int z = (int)(zc % g.P3);
    const int comp = (int)(zc / g.P3);
    double2* out = cx.spec + ((long long)load * g.c + comp) * g.nspec + (long long)z * g.N2 + y0;
    const long long plane = (long long)g.P3 * g.N2;
    for (int it = t; it < (M / 2 + 1) * 8; it += T) {
      const int c = it & 7, kk = it >> 3;
      const double2 a = xs[c * XS + swz(kk)];
      const double2 b = cconj(xs[c * XS + swz((M - kk) & (M - 1))]);
      const double2 E = make_double2(0.5 * (a.x + b.x), 0.5 * (a.y + b.y));
      const double2 O = mul_mi(make_double2(0.5 * (a.x - b.x), 0.5 * (a.y - b.y)));
      __stcg(out + (long long)kk * plane + c, cadd(E, cmul(twp[kk], O)));
      if (kk != M - kk) __stcg(out + (long long)(M - kk) * plane + c, cadd(cconj(E), cmul(twp[M - kk], cconj(O))));
    }
    if (MODE == CG) partial_write<true>(cx, RED_RNORM, load, (int)bx, mx, red_sh);
    else __syncthreads();  // xs is rewritten by the next unit
  }
}

bool xfwd256p_supported(const Geo& g) { return UNO_XFWD256P && g.N1 == 256 && !g.halo; }

int launch_xfwd256p(const Ctx& cx, int mode, const double* src, cudaStream_t s) {
  using namespace x2p;
  const Geo& g = cx.g;
  const long long total = (long long)g.c * g.P3 * g.N2 / 8 * g.nrhs;
  const dim3 grid((unsigned)(total < kCtas ? total : kCtas));
  constexpr int sm = (2 * NSTG * 8 * M + 8 * RS + 8 * XS + M + (M + 1) + 8) * (int)sizeof(double2);
  auto go = [&](auto k) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);  // per device: set on every launch
    k<<<grid, T, sm, s>>>(cx, src);
    return 1;
  };
  if (mode == CG) return go(xfwd256p_kernel<CG>);
  if (mode == PLAIN) return go(xfwd256p_kernel<PLAIN>);
  return go(xfwd256p_kernel<STANDALONE>);
}

}  // namespace uno
