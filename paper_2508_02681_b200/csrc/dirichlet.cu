// dirichlet.cu — all-Dirichlet boundaries (bc = {1,1,1}; Table 1 row "Dirichlet", P:451;
// SURVEY §8(f) rank 1): U = DST-I along every axis.
//
// Storage: the periodic layout [N3][N2][N1] with the boundary nodes (index 0 on any axis) held
// at zero.  Node N_i on the far face is node 0 of the periodic wrap, so the periodic K gather
// reads exactly the Dirichlet zeros, and K / RHS outputs are masked on the index-0 planes.
// P r: DST-I of every axis (odd extension of length 2N as a complex FFT on two packed real
// sequences, as dst.cu does along z), the per-mode c x c symbol multiply, and the DST-I again
// (self-inverse up to N/2 per axis, folded into the table).  The CG loop runs it as an opaque
// s = P r between the fused r and d passes of precond.cu, with gamma = r.s in its own pass.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "dev_common.cuh"
#include "fft.cuh"
#include "kernels.cuh"

namespace uno {

template <int L2>
__host__ __device__ constexpr int d3_smem_bytes() {
  return (8 * L2 + L2) * (int)sizeof(double2);
}

// One DST-I pass along `axis` (0 x, 1 y, 2 z) of every (load, comp) field, src -> dst (may alias).
// A CTA transforms 8 packed sequences (16 real ones): axes y, z pack adjacent x pairs (16-byte
// accesses, consecutive threads = consecutive pairs); axis x packs the rows y, y+1 (consecutive
// threads = consecutive x of one row).  gmul (c = 1, last forward axis): the scalar symbol
// multiply s_hat = G_hat r_hat of every sine mode is applied to the output (no separate pass).
template <int L2>
__global__ void __launch_bounds__(fft_threads(L2)) dst3_kernel(Ctx cx, const double* __restrict__ src,
                                                              double* __restrict__ dst, int axis, const double2* twl,
                                                              int gmul) {
  constexpr int T = fft_threads(L2);
  constexpr int N = L2 / 2;
  const Geo g = cx.g;
  extern __shared__ double2 smem[];
  double2* tile = smem;
  double2* tw = smem + 8 * L2;
  const int t = threadIdx.x;
  const int N1 = g.N1, N2 = g.N2;
  const long long plane = (long long)N1 * N2;
  long long base;   // offset of element j = 0 of packed sequence 0
  long long es;     // element stride (doubles)
  long long qs;     // stride between packed sequences (doubles)
  long long ps;     // stride between the two real halves of a packed sequence
  long long fbase;  // offset of the (load, comp) field
  {
    int b = blockIdx.x;
    if (axis == 0) {  // rows: 8 packed pairs = 16 rows y0..y0+15 of plane z
      const int nyb = N2 / 16;
      const int yb = b % nyb;
      b /= nyb;
      const int z = b % g.N3;
      const int lc = b / g.N3;
      fbase = (long long)lc * g.n;
      base = fbase + z * plane + (long long)yb * 16 * N1;
      es = 1;
      qs = 2LL * N1;
      ps = N1;
    } else {  // columns: 8 packed pairs = x0..x0+15 at fixed (y | z)
      const int nxb = N1 / 16;
      const int xb = b % nxb;
      b /= nxb;
      const int other = axis == 1 ? g.N3 : N2;
      const int o = b % other;
      const int lc = b / other;
      fbase = (long long)lc * g.n;
      base = fbase + xb * 16 + (axis == 1 ? (long long)o * plane : (long long)o * N1);
      es = axis == 1 ? N1 : plane;
      qs = 2;
      ps = 1;
    }
  }
  // every load of the tile is issued before the first smem store (unrolled: memory-level
  // parallelism); axes y, z read the packed pair (x, x+1) as one 16-byte access
  constexpr int NE = (8 * N + T - 1) / T;
  constexpr int LN = N >= 2 ? 31 - __builtin_clz(N) : 0;  // log2 N
  const bool vec = ps == 1, rowmap = axis == 0;
  auto jq = [&](int e, int& j, int& q) {
    j = rowmap ? (e & (N - 1)) : (e >> 3);
    q = rowmap ? (e >> LN) : (e & 7);
  };
  double2 vals[NE];
#pragma unroll
  for (int i = 0; i < NE; ++i) {
    const int e = t + i * T;
    int j, q;
    jq(e, j, q);
    vals[i] = make_double2(0.0, 0.0);
    if (e < 8 * N && j > 0) {
      const long long a = base + q * qs + j * es;
      vals[i] = vec ? __ldcg(reinterpret_cast<const double2*>(src + a)) : make_double2(__ldcg(src + a), __ldcg(src + a + ps));
    }
  }
  for (int i = t; i < L2; i += T) tw[i] = twl[i];
#pragma unroll
  for (int i = 0; i < NE; ++i) {
    const int e = t + i * T;
    int j, q;
    jq(e, j, q);
    if (e < 8 * N) {
      tile[tidx(j, q)] = vals[i];
      if (j > 0) tile[tidx(L2 - j, q)] = make_double2(-vals[i].x, -vals[i].y);
    }
  }
  if (t < 8) tile[tidx(N, t)] = make_double2(0.0, 0.0);
  __syncthreads();
  fft_tile<L2, false>(tile, tw);
  // sine coefficients m = 1..N-1 of the two halves: (-Im Y_m, Re Y_m) / 2; m = 0 stays 0
#pragma unroll
  for (int i = 0; i < NE; ++i) {
    const int e = t + i * T;
    int m, q;
    jq(e, m, q);
    if (e < 8 * N) {
      const long long a = base + q * qs + m * es;
      double2 o = make_double2(0.0, 0.0);
      if (m > 0) {
        const double2 Y = tile[tidx(m, q)];
        o = make_double2(-0.5 * Y.y, 0.5 * Y.x);
        if (gmul) {
          o.x *= __ldg(cx.gtab + (a - fbase));
          o.y *= __ldg(cx.gtab + (a + ps - fbase));
        }
      }
      if (vec) {
        __stcg(reinterpret_cast<double2*>(dst + a), o);
      } else {
        __stcg(dst + a, o.x);
        __stcg(dst + a + ps, o.y);
      }
    }
  }
}

// Register-direct DST-I pass for N = 256 (odd extension of length 512): 4 packed sequences per
// CTA, thread (q, l) = (t & 3, t >> 2).  Each thread loads its 16 odd-extension entries
// y_{l + 32 n2} straight into registers (y_j = x_j for j < 256, y_j = -x_{512-j} above; x_0 =
// x_256 = 0 are the Dirichlet nodes — the mirrored half re-reads the tile through L1), then the
// four-step FFT of gpass512_kernel (DFT16 -> twiddle -> transpose -> DFT32 split between thread
// pairs) leaves bins k1 + 16 (2m + h) in registers, of which the 255 sine modes k < 256 are stored
// (-Im Y_k, Re Y_k) / 2 (times the scalar symbol when gmul).  Buffers 546 apart, rows of 34: the
// quarter-warp patterns of gpass512_kernel, conflict-free.
constexpr int D5_C = 4, D5_CS = 546, D5_T = 32 * D5_C;
constexpr int dst512r_smem = (D5_C * D5_CS + 16 * 32 + 16) * 16;
__global__ void __launch_bounds__(D5_T, 4) dst512r_kernel(Ctx cx, const double* __restrict__ src,
                                                          double* __restrict__ dst, int axis, const double2* twl,
                                                          int gmul) {
  constexpr int L = 512, N = 256;
  const Geo g = cx.g;
  extern __shared__ double2 dsm[];
  double2* buf = dsm;                 // [D5_C][D5_CS]
  double2* tw = buf + D5_C * D5_CS;   // [k1][n1] = w_512^{k1 n1}
  double2* tw32 = tw + 16 * 32;       // w_32^r
  const int t = threadIdx.x, c = t & (D5_C - 1), l32 = t >> 2;
  const int N1 = g.N1, N2 = g.N2;
  const long long plane = (long long)N1 * N2;
  long long base, es, qs, ps, fbase;
  {
    int b = blockIdx.x;
    if (axis == 0) {  // rows: 4 packed pairs = rows y0..y0+7 of plane z
      const int nyb = N2 / 8;
      const int yb = b % nyb;
      b /= nyb;
      const int z = b % g.N3;
      fbase = (long long)(b / g.N3) * g.n;
      base = fbase + z * plane + (long long)yb * 8 * N1;
      es = 1;
      qs = 2LL * N1;
      ps = N1;
    } else {  // columns: 4 packed pairs = x0..x0+7 at fixed (y | z)
      const int nxb = N1 / 8;
      const int xb = b % nxb;
      b /= nxb;
      const int other = axis == 1 ? g.N3 : N2;
      const int o = b % other;
      fbase = (long long)(b / other) * g.n;
      base = fbase + xb * 8 + (axis == 1 ? (long long)o * plane : (long long)o * N1);
      es = axis == 1 ? N1 : plane;
      qs = 2;
      ps = 1;
    }
  }
  const bool vec = ps == 1;
  const long long sq = base + c * qs;
  auto ld = [&](int j) -> double2 {  // x_j of this packed sequence, 0 < j < N
    const double* p = src + sq + j * es;
    return vec ? __ldg(reinterpret_cast<const double2*>(p)) : make_double2(__ldg(p), __ldg(p + ps));
  };
  double2 v[16];
#pragma unroll
  for (int n2 = 0; n2 < 16; ++n2) {
    const int j = l32 + 32 * n2;
    if (n2 < 8) {
      v[n2] = j == 0 ? make_double2(0.0, 0.0) : ld(j);
    } else {
      const int jj = L - j;  // 1 .. 256
      const double2 x = jj == N ? make_double2(0.0, 0.0) : ld(jj);
      v[n2] = make_double2(-x.x, -x.y);
    }
  }
  for (int i = t; i < 16 * 32; i += D5_T) tw[i] = twl[((i & 31) * (i >> 5)) & (L - 1)];
  if (t < 16) tw32[t] = twl[16 * t];
  __syncthreads();
  double2* B = buf + c * D5_CS;
  dft_reg<16, false>(v);  // thread = n1: over n2 -> k1
#pragma unroll
  for (int k1 = 1; k1 < 16; ++k1) v[k1] = cmul(v[k1], tw[k1 * 32 + l32]);
#pragma unroll
  for (int k1 = 0; k1 < 16; ++k1) B[k1 * 34 + l32] = v[k1];
  __syncthreads();
  const int k1 = l32 >> 1, h = l32 & 1;
  double2 o[16];
  {
    double2 a[32];
#pragma unroll
    for (int n1 = 0; n1 < 32; ++n1) a[n1] = B[k1 * 34 + n1];
    dft_half<32, false>(a, h, tw32, o);  // o[m] = Y(k1 + 16 (2m + h))
  }
#pragma unroll
  for (int m = 0; m < 8; ++m) {  // sine modes k = k1 + 16 (2m + h) < 256
    const int k = k1 + 16 * (2 * m + h);
    const long long a = sq + k * es;
    double2 r = make_double2(0.0, 0.0);
    if (k > 0) {
      r = make_double2(-0.5 * o[m].y, 0.5 * o[m].x);
      if (gmul) {
        r.x *= __ldg(cx.gtab + (a - fbase));
        r.y *= __ldg(cx.gtab + (a + ps - fbase));
      }
    }
    if (vec) {
      __stcg(reinterpret_cast<double2*>(dst + a), r);
    } else {
      __stcg(dst + a, r.x);
      __stcg(dst + a + ps, r.y);
    }
  }
}

// s_hat = G_hat s_hat per sine mode (c x c, unique entries in Eq B7 order), in place
__global__ void d3_gmul_kernel(Ctx cx, double* __restrict__ v) {
  const Geo g = cx.g;
  const long long n = g.n;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    for (int l = 0; l < g.nrhs; ++l) {
      double* w = v + (long long)l * g.c * n;
      if (g.c == 1) {
        w[i] *= cx.gtab[i];
      } else if (g.c == 2) {
        const double g1 = cx.gtab[i], g2 = cx.gtab[n + i], g3 = cx.gtab[2 * n + i];
        const double a = w[i], b = w[n + i];
        w[i] = fma(g1, a, g3 * b);
        w[n + i] = fma(g3, a, g2 * b);
      } else {
        const double* G = cx.gtab;
        const double g1 = G[i], g2 = G[n + i], g3 = G[2 * n + i], g4 = G[3 * n + i], g5 = G[4 * n + i],
                     g6 = G[5 * n + i];
        const double a = w[i], b = w[n + i], c = w[2 * n + i];
        w[i] = fma(g1, a, fma(g3, b, g6 * c));
        w[n + i] = fma(g3, a, fma(g2, b, g5 * c));
        w[2 * n + i] = fma(g6, a, fma(g5, b, g4 * c));
      }
    }
  }
}

// gamma_1 = r.s partial per CTA (fixed grid: jacobi_nblk)
__global__ void __launch_bounds__(256) d3_dot_kernel(Ctx cx, const double* __restrict__ a, const double* __restrict__ b,
                                                     int mode) {
  const Geo g = cx.g;
  const int load = blockIdx.y;
  if (mode == CG && !cx.st[load].active) return;
  __shared__ double red_sh[32];
  const long long cn = (long long)g.c * g.n;
  const double* x = a + (long long)load * cn;
  const double* y = b + (long long)load * cn;
  double acc = 0.0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < cn; i += (long long)gridDim.x * blockDim.x)
    acc = fma(x[i], y[i], acc);
  partial_write<false>(cx, RED_GAMMA, load, blockIdx.x, acc, red_sh);
}

// all-Dirichlet symbol on [N3][N2][N1] (mode m_i at index m_i; index-0 entries 0), already
// scaled by (2/N1)(2/N2)(2/N3) (unnormalised DST-I round trips).  Closed form of the diagonal
// block (SURVEY A3 with theta_i = pi m_i / N_i and S_ij = 0 for i != j); perturbation of
// SURVEY A8 at canon(m) = ((m3-1)(N2-1) + (m2-1))(N1-1) + (m1-1) (oracle/greens.ghat_dirichlet).
__global__ void d3_symbol_kernel(Ctx cx, double* gtab, double ref0, double ref1, unsigned long long seed, double amp) {
  const Geo g = cx.g;
  const long long b = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= g.n) return;
  const int N1 = g.N1, N2 = g.N2, N3 = g.N3;
  const int s1 = __ffs(N1) - 1, s2 = __ffs(N2) - 1;
  const int m1 = (int)(b & (N1 - 1)), m2 = (int)((b >> s1) & (N2 - 1)), m3 = (int)(b >> (s1 + s2));
  const long long n = g.n;
  if (m1 == 0 || m2 == 0 || m3 == 0) {
    for (int q = 0; q < g.C; ++q) gtab[q * n + b] = 0.0;
    return;
  }
  double cs[3], omc[3];  // cos theta_i and 1 - cos theta_i = 2 sin^2(theta_i / 2), theta_i = pi m_i / N_i
  const int mm[3] = {m1, m2, m3}, NN[3] = {N1, N2, N3};
  for (int i = 0; i < 3; ++i) {
    cs[i] = cospi((double)mm[i] / NN[i]);
    const double sh = sinpi((double)mm[i] / (2.0 * NN[i]));
    omc[i] = 2.0 * sh * sh;
  }
  const double h = g.h;
  double mass[3], S[3];
  for (int i = 0; i < 3; ++i) mass[i] = (h / 3.0) * (2.0 + cs[i]);
  for (int i = 0; i < 3; ++i) {
    double v = (2.0 / h) * omc[i];
    for (int j = 0; j < 3; ++j)
      if (j != i) v *= mass[j];
    S[i] = v;
  }
  const double scale = 8.0 / ((double)N1 * N2 * N3);
  const unsigned long long canon = ((unsigned long long)(m3 - 1) * (N2 - 1) + (m2 - 1)) * (N1 - 1) + (m1 - 1);
  const double tr = (S[0] + S[1]) + S[2];
  if (g.c == 1) {
    const double rho = seed ? (1.0 - amp + 2.0 * amp * u01(seed, 2, canon)) : 1.0;
    gtab[b] = rho / (tr * ref0) * scale;
    return;
  }
  double P[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
  for (int i = 0; i < 3; ++i) P[i][i] = 1.0 / ((ref0 + ref1) * S[i] + ref1 * tr);
  if (seed) {
    double th[6];
    for (int t = 0; t < 6; ++t) th[t] = u01(seed, 2, 8ULL * canon + t);
    th[0] = 0.5 + 0.5 * th[0];
    th[1] = 0.5 + 0.5 * th[1];
    th[3] = 0.5 + 0.5 * th[3];
    th[2] -= 0.5;
    th[4] -= 0.5;
    th[5] -= 0.5;
    const double t1 = th[0], t2 = th[1], t3 = th[2], t4 = th[3], t5 = th[4], t6 = th[5];
    const double psi[3][3] = {{t1 * t1, t1 * t3, t1 * t6},  // psi = L L^T, Eq B5
                              {t1 * t3, t2 * t2 + t3 * t3, t2 * t5 + t3 * t6},
                              {t1 * t6, t2 * t5 + t3 * t6, t4 * t4 + t5 * t5 + t6 * t6}};
    const double a = amp * (P[0][0] + P[1][1] + P[2][2]) / 3.0;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) P[i][j] += a * psi[i][j];
  }
  gtab[b] = P[0][0] * scale;
  gtab[n + b] = P[1][1] * scale;
  gtab[2 * n + b] = P[0][1] * scale;
  gtab[3 * n + b] = P[2][2] * scale;
  gtab[4 * n + b] = P[1][2] * scale;
  gtab[5 * n + b] = P[0][2] * scale;
}

// 2D symbols of the padded storage: dmask 3 (Dirichlet x, y: real per node [y][x], modes at index m)
// and dmask 2 (periodic x, Dirichlet y: R2C half spectrum [kx][y-mode]); closed form of the diagonal
// block (SURVEY A3 in 2D, S_xy dropped), perturbation of SURVEY A8 with Eq 45 for c = 2 at the canon
// index of oracle/greens.ghat_dirichlet / ghat_mixed2d.
__global__ void d2_symbol_kernel(Ctx cx, double* gtab, double ref0, double ref1, unsigned long long seed, double amp) {
  const Geo g = cx.g;
  const long long b = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long ns = g.nspec;
  if (b >= ns) return;
  const int N1 = g.N1, N2 = g.N2;
  int kx, m;
  double cx_, cy, scale, omx, omy;  // cosines and 1 - cos = 2 sin^2(half angle)
  unsigned long long canon;
  bool zero;
  if (g.dmask == 3) {
    kx = (int)(b % N1);  // sine mode m1
    m = (int)(b / N1);
    zero = kx == 0 || m == 0;
    cx_ = cospi((double)kx / N1);
    const double sh = sinpi((double)kx / (2.0 * N1));
    omx = 2.0 * sh * sh;
    scale = 4.0 / ((double)N1 * N2);
    canon = zero ? 0 : (unsigned long long)(m - 1) * (N1 - 1) + (kx - 1);
  } else {
    kx = (int)(b / N2);  // layout [kx][z = 0][y]
    m = (int)(b % N2);
    zero = m == 0;
    const int ka = 2 * kx <= N1 ? kx : N1 - kx;
    cx_ = cospi(2.0 * ka / N1);
    const double sh = sinpi((double)ka / N1);
    omx = 2.0 * sh * sh;
    scale = 2.0 / ((double)N1 * N2);
    const unsigned long long p = zero ? 0 : (unsigned long long)(m - 1);
    const unsigned long long f1 = p * N1 + kx, f2 = p * N1 + (unsigned long long)((N1 - kx) % N1);
    canon = f1 < f2 ? f1 : f2;
  }
  if (zero) {
    for (int q = 0; q < g.C; ++q) gtab[q * ns + b] = 0.0;
    return;
  }
  cy = cospi((double)m / N2);
  {
    const double sh = sinpi((double)m / (2.0 * N2));
    omy = 2.0 * sh * sh;
  }
  const double Sxx = (2.0 / 3.0) * omx * (2.0 + cy), Syy = (2.0 / 3.0) * omy * (2.0 + cx_);
  const double tr = Sxx + Syy;
  if (g.c == 1) {
    const double rho = seed ? (1.0 - amp + 2.0 * amp * u01(seed, 2, canon)) : 1.0;
    gtab[b] = rho / (tr * ref0) * scale;
    return;
  }
  double P11 = 1.0 / ((ref0 + ref1) * Sxx + ref1 * tr), P22 = 1.0 / ((ref0 + ref1) * Syy + ref1 * tr), P12 = 0.0;
  if (seed) {  // Eq 45: theta_1,2 in [0.5, 1], theta_3 in [-0.5, 0.5]
    const double t1 = 0.5 + 0.5 * u01(seed, 2, 8ULL * canon), t2 = 0.5 + 0.5 * u01(seed, 2, 8ULL * canon + 1);
    const double t3 = u01(seed, 2, 8ULL * canon + 2) - 0.5;
    const double a = amp * (P11 + P22) / 2.0;
    P11 += a * t1 * t1;
    P22 += a * (t2 * t2 + t3 * t3);
    P12 += a * t1 * t3;
  }
  gtab[b] = P11 * scale;
  gtab[ns + b] = P22 * scale;
  gtab[2 * ns + b] = P12 * scale;
}

template <class F>
static int d3_dispatch(int L2, F&& f) {
  switch (L2) {
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

static int launch_dst3(const Ctx& cx, const double* src, double* dst, int axis, const double2* twl, cudaStream_t s,
                       int gmul = 0) {
  const Geo& g = cx.g;
  const int N = axis == 0 ? g.N1 : (axis == 1 ? g.N2 : g.N3);
  const long long nlc = (long long)g.nrhs * g.c;
  const long long nb = axis == 0 ? nlc * g.N3 * (g.N2 / 16) : nlc * (axis == 1 ? g.N3 : g.N2) * (g.N1 / 16);
  if (N == 256 && (axis == 0 ? g.N2 % 8 == 0 : g.N1 % 8 == 0)) {
    const long long nb8 = axis == 0 ? nlc * g.N3 * (g.N2 / 8) : nlc * (axis == 1 ? g.N3 : g.N2) * (g.N1 / 8);
    dst512r_kernel<<<(unsigned)nb8, D5_T, dst512r_smem, s>>>(cx, src, dst, axis, twl, gmul);
    return 1;
  }
  return d3_dispatch(2 * N, [&](auto Lc) {
    constexpr int L2 = decltype(Lc)::value;
    const int sm = d3_smem_bytes<L2>();
    if (sm > 48 * 1024) cudaFuncSetAttribute(dst3_kernel<L2>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    dst3_kernel<L2><<<(unsigned)nb, fft_threads(L2), sm, s>>>(cx, src, dst, axis, twl, gmul);
    return 1;
  });
}

// 2D mixed (periodic x, Dirichlet y): s_hat = G_hat s_hat on the R2C half spectrum [c][kx][y-mode]
// (complex values, real symmetric c x c symbol), in place
__global__ void d2m_gmul_kernel(Ctx cx, double2* __restrict__ spec) {
  const Geo g = cx.g;
  const long long ns = g.nspec;
  for (long long b = (long long)blockIdx.x * blockDim.x + threadIdx.x; b < ns; b += (long long)gridDim.x * blockDim.x) {
    for (int l = 0; l < g.nrhs; ++l) {
      double2* w = spec + (long long)l * g.c * ns;
      if (g.c == 1) {
        w[b] = cscale(w[b], cx.gtab[b]);
      } else {
        const double g1 = cx.gtab[b], g2 = cx.gtab[ns + b], g3 = cx.gtab[2 * ns + b];
        const double2 a = w[b], c = w[ns + b];
        w[b] = make_double2(fma(g1, a.x, g3 * c.x), fma(g1, a.y, g3 * c.y));
        w[ns + b] = make_double2(fma(g3, a.x, g2 * c.x), fma(g3, a.y, g2 * c.y));
      }
    }
  }
}

// s = P r for all nrhs fields: DST-I on every Dirichlet axis of the padded storage; for the 2D
// mixed case the x axis in between is the periodic R2C machinery (xfwd / xinv, standalone).
int launch_d3_precond(const Ctx& cx, const double* r, double* sbuf, const double2* const tw2[3], cudaStream_t s) {
  const Geo& g = cx.g;
  int n = 0, k;
  const long long gb = std::min<long long>((g.n + 255) / 256, 148 * 16);
  if (g.dim == 2 && g.dmask == 2) {  // F_x (x) S_y
    if ((k = launch_dst3(cx, r, sbuf, 1, tw2[1], s)) < 0) return -1;
    n += k;
    if ((k = launch_xfwd(cx, STANDALONE, sbuf, s)) < 0) return -1;
    n += k;
    const long long sb = std::min<long long>((g.nspec + 255) / 256, 148 * 16);
    d2m_gmul_kernel<<<(unsigned)sb, 256, 0, s>>>(cx, cx.spec);
    ++n;
    if ((k = launch_xinv(cx, STANDALONE, sbuf, s)) < 0) return -1;
    n += k;
    if ((k = launch_dst3(cx, sbuf, sbuf, 1, tw2[1], s)) < 0) return -1;
    return n + k;
  }
  const int fuse = g.c == 1;  // scalar symbol: multiplied in the last forward DST pass
  if ((k = launch_dst3(cx, r, sbuf, 0, tw2[0], s, fuse && g.dim == 1)) < 0) return -1;
  n += k;
  for (int axis = 1; axis < g.dim; ++axis) {
    if ((k = launch_dst3(cx, sbuf, sbuf, axis, tw2[axis], s, fuse && axis == g.dim - 1)) < 0) return -1;
    n += k;
  }
  if (!fuse) {
    d3_gmul_kernel<<<(unsigned)gb, 256, 0, s>>>(cx, sbuf);
    ++n;
  }
  for (int axis = g.dim - 1; axis >= 0; --axis) {
    if ((k = launch_dst3(cx, sbuf, sbuf, axis, tw2[axis], s)) < 0) return -1;
    n += k;
  }
  return n;
}

int launch_d3_dot(const Ctx& cx, const double* a, const double* b, int mode, cudaStream_t s) {
  const dim3 grid(jacobi_nblk(cx.g), cx.g.nrhs);
  d3_dot_kernel<<<grid, 256, 0, s>>>(cx, a, b, mode);
  return 1;
}

int launch_d3_symbol(const Ctx& cx, double* gtab, double ref0, double ref1, unsigned long long seed, double amp,
                     cudaStream_t s) {
  if (cx.g.dim == 2)
    d2_symbol_kernel<<<(unsigned)((cx.g.nspec + 255) / 256), 256, 0, s>>>(cx, gtab, ref0, ref1, seed, amp);
  else
    d3_symbol_kernel<<<(unsigned)((cx.g.n + 255) / 256), 256, 0, s>>>(cx, gtab, ref0, ref1, seed, amp);
  return 1;
}

}  // namespace uno
