// slab.cu — z-slab decomposition of one UNO-CG problem (include/uno_cg_slab.h).
//
// Three views of the same rank-local data drive the existing kernels unchanged:
//   gxy  the slab as a grid of Z planes (x and y passes, CG vector updates): N3 := Z
//   gz   this rank's pencil: k_y chunk [ky0, ky0 + Yc) of every kx plane with all N3 k_z
//        (z FFT, symbol, Parseval gamma partial): N2 := Yc, N3 global, Ny/ky0 for the symbol
//   gk   the slab inside the global grid (K, RHS): N3 global, P3 := Z, zlo = rank Z, halo
//        planes from Ctx::hlo / Ctx::hhi
// plus pack / unpack kernels between the slab spectrum [l][c][kx][z][y] and the all-to-all
// blocks [q][l][c][kx][z][yc].  Scalars: per-rank partial (scalar_kernel, standalone mode)
// -> caller all-reduce -> slab_apply_kernel (the same device CG logic as the whole-grid loop).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/uno_cg_slab.h"
#include "common.cuh"
#include "dev_common.cuh"
#include "kernels.cuh"

namespace uno {
uno_status set_last_error(uno_status s, const char* msg);  // uno_cg.cu
}
using namespace uno;

static uno_status sfail(uno_status s, const std::string& m) { return set_last_error(s, m.c_str()); }
#define SCK(call)                                                                                  \
  do {                                                                                             \
    cudaError_t e_ = (call);                                                                       \
    if (e_ != cudaSuccess) return sfail(UNO_ERR_CUDA, std::string(#call ": ") + cudaGetErrorString(e_)); \
  } while (0)
#define SKL(expr)                                                                     \
  do {                                                                                \
    if ((expr) < 0) return sfail(UNO_ERR_SHAPE, "no kernel instance for this slab"); \
  } while (0)

struct uno_slab_handle {
  uno_cg_desc desc;
  int rank, nranks, Z, Yc;
  cudaStream_t s;
  const uint8_t* phase;
  Geo gxy, gz, gk;
  Ctx cxy, cz, ck;
  double ref0, ref1;
  double *r, *d, *p, *u;
  double2 *spec, *pencil;
  double* gtab;
  double2 *twx, *twxp, *twy, *twz, *twz2;
  LoadState* st;
  LoadState* h_st;
  double *partials, *results, *scratch;
  unsigned* counters;
};

// ---------------------------------------------------------------------------------------- kernels
// forward pack: slab spectrum S[row][y] (row = (lc, kx, z), N2 per row) -> send[q][row][yc],
// y = q Yc + yc; unpack is the inverse.  grid.z = q, grid.y strides the rows, threads the yc
// of a row (contiguous on both sides), 16-byte elements, no 64-bit divisions.
__global__ void slab_pack_kernel(const double2* __restrict__ S, double2* __restrict__ out, long long rows, int Yc,
                                 int N2) {
  const int q = blockIdx.z;
  const int ty = threadIdx.x / Yc, yc = threadIdx.x - ty * Yc, rpb = blockDim.x / Yc;
  double2* o = out + (long long)q * rows * Yc;
  for (long long row = (long long)blockIdx.y * rpb + ty; row < rows; row += (long long)gridDim.y * rpb)
    o[row * Yc + yc] = S[row * N2 + (long long)q * Yc + yc];
}
// peer variant: block q goes straight to rank q's receive buffer (block `rank` of it)
constexpr int kMaxRanks = 8;
struct SlabPeers {
  double2* p[kMaxRanks];
};
__global__ void slab_pack_peer_kernel(const double2* __restrict__ S, SlabPeers peers, int rank, long long rows, int Yc,
                                      int N2) {
  const int q = blockIdx.z;
  const int ty = threadIdx.x / Yc, yc = threadIdx.x - ty * Yc, rpb = blockDim.x / Yc;
  double2* o = peers.p[q] + (long long)rank * rows * Yc;
  for (long long row = (long long)blockIdx.y * rpb + ty; row < rows; row += (long long)gridDim.y * rpb)
    o[row * Yc + yc] = S[row * N2 + (long long)q * Yc + yc];
  __threadfence_system();
}
__global__ void slab_unpack_kernel(const double2* __restrict__ in, double2* __restrict__ S, long long rows, int Yc,
                                   int N2) {
  const int q = blockIdx.z;
  const int ty = threadIdx.x / Yc, yc = threadIdx.x - ty * Yc, rpb = blockDim.x / Yc;
  const double2* src = in + (long long)q * rows * Yc;
  for (long long row = (long long)blockIdx.y * rpb + ty; row < rows; row += (long long)gridDim.y * rpb)
    S[row * N2 + (long long)q * Yc + yc] = src[row * Yc + yc];
}
// recv[q][lckx][zq][yc] <-> pencil P[lckx][q Z + zq][yc]: both sides are contiguous runs of Z Yc
// (dir 0: into the pencil)
__global__ void slab_pencil_kernel(double2* __restrict__ buf, double2* __restrict__ P, long long nlckx, int Z, int Yc,
                                   int N3, int dir) {
  const int q = blockIdx.z;
  const long long run = (long long)Z * Yc;
  for (long long lk = blockIdx.y; lk < nlckx; lk += gridDim.y) {
    double2* b = buf + ((long long)q * nlckx + lk) * run;
    double2* p = P + lk * (long long)N3 * Yc + (long long)q * run;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < run; i += (long long)gridDim.x * blockDim.x) {
      if (dir == 0)
        p[i] = b[i];
      else
        b[i] = p[i];
    }
  }
}
// pencil -> block `rank` of every rank q's receive buffer (peer variant of dir 1)
__global__ void slab_pencil_peer_kernel(SlabPeers peers, int rank, const double2* __restrict__ P, long long nlckx,
                                        int Z, int Yc, int N3) {
  const int q = blockIdx.z;
  const long long run = (long long)Z * Yc;
  for (long long lk = blockIdx.y; lk < nlckx; lk += gridDim.y) {
    double2* b = peers.p[q] + ((long long)rank * nlckx + lk) * run;
    const double2* p = P + lk * (long long)N3 * Yc + (long long)q * run;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < run; i += (long long)gridDim.x * blockDim.x)
      b[i] = p[i];
  }
  __threadfence_system();
}
// halo send: plane 0 and plane Z-1 of every (load, comp) slab of d -> out[2][lc][plane]
// peer variant: my first plane -> recv[1] of rank-1, my last plane -> recv[0] of rank+1
__global__ void slab_halo_peer_kernel(const double* __restrict__ d, double* lo_dst, double* hi_dst, int nlc, int Z,
                                      long long plane) {
  const long long tot = 2LL * nlc * plane;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (long long)gridDim.x * blockDim.x) {
    const long long side = e / ((long long)nlc * plane), rem = e - side * nlc * plane;
    const long long lc = rem / plane, xy = rem - lc * plane;
    (side ? hi_dst : lo_dst)[rem] = d[(lc * Z + (side ? Z - 1 : 0)) * plane + xy];
  }
  __threadfence_system();
}
__global__ void slab_halo_kernel(const double* __restrict__ d, double* __restrict__ out, int nlc, int Z, long long plane) {
  const long long tot = 2LL * nlc * plane;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (long long)gridDim.x * blockDim.x) {
    const long long side = e / ((long long)nlc * plane), rem = e - side * nlc * plane;
    const long long lc = rem / plane, xy = rem - lc * plane;
    out[e] = d[(lc * Z + (side ? Z - 1 : 0)) * plane + xy];
  }
}
// cross-rank totals -> CG scalar logic (dev_common.cuh), one thread per load
__global__ void slab_apply_kernel(LoadState* st, int nrhs, int slot, const double* tot) {
  const int l = threadIdx.x;
  if (l >= nrhs || !st[l].active) return;
  if (slot == RED_RNORM) scalar_after_rnorm(st + l, tot[l], nullptr, 0, l);
  else if (slot == RED_GAMMA) scalar_after_gamma(st + l, tot[l]);
  else scalar_after_dp(st + l, tot[l]);
}
__global__ void slab_means_kernel(const double* __restrict__ u, long long n, double* means) {
  __shared__ double sh[32];
  const double* v = u + (long long)blockIdx.x * n;
  double acc = 0.0;
  for (long long i = threadIdx.x; i < n; i += blockDim.x) acc += v[i];  // fixed order per thread
  const double b = block_reduce<false>(acc, sh);
  if (threadIdx.x == 0) means[blockIdx.x] = b / (double)n;
}
__global__ void slab_subtract_kernel(double* __restrict__ u, long long n, const double* mean_sums, double inv_ranks) {
  const double m = mean_sums[blockIdx.y] * inv_ranks;  // equal slabs: global mean = mean of slab means
  double* v = u + (long long)blockIdx.y * n;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    v[i] -= m;
}

static unsigned grid_for(long long n) {
  long long b = (n + 255) / 256;
  return (unsigned)(b > 148 * 16 ? 148 * 16 : (b < 1 ? 1 : b));
}

static int pack_threads(int Yc) { return Yc >= 256 ? Yc : 256; }  // whole rows per CTA (Yc | 256 or Yc >= 256)
static dim3 pack_grid(long long rows, int Yc, int nranks) {
  const long long rpb = pack_threads(Yc) / Yc;
  const long long nb = (rows + rpb - 1) / rpb;
  return dim3(1, (unsigned)std::min<long long>(nb, 8192), nranks);
}

static void twid(int L, int denom, std::vector<double2>& out) {
  out.resize(L);
  for (int m = 0; m < L; ++m) {
    const long double a = -2.0L * 3.14159265358979323846264338327950288L * (long double)m / (long double)denom;
    out[m].x = (double)cosl(a);
    out[m].y = (double)sinl(a);
  }
}

static void free_slab(uno_slab_handle* h) {
  if (!h) return;
  void* bufs[] = {h->r, h->d, h->p, h->u, h->spec, h->pencil, h->gtab, h->twx, h->twxp, h->twy, h->twz, h->twz2,
                  h->st, h->partials, h->results, h->scratch, h->counters};
  for (void* b : bufs)
    if (b) cudaFreeAsync(b, h->s);
  if (h->h_st) cudaFreeHost(h->h_st);
  delete h;
}

static bool pow2(int v) { return v > 0 && (v & (v - 1)) == 0; }

extern "C" uno_status uno_slab_create(const uno_cg_desc* desc, int32_t rank, int32_t nranks, const uint8_t* d_phase,
                                      uno_slab_handle** out) {
  if (!desc || !d_phase || !out) return sfail(UNO_ERR_ARG, "null argument");
  *out = nullptr;
  const uno_cg_desc& D = *desc;
  if (D.dim != 3) return sfail(UNO_ERR_UNSUPPORTED, "slab mode: 3D grids only");
  const bool dirz = D.bc[0] == 0 && D.bc[1] == 0 && D.bc[2] == 1;  // mixed BC of config 4 (Eq 82)
  if (!dirz && (D.bc[0] || D.bc[1] || D.bc[2]))
    return sfail(UNO_ERR_UNSUPPORTED, "slab mode: periodic, or periodic x, y with Dirichlet z");
  if (nranks < 1 || rank < 0 || rank >= nranks) return sfail(UNO_ERR_ARG, "rank / nranks");
  const int N1 = D.n[0], N2 = D.n[1], N3 = D.n[2];
  const int c = D.physics == UNO_THERMAL ? 1 : 3;
  if (!pow2(N1) || !pow2(N2) || !pow2(N3) || !pow2(nranks) || N3 % nranks || N2 % nranks)
    return sfail(UNO_ERR_SHAPE, "slab mode: powers of two with N2, N3 divisible by nranks");
  const int Z = N3 / nranks, Yc = N2 / nranks;
  if (Yc < 8 || N1 > 1024 || N2 > 1024 || N3 > 1024 || (c == 1 && (N1 < 32 || N2 < 16)) || (c == 3 && N1 < 16))
    return sfail(UNO_ERR_SHAPE, "slab mode: Yc = N2/nranks >= 8; thermal N1 >= 32, N2 >= 16; elastic N1 >= 16");
  if (D.nrhs < 1 || D.nrhs > kMaxRhs) return sfail(UNO_ERR_ARG, "nrhs must be 1..8");
  if (D.physics == UNO_THERMAL) {
    if (!(D.mat[0][0] > 0) || !(D.mat[1][0] > 0)) return sfail(UNO_ERR_ARG, "conductivities must be > 0");
  } else {
    for (int p = 0; p < 2; ++p)
      if (!(D.mat[p][1] > 0) || !(D.mat[p][0] >= 0)) return sfail(UNO_ERR_ARG, "need mu > 0, lambda >= 0");
  }
  uno_slab_handle* h = new uno_slab_handle();
  h->desc = D;
  h->rank = rank;
  h->nranks = nranks;
  h->Z = Z;
  h->Yc = Yc;
  h->s = (cudaStream_t)D.stream;
  h->phase = d_phase;
  Geo base;
  std::memset(&base, 0, sizeof(base));
  base.dim = 3;
  base.c = c;
  base.nrhs = D.nrhs;
  base.N1 = N1;
  base.M = N1 / 2;
  base.H1 = base.M + 1;
  base.h = D.h > 0 ? D.h : 1.0 / N1;
  base.C = c * (c + 1) / 2;
  // slab as a Z-plane grid
  Geo& gxy = h->gxy;
  gxy = base;
  gxy.N2 = N2;
  gxy.N3 = Z;
  gxy.P3 = Z;
  gxy.n = (long long)N1 * N2 * Z;
  gxy.nspec = (long long)gxy.H1 * N2 * Z;
  gxy.KZC = Z < 32 ? Z : 32;
  gxy.Ny = N2;
  // pencil
  Geo& gz = h->gz;
  gz = base;
  gz.N2 = Yc;
  gz.N3 = N3;
  gz.P3 = N3;
  gz.n = (long long)N1 * Yc * N3;
  gz.nspec = (long long)gz.H1 * Yc * N3;
  gz.KZC = N3 < 32 ? N3 : 32;
  gz.Ny = N2;
  gz.ky0 = rank * Yc;
  // slab inside the global grid
  Geo& gk = h->gk;
  gk = base;
  gk.N2 = N2;
  gk.N3 = N3;
  gk.P3 = Z;
  gk.n = (long long)N1 * N2 * Z;
  gk.nspec = gxy.nspec;
  gk.KZC = Z < 32 ? Z : 32;
  gk.zlo = rank * Z;
  gk.halo = 1;
  gk.Ny = N2;
  if (dirz) {  // padded storage: node plane 0 is the Dirichlet face, held at 0 (K, RHS, pencil mode 0)
    gk.zpad = 1;
    gk.dmask = 4;
    gz.zpad = 1;
  }
  cudaStream_t s = h->s;
  const long long vec = (long long)D.nrhs * c * gxy.n;
  int maxb = blocks_needed_max(gxy);
  maxb = std::max(maxb, blocks_needed_max(gz));
  maxb = std::max(maxb, blocks_needed_max(gk));
  auto al = [&](void** p, size_t bytes) -> cudaError_t { return cudaMallocAsync(p, bytes ? bytes : 8, s); };
  cudaError_t e = cudaSuccess;
  if ((e = al((void**)&h->r, vec * 8)) || (e = al((void**)&h->d, vec * 8)) || (e = al((void**)&h->p, vec * 8)) ||
      (e = al((void**)&h->u, vec * 8)) || (e = al((void**)&h->spec, (size_t)D.nrhs * c * gxy.nspec * 16)) ||
      (e = al((void**)&h->pencil, (size_t)D.nrhs * c * gz.nspec * 16)) ||
      (e = al((void**)&h->gtab, (size_t)gz.C * gz.nspec * 8)) || (e = al((void**)&h->twx, base.M * 16)) ||
      (e = al((void**)&h->twxp, (base.M + 1) * 16)) || (e = al((void**)&h->twy, N2 * 16)) ||
      (e = al((void**)&h->twz, N3 * 16)) || (e = al((void**)&h->twz2, 2 * N3 * 16)) ||
      (e = al((void**)&h->st, kMaxRhs * sizeof(LoadState))) ||
      (e = al((void**)&h->partials, (size_t)RED_NSLOT * kMaxRhs * maxb * 8)) ||
      (e = al((void**)&h->counters, RED_NSLOT * kMaxRhs * sizeof(unsigned))) ||
      (e = al((void**)&h->results, RED_NSLOT * kMaxRhs * 8)) ||
      (e = al((void**)&h->scratch, (size_t)(2 * 148 * 4 + 64) * 8)) ||
      (e = cudaMallocHost((void**)&h->h_st, kMaxRhs * sizeof(LoadState)))) {
    free_slab(h);
    return sfail(UNO_ERR_CUDA, std::string("slab allocation: ") + cudaGetErrorString(e));
  }
  cudaMemsetAsync(h->counters, 0, RED_NSLOT * kMaxRhs * sizeof(unsigned), s);
  cudaMemsetAsync(h->st, 0, kMaxRhs * sizeof(LoadState), s);
  std::vector<double2> t;
  auto up = [&](double2* dst, int L, int denom) {
    twid(L, denom, t);
    cudaMemcpyAsync(dst, t.data(), (size_t)L * 16, cudaMemcpyHostToDevice, s);
    cudaStreamSynchronize(s);
  };
  up(h->twx, base.M, base.M);
  up(h->twxp, base.M + 1, N1);
  up(h->twy, N2, N2);
  up(h->twz, N3, N3);
  up(h->twz2, 2 * N3, 2 * N3);
  // contexts
  auto mk = [&](const Geo& g, double2* spec) {
    Ctx cx;
    std::memset(&cx, 0, sizeof(cx));
    cx.g = g;
    cx.tw.x = h->twx;
    cx.tw.xpost = h->twxp;
    cx.tw.y = h->twy;
    cx.tw.z = h->twz;
    cx.tw.z2 = h->twz2;
    cx.st = h->st;
    cx.sc.partials = h->partials;
    cx.sc.counters = h->counters;
    cx.sc.results = h->results;
    cx.sc.max_blocks = maxb;
    cx.phase = h->phase;
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 2; ++b) cx.mat[a][b] = D.mat[a][b];
    cx.gtab = h->gtab;
    cx.spec = spec;
    cx.r = h->r;
    cx.d = h->d;
    cx.p = h->p;
    cx.u = h->u;
    return cx;
  };
  h->cxy = mk(gxy, h->spec);
  h->cz = mk(gz, h->pencil);
  h->ck = mk(gk, h->spec);
  // a0 on the pencil: reference medium, symbol, Eq 55
  h->ref0 = D.ref[0] > 0 ? D.ref[0] : 0.5 * (D.mat[0][0] + D.mat[1][0]);
  h->ref1 = D.ref[0] > 0 ? D.ref[1] : 0.5 * (D.mat[0][1] + D.mat[1][1]);
  launch_build_symbol(h->cz, h->gtab, h->ref0, h->ref1, D.seed, D.seed ? D.amp : 0.0, s);
  int nblk = 0;
  launch_eq55(h->cz, h->gtab, h->scratch, &nblk, s);
  std::vector<double> mm(2 * nblk);
  cudaMemcpyAsync(mm.data(), h->scratch, 2 * nblk * 8, cudaMemcpyDeviceToHost, s);
  e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) {
    free_slab(h);
    return sfail(UNO_ERR_CUDA, std::string("slab create: ") + cudaGetErrorString(e));
  }
  double lo = 1e300;
  for (int i = 0; i < nblk; ++i) lo = std::min(lo, mm[i]);
  if (!(lo > 1e-14)) {
    free_slab(h);
    return sfail(UNO_ERR_NOT_SPD, "Eq 55 safety check failed on this rank's pencil");
  }
  *out = h;
  return UNO_OK;
}

extern "C" uno_status uno_slab_destroy(uno_slab_handle* h) {
  if (!h) return sfail(UNO_ERR_ARG, "null handle");
  cudaStreamSynchronize(h->s);
  free_slab(h);
  return UNO_OK;
}

extern "C" uno_status uno_slab_set_stream(uno_slab_handle* h, void* stream) {
  if (!h) return sfail(UNO_ERR_ARG, "null handle");
  h->s = (cudaStream_t)stream;
  h->desc.stream = stream;
  return UNO_OK;
}

extern "C" uno_status uno_slab_sizes(uno_slab_handle* h, int64_t out[4]) {
  if (!h || !out) return sfail(UNO_ERR_ARG, "null argument");
  const Geo& g = h->gxy;
  out[0] = (int64_t)g.nrhs * g.c * g.n;
  out[1] = (int64_t)g.nrhs * g.c * g.H1 * h->Z * h->Yc;
  out[2] = (int64_t)g.nrhs * g.c * g.N1 * g.N2;
  out[3] = h->Z;
  return UNO_OK;
}

extern "C" uno_status uno_slab_begin(uno_slab_handle* h, const double* h_loads, double rel_tol, int32_t max_iter,
                                     int32_t fixed_iters) {
  if (!h || !h_loads) return sfail(UNO_ERR_ARG, "null argument");
  if (!(rel_tol >= 0) || max_iter < 0) return sfail(UNO_ERR_ARG, "rel_tol >= 0, max_iter >= 0 required");
  const Geo& g = h->gk;
  const int nv = g.c == 1 ? 3 : 6;
  LoadParams lp;
  std::memset(&lp, 0, sizeof(lp));
  for (int l = 0; l < g.nrhs; ++l)
    for (int j = 0; j < nv; ++j) lp.v[l][j] = h_loads[l * nv + j];
  SKL(launch_rhs(h->ck, lp, h->r, h->s));  // a1 on this slab's nodes
  SKL(launch_zero(h->u, (long long)g.nrhs * g.c * g.n, h->s));
  const uno_cg_desc& D = h->desc;
  const double mod = g.c == 1 ? std::max(std::fabs(D.mat[0][0]), std::fabs(D.mat[1][0]))
                              : std::max(D.mat[0][0] + 2 * D.mat[0][1], D.mat[1][0] + 2 * D.mat[1][1]);
  for (int l = 0; l < g.nrhs; ++l) {
    LoadState& st = h->h_st[l];
    std::memset(&st, 0, sizeof(st));
    st.active = 1;
    st.rel_tol = rel_tol;
    st.fixed_iters = fixed_iters;
    st.max_iter = max_iter;
    st.gamma1 = 1.0;
    double lm = 0;
    for (int j = 0; j < nv; ++j) lm = std::max(lm, std::fabs(h_loads[l * nv + j]));
    st.zero_floor = 1e-13 * mod * g.h * g.h * lm;  // reading R7 (3D: h^(d-1) = h^2)
  }
  SCK(cudaMemcpyAsync(h->st, h->h_st, g.nrhs * sizeof(LoadState), cudaMemcpyHostToDevice, h->s));
  SCK(cudaStreamSynchronize(h->s));
  return UNO_OK;
}

extern "C" uno_status uno_slab_forward(uno_slab_handle* h, double* d_send) {
  if (!h || !d_send) return sfail(UNO_ERR_ARG, "null argument");
  SKL(launch_xfwd(h->cxy, CG, h->r, h->s));
  SKL(launch_ypass(h->cxy, CG, false, h->s));
  const Geo& g = h->gxy;
  const long long rows = (long long)g.nrhs * g.c * g.H1 * h->Z;
  slab_pack_kernel<<<pack_grid(rows, h->Yc, h->nranks), pack_threads(h->Yc), 0, h->s>>>(
      h->spec, reinterpret_cast<double2*>(d_send), rows, h->Yc, g.N2);
  SCK(cudaGetLastError());
  return UNO_OK;
}

static bool fill_peers(const uno_slab_handle* h, double* const* hp, SlabPeers& P) {
  if (!hp || h->nranks > kMaxRanks) return false;
  for (int q = 0; q < kMaxRanks; ++q) P.p[q] = nullptr;
  for (int q = 0; q < h->nranks; ++q) {
    if (!hp[q]) return false;
    P.p[q] = reinterpret_cast<double2*>(hp[q]);
  }
  return true;
}

extern "C" uno_status uno_slab_forward_peer(uno_slab_handle* h, double* const* h_peer_recv) {
  SlabPeers P;
  if (!h) return sfail(UNO_ERR_ARG, "null handle");
  if (!fill_peers(h, h_peer_recv, P)) return sfail(UNO_ERR_NCCL, "peer receive-buffer table incomplete");
  SKL(launch_xfwd(h->cxy, CG, h->r, h->s));
  const Geo& g = h->gxy;
  const long long rows = (long long)g.nrhs * g.c * g.H1 * h->Z;
  if (g.N2 == 256 || g.N2 == 512) {  // the y pass itself stores every bin into its owner's receive buffer
    Ctx cp = h->cxy;
    for (int q = 0; q < 8; ++q) cp.peer[q] = P.p[q];
    cp.peer_off = (long long)h->rank * rows * h->Yc;
    cp.peer_yc = h->Yc;
    SKL(launch_ypass_peer(cp, h->s));
  } else {
    SKL(launch_ypass(h->cxy, CG, false, h->s));
    slab_pack_peer_kernel<<<pack_grid(rows, h->Yc, h->nranks), pack_threads(h->Yc), 0, h->s>>>(h->spec, P, h->rank,
                                                                                               rows, h->Yc, g.N2);
  }
  SCK(cudaGetLastError());
  return UNO_OK;
}

extern "C" uno_status uno_slab_green_peer(uno_slab_handle* h, const double* d_recv, double* const* h_peer_recv) {
  SlabPeers P;
  if (!h || !d_recv) return sfail(UNO_ERR_ARG, "null argument");
  if (!fill_peers(h, h_peer_recv, P)) return sfail(UNO_ERR_NCCL, "peer receive-buffer table incomplete");
  const Geo& g = h->gxy;
  const long long nlckx = (long long)g.nrhs * g.c * g.H1;
  const dim3 gb(1, (unsigned)std::min<long long>(nlckx, 4096), h->nranks);
  slab_pencil_kernel<<<gb, 256, 0, h->s>>>(const_cast<double2*>(reinterpret_cast<const double2*>(d_recv)), h->pencil,
                                          nlckx, h->Z, h->Yc, h->gz.N3, 0);
  // the z pass itself stores every plane into its owner's receive buffer where the tiled z pass
  // is the production kernel (config 4: 512^3 elastic); otherwise G pass + peer pack
  Ctx cp = h->cz;
  for (int q = 0; q < 8; ++q) cp.peer[q] = P.p[q];
  cp.peer_rank = h->rank;
  cp.peer_z = h->Z;
  cp.peer_nlckx = nlckx;
  if (h->gz.zpad) {
    SKL(launch_pencil_dst_green(h->cz, h->pencil, CG, h->s));
    slab_pencil_peer_kernel<<<gb, 256, 0, h->s>>>(P, h->rank, h->pencil, nlckx, h->Z, h->Yc, h->gz.N3);
  } else if (launch_gpass_peer(cp, h->s) < 0) {
    SKL(launch_gpass(h->cz, CG, h->s));
    slab_pencil_peer_kernel<<<gb, 256, 0, h->s>>>(P, h->rank, h->pencil, nlckx, h->Z, h->Yc, h->gz.N3);
  }
  SCK(cudaGetLastError());
  return UNO_OK;
}

extern "C" uno_status uno_slab_green(uno_slab_handle* h, const double* d_recv, double* d_send) {
  if (!h || !d_recv || !d_send) return sfail(UNO_ERR_ARG, "null argument");
  const Geo& g = h->gxy;
  const long long nlckx = (long long)g.nrhs * g.c * g.H1;
  const dim3 gb(1, (unsigned)std::min<long long>(nlckx, 4096), h->nranks);
  slab_pencil_kernel<<<gb, 256, 0, h->s>>>(const_cast<double2*>(reinterpret_cast<const double2*>(d_recv)), h->pencil,
                                          nlckx, h->Z, h->Yc, h->gz.N3, 0);
  if (h->gz.zpad)
    SKL(launch_pencil_dst_green(h->cz, h->pencil, CG, h->s));  // Dirichlet z: DST-I . G . DST-I
  else
    SKL(launch_gpass(h->cz, CG, h->s));
  slab_pencil_kernel<<<gb, 256, 0, h->s>>>(reinterpret_cast<double2*>(d_send), h->pencil, nlckx, h->Z, h->Yc, h->gz.N3,
                                          1);
  SCK(cudaGetLastError());
  return UNO_OK;
}

extern "C" uno_status uno_slab_inverse(uno_slab_handle* h, const double* d_recv, double* d_halo_send) {
  if (!h || !d_recv || !d_halo_send) return sfail(UNO_ERR_ARG, "null argument");
  const Geo& g = h->gxy;
  const long long rows = (long long)g.nrhs * g.c * g.H1 * h->Z;
  slab_unpack_kernel<<<pack_grid(rows, h->Yc, h->nranks), pack_threads(h->Yc), 0, h->s>>>(
      reinterpret_cast<const double2*>(d_recv), h->spec, rows, h->Yc, g.N2);
  SKL(launch_ypass(h->cxy, CG, true, h->s));
  SKL(launch_xinv(h->cxy, CG, nullptr, h->s));
  const long long plane = (long long)g.N1 * g.N2;
  const int nlc = g.nrhs * g.c;
  slab_halo_kernel<<<grid_for(2LL * nlc * plane), 256, 0, h->s>>>(h->d, d_halo_send, nlc, h->Z, plane);
  SCK(cudaGetLastError());
  return UNO_OK;
}

extern "C" uno_status uno_slab_inverse_peer(uno_slab_handle* h, const double* d_recv, double* const* h_peer_halo_recv) {
  if (!h || !d_recv) return sfail(UNO_ERR_ARG, "null argument");
  if (!h_peer_halo_recv || h->nranks > kMaxRanks) return sfail(UNO_ERR_NCCL, "peer halo table missing / > 8 ranks");
  const int n = h->nranks, lo = (h->rank + n - 1) % n, hi = (h->rank + 1) % n;
  if (!h_peer_halo_recv[lo] || !h_peer_halo_recv[hi]) return sfail(UNO_ERR_NCCL, "null peer halo pointer");
  const Geo& g = h->gxy;
  const long long rows = (long long)g.nrhs * g.c * g.H1 * h->Z;
  slab_unpack_kernel<<<pack_grid(rows, h->Yc, h->nranks), pack_threads(h->Yc), 0, h->s>>>(
      reinterpret_cast<const double2*>(d_recv), h->spec, rows, h->Yc, g.N2);
  SKL(launch_ypass(h->cxy, CG, true, h->s));
  SKL(launch_xinv(h->cxy, CG, nullptr, h->s));
  const long long plane = (long long)g.N1 * g.N2;
  const int nlc = g.nrhs * g.c;
  slab_halo_peer_kernel<<<grid_for(2LL * nlc * plane), 256, 0, h->s>>>(h->d, h_peer_halo_recv[lo] + nlc * plane,
                                                                       h_peer_halo_recv[hi], nlc, h->Z, plane);
  SCK(cudaGetLastError());
  return UNO_OK;
}

extern "C" uno_status uno_slab_kapply(uno_slab_handle* h, const double* d_halo_recv) {
  if (!h || !d_halo_recv) return sfail(UNO_ERR_ARG, "null argument");
  const Geo& g = h->gk;
  h->ck.hlo = d_halo_recv;
  h->ck.hhi = d_halo_recv + (long long)g.nrhs * g.c * g.N1 * g.N2;
  SKL(launch_kapply(h->ck, CG, h->d, h->p, h->s));
  return UNO_OK;
}

extern "C" uno_status uno_slab_reduce(uno_slab_handle* h, int32_t slot, double* d_out) {
  if (!h || !d_out || slot < 0 || slot > 2) return sfail(UNO_ERR_ARG, "slot / null");
  const Ctx& cx = slot == UNO_SLAB_RNORM ? h->cxy : (slot == UNO_SLAB_GAMMA ? h->cz : h->ck);
  SKL(launch_scalar(cx, slot, STANDALONE, h->s));  // fixed-order combine of this rank's CTA partials
  SCK(cudaMemcpyAsync(d_out, h->results + slot * kMaxRhs, h->gxy.nrhs * 8, cudaMemcpyDeviceToDevice, h->s));
  return UNO_OK;
}

extern "C" uno_status uno_slab_apply(uno_slab_handle* h, int32_t slot, const double* d_in) {
  if (!h || !d_in || slot < 0 || slot > 2) return sfail(UNO_ERR_ARG, "slot / null");
  slab_apply_kernel<<<1, 32, 0, h->s>>>(h->st, h->gxy.nrhs, slot, d_in);
  SCK(cudaGetLastError());
  return UNO_OK;
}

extern "C" uno_status uno_slab_state(uno_slab_handle* h, int32_t* any_active, uno_cg_report* rep) {
  if (!h) return sfail(UNO_ERR_ARG, "null handle");
  const int nrhs = h->gxy.nrhs;
  SCK(cudaMemcpyAsync(h->h_st, h->st, nrhs * sizeof(LoadState), cudaMemcpyDeviceToHost, h->s));
  SCK(cudaStreamSynchronize(h->s));
  int any = 0;
  for (int l = 0; l < nrhs; ++l) {
    const LoadState& st = h->h_st[l];
    any |= st.active;
    if (rep) {
      rep[l].iterations = st.iters;
      rep[l].converged = st.converged;
      rep[l].status = st.status;
      rep[l].pad_ = 0;
      rep[l].r0_inf = st.r0;
      rep[l].rel_res = st.r0 > 0 ? st.rn / st.r0 : 0.0;
      rep[l].gamma_last = st.gamma1;
    }
  }
  if (any_active) *any_active = any;
  return UNO_OK;
}

extern "C" uno_status uno_slab_finish(uno_slab_handle* h, double* d_u) {
  if (!h || !d_u) return sfail(UNO_ERR_ARG, "null argument");
  SKL(launch_finalize(h->cxy, h->s));  // the deferred u += alpha d of the last iteration
  const Geo& g = h->gxy;
  SCK(cudaMemcpyAsync(d_u, h->u, (size_t)g.nrhs * g.c * g.n * 8, cudaMemcpyDeviceToDevice, h->s));
  return UNO_OK;
}

extern "C" uno_status uno_slab_local_means(uno_slab_handle* h, const double* d_u, double* d_means) {
  if (!h || !d_u || !d_means) return sfail(UNO_ERR_ARG, "null argument");
  const Geo& g = h->gxy;
  slab_means_kernel<<<g.nrhs * g.c, 1024, 0, h->s>>>(d_u, g.n, d_means);
  SCK(cudaGetLastError());
  return UNO_OK;
}

extern "C" uno_status uno_slab_subtract_means(uno_slab_handle* h, double* d_u, const double* d_means) {
  if (!h || !d_u || !d_means) return sfail(UNO_ERR_ARG, "null argument");
  const Geo& g = h->gxy;
  slab_subtract_kernel<<<dim3(grid_for(g.n), g.nrhs * g.c), 256, 0, h->s>>>(d_u, g.n, d_means, 1.0 / h->nranks);
  SCK(cudaGetLastError());
  return UNO_OK;
}
