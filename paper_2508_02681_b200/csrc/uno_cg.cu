// uno_cg.cu — C ABI of libunocg.so (see include/uno_cg.h for the contract).
//
// Host-side orchestration only: validation, workspace, twiddle tables, element
// matrices, CUDA-graph capture of the PCG iteration and report read-back.  Every
// arithmetic step of the hot path runs in kernels.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include "../../include/uno_cg.h"
#include "common.cuh"
#include "kernels.cuh"
#include <nvtx3/nvToolsExt.h>  // header-only: ranges are no-ops unless a profiler (nsys) is attached

using namespace uno;

static thread_local std::string g_err;

static uno_status fail(uno_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

namespace uno {
uno_status set_last_error(uno_status s, const char* msg) {  // shared with slab.cu
  g_err = msg;
  return s;
}
}  // namespace uno

#define CK(call)                                                                                  \
  do {                                                                                            \
    cudaError_t e_ = (call);                                                                      \
    if (e_ != cudaSuccess) return fail(UNO_ERR_CUDA, std::string(#call ": ") + cudaGetErrorString(e_)); \
  } while (0)

enum { KC_K = 0, KC_XF = 1, KC_Y = 2, KC_G = 3, KC_XI = 4, KC_OTHER = 5, KC_N = 6 };


// NVTX range around each public call (visible in an nsys / ncu --nvtx timeline)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

struct uno_cg_handle {
  uno_cg_desc desc;
  Geo g;
  cudaStream_t stream;
  const uint8_t* phase;
  double ref0, ref1;
  // device buffers
  double *r, *d, *p, *u;
  double* d2;             // second direction buffer of the paired u updates (null: not used)
  double2* spec;
  double* gtab;
  double* kel;
  double2 *twx, *twxp, *twy, *twz, *twz2;
  double2 *twx2, *twy2;    // all-Dirichlet: length-2N1 / 2N2 tables of the odd-extension FFTs
  double* rt;             // all-Dirichlet / 2D mixed: intermediate vector [nrhs][c][n]
  char* arena;            // device workspace (uno_cg_workspace_size bytes), see ws_layout
  bool own_arena;         // allocated by the library (else borrowed from the caller)
  LoadState* st;
  double* partials;
  unsigned* counters;
  double* results;
  double* scratch;        // mean removal / effective / eq55
  size_t scratch_len;
  double* hist;
  int hist_stride;
  LoadState* h_st;        // pinned
  double* h_small;        // pinned scratch for results
  Ctx cx;
  // graph of one chunk of iterations
  cudaGraphExec_t gexec;
  int gchunk;
  bool gtimed;
  int gcap;               // safety cap of the device-side WHILE loop (body executions)
  int* loopctr;           // device counter used by the loop-control kernel
  // timing
  bool timing;
  std::vector<cudaEvent_t> tev;  // per chunk: [iter][class][2]
  double kms[KC_N];
  long long kcnt[KC_N];   // timed launches per class
  long long lcnt[KC_N];   // all launches per class
  double last_ms;
  long long last_launches;
  cudaEvent_t e0, e1;
  double lam_min, lam_max;
  // preconditioner kind (0 UNO, 1 identity, 2 Jacobi) and the Jacobi inverse diagonal [n]
  int precond;
  double* dinv;
  double2* tspec;  // training: spectrum of r while s is transformed (train.cu)
};

// ------------------------------------------------------------------------------ helpers
static void twiddles(int L, int denom, std::vector<double2>& out) {
  out.resize(L);
  for (int m = 0; m < L; ++m) {
    long double a = -2.0L * 3.14159265358979323846264338327950288L * (long double)m / (long double)denom;
    out[m].x = (double)cosl(a);
    out[m].y = (double)sinl(a);
  }
}

// Q1 element matrices by 2-point Gauss quadrature (independent of oracle/): corner a = ax + 2ay + 4az,
// dof (a, alpha) -> c*a + alpha; Mandel-free form: K_lam = int (div N)(div N)^T,
// K_mu = int (grad N : grad N + grad N : grad N^T)  (D = lam I(x)I + 2 mu I^s, Eq 80).
static void elastic_element(int d, double h, std::vector<double>& Kl, std::vector<double>& Km) {
  const int nc = 1 << d, nd = d * nc;
  Kl.assign(nd * nd, 0.0);
  Km.assign(nd * nd, 0.0);
  const double gp[2] = {0.5 - 0.5 / std::sqrt(3.0), 0.5 + 0.5 / std::sqrt(3.0)};
  const double w = std::pow(h, d) / (double)(1 << d);
  const int nq = 1 << d;
  for (int q = 0; q < nq; ++q) {
    double xi[3] = {gp[q & 1], gp[(q >> 1) & 1], gp[(q >> 2) & 1]};
    double G[8][3];
    for (int a = 0; a < nc; ++a) {
      for (int i = 0; i < d; ++i) {
        double v = (((a >> i) & 1) ? 1.0 : -1.0) / h;
        for (int j = 0; j < d; ++j)
          if (j != i) v *= ((a >> j) & 1) ? xi[j] : 1.0 - xi[j];
        G[a][i] = v;
      }
    }
    for (int a = 0; a < nc; ++a)
      for (int al = 0; al < d; ++al)
        for (int b = 0; b < nc; ++b)
          for (int be = 0; be < d; ++be) {
            const int r = d * a + al, s = d * b + be;
            Kl[r * nd + s] += w * G[a][al] * G[b][be];
            double gg = 0.0;
            for (int j = 0; j < d; ++j) gg += G[a][j] * G[b][j];
            Km[r * nd + s] += w * ((al == be ? gg : 0.0) + G[a][be] * G[b][al]);
          }
  }
}

static bool is_pow2(int v) { return v > 0 && (v & (v - 1)) == 0; }
static bool g_pool_cfg[64];  // default memory pool configured, per device ordinal

static Ctx make_ctx(uno_cg_handle* h) {
  Ctx cx;
  std::memset(&cx, 0, sizeof(cx));
  cx.g = h->g;
  cx.tw.x = h->twx;
  cx.tw.xpost = h->twxp;
  cx.tw.y = h->twy;
  cx.tw.z = h->twz;
  cx.tw.z2 = h->twz2;
  cx.st = h->st;
  cx.sc.partials = h->partials;
  cx.sc.counters = h->counters;
  cx.sc.results = h->results;
  cx.sc.max_blocks = blocks_needed_max(h->g);
  cx.phase = h->phase;
  for (int a = 0; a < 2; ++a)
    for (int b = 0; b < 2; ++b) cx.mat[a][b] = h->desc.mat[a][b];
  cx.gtab = h->gtab;
  cx.kel = h->kel;
  cx.spec = h->spec;
  cx.d2 = h->precond == 0 ? h->d2 : nullptr;  // the baseline preconditioners keep one buffer
  cx.r = h->r;
  cx.d = h->d;
  cx.p = h->p;
  cx.u = h->u;
  cx.hist = h->hist;
  cx.hist_stride = h->hist_stride;
  return cx;
}

static void free_all(uno_cg_handle* h) {
  if (!h) return;
  if (h->gexec) cudaGraphExecDestroy(h->gexec);
  for (auto e : h->tev) cudaEventDestroy(e);
  if (h->arena && h->own_arena) cudaFreeAsync(h->arena, h->stream);
  void* bufs[] = {h->tspec, h->hist, h->dinv};  // allocated on demand, outside the workspace
  for (void* b : bufs)
    if (b) cudaFreeAsync(b, h->stream);
  if (h->h_st) cudaFreeHost(h->h_st);
  if (h->h_small) cudaFreeHost(h->h_small);
  if (h->e0) cudaEventDestroy(h->e0);
  if (h->e1) cudaEventDestroy(h->e1);
  delete h;
}

#define KL(expr, cls)                                                                 \
  do {                                                                                \
    int n_ = (expr);                                                                  \
    if (n_ < 0) return fail(UNO_ERR_SHAPE, "no kernel instance for this grid size"); \
    h->lcnt[cls] += n_;                                                               \
    launches += n_;                                                                   \
  } while (0)

// a0: element matrices (elastic), tabulated G_hat(k)/n and the Eq 55 check.
static uno_status setup_problem(uno_cg_handle* h) {
  const uno_cg_desc& D = h->desc;
  const Geo& g = h->g;
  const int c = g.c;
  cudaStream_t s = h->stream;
  cudaError_t e;
  if (D.ref[0] > 0) {
    h->ref0 = D.ref[0];
    h->ref1 = D.ref[1];
  } else {  // arithmetic mean of the phases
    h->ref0 = 0.5 * (D.mat[0][0] + D.mat[1][0]);
    h->ref1 = 0.5 * (D.mat[0][1] + D.mat[1][1]);
  }
  if (h->gexec) {  // materials are kernel parameters: re-capture on the next solve
    cudaGraphExecDestroy(h->gexec);
    h->gexec = nullptr;
  }
  if (c > 1) {
    std::vector<double> Kl, Km, Kp;
    elastic_element(g.dim, g.h, Kl, Km);
    const size_t nn = Kl.size();
    Kp.resize(2 * nn);
    for (int ph = 0; ph < 2; ++ph)
      for (size_t i = 0; i < nn; ++i) Kp[ph * nn + i] = D.mat[ph][0] * Kl[i] + D.mat[ph][1] * Km[i];
    cudaMemcpyAsync(h->kel, Kp.data(), Kp.size() * 8, cudaMemcpyHostToDevice, s);
    cudaStreamSynchronize(s);
  }
  h->cx = make_ctx(h);
  if (h->precond == 2 && h->dinv) launch_jacobi_dinv(h->cx, h->dinv, s);  // Eq 25 for the new problem
  // a0: symbol table + Eq 55 check
  if (g.dmask)
    launch_d3_symbol(h->cx, h->gtab, h->ref0, h->ref1, D.seed, D.seed ? D.amp : 0.0, s);
  else
    launch_build_symbol(h->cx, h->gtab, h->ref0, h->ref1, D.seed, D.seed ? D.amp : 0.0, s);
  int nblk = 0;
  launch_eq55(h->cx, h->gtab, h->scratch, &nblk, s);
  std::vector<double> mm(2 * nblk);
  cudaMemcpyAsync(mm.data(), h->scratch, 2 * nblk * 8, cudaMemcpyDeviceToHost, s);
  e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return fail(UNO_ERR_CUDA, std::string("create: ") + cudaGetErrorString(e));
  double lo = 1e300, hi = -1e300;
  for (int i = 0; i < nblk; ++i) {
    lo = std::min(lo, mm[i]);
    hi = std::max(hi, mm[nblk + i]);
  }
  h->lam_min = lo;
  h->lam_max = hi;
  if (!(lo > 1e-14)) {  // Eq 55
    char buf[160];
    std::snprintf(buf, sizeof buf, "Eq 55 safety check failed: min block eigenvalue %.3e", lo);
    return fail(UNO_ERR_NOT_SPD, buf);
  }
  return UNO_OK;
}

// Validate a descriptor and derive the handle's geometry (shared by uno_cg_workspace_size and
// uno_cg_create, so both see the same grid).
static uno_status make_geo(const uno_cg_desc& D, Geo& g) {
  if (D.dim != 2 && D.dim != 3) return fail(UNO_ERR_ARG, "dim must be 2 or 3");
  if (D.physics != UNO_THERMAL && D.physics != UNO_ELASTIC) return fail(UNO_ERR_ARG, "physics must be 0 or 1");
  // boundary conditions: all periodic, or (3D) periodic x, y with Dirichlet z (mixed)
  const bool dirz = D.dim == 3 && D.bc[0] == 0 && D.bc[1] == 0 && D.bc[2] == 1;
  const bool dir3 = D.dim == 3 && D.bc[0] == 1 && D.bc[1] == 1 && D.bc[2] == 1;
  const int dmask2 = D.dim == 2 ? (D.bc[0] ? 1 : 0) | (D.bc[1] ? 2 : 0) : 0;  // 2D: 3 Dirichlet, 2 mixed
  for (int i = 0; i < D.dim; ++i)
    if (D.bc[i] != 0 && !dirz && !dir3 && dmask2 != 3 && dmask2 != 2)
      return fail(UNO_ERR_UNSUPPORTED,
                  "boundary conditions: all periodic, periodic x,y + Dirichlet z, all Dirichlet, or (2D) "
                  "periodic x + Dirichlet y");
  const int N1 = D.n[0], N2 = D.n[1], N3 = D.dim == 3 ? D.n[2] : 1;
  if (!is_pow2(N1) || !is_pow2(N2) || !is_pow2(N3) || N1 < 8 || N2 < 8 || N1 > 1024 || N2 > 1024 ||
      (D.dim == 3 && (N3 < 4 || N3 > 1024)))
    return fail(UNO_ERR_SHAPE, "N1,N2 in {8..1024}, N3 in {4..1024} (3D), powers of two");
  if (D.nrhs < 1 || D.nrhs > kMaxRhs) return fail(UNO_ERR_ARG, "nrhs must be 1..8");
  const int c = D.physics == UNO_THERMAL ? 1 : D.dim;
  if (D.physics == UNO_THERMAL) {
    if (!(D.mat[0][0] > 0) || !(D.mat[1][0] > 0)) return fail(UNO_ERR_ARG, "conductivities must be > 0");
  } else {
    for (int p = 0; p < 2; ++p)
      if (!(D.mat[p][1] > 0) || !(D.mat[p][0] >= 0)) return fail(UNO_ERR_ARG, "need mu > 0, lambda >= 0");
    if (D.dim == 3 && N1 < 16) return fail(UNO_ERR_SHAPE, "elastic 3D needs N1 >= 16");
  }
  if (dirz && ((c == 1 && N1 < 32) || N1 < 16 || N3 < 8 || N3 > 512))
    return fail(UNO_ERR_SHAPE, "mixed BC needs N1 >= 32 (thermal) / 16 (elastic), 8 <= N3 <= 512");
  if (dir3 && ((c == 1 && (N1 < 32 || N2 < 16)) || N1 < 16 || N2 < 16 || N3 < 8 || N1 > 512 || N2 > 512 || N3 > 512))
    return fail(UNO_ERR_SHAPE, "all-Dirichlet needs N1 >= 32 (thermal) / 16 (elastic), N2 >= 16, N3 >= 8, all <= 512");
  if (dmask2 && (N1 < 16 || N2 < 16 || N1 > 512 || N2 > 512))
    return fail(UNO_ERR_SHAPE, "2D Dirichlet / mixed needs 16 <= N1, N2 <= 512");
  if (D.seed != 0 && !(D.amp >= 0 && D.amp < 1)) return fail(UNO_ERR_ARG, "amp must be in [0, 1)");
  std::memset(&g, 0, sizeof(g));
  g.dim = D.dim;
  g.c = c;
  g.nrhs = D.nrhs;
  g.N1 = N1;
  g.N2 = N2;
  g.N3 = N3;
  g.M = N1 / 2;
  g.H1 = g.M + 1;
  g.dirz = dirz ? 1 : 0;
  g.dir3 = dir3 ? 1 : 0;
  g.dmask = dir3 ? 7 : dmask2;
  g.P3 = dirz ? N3 - 1 : N3;
  g.n = (long long)N1 * N2 * g.P3;
  // all-Dirichlet: real sine coefficients on the node grid; 2D mixed: R2C half spectrum along x
  g.nspec = (dir3 || dmask2 == 3) ? g.n : (long long)g.H1 * N2 * g.P3;
  g.h = D.h > 0 ? D.h : 1.0 / N1;
  g.C = c * (c + 1) / 2;
  // z planes per K CTA: 32, halved (down to 4) while the K grid is under two waves of 2 CTAs per
  // SM (small grids such as configs 1 and 2 would otherwise leave most SMs idle)
  g.KZC = g.N3 < 32 ? g.N3 : 32;
  if (g.dim == 3) {
    const long long per = c == 1 ? (long long)std::max(1, N1 / 32) * std::max(1, N2 / 16)
                                 : (long long)std::max(1, N1 / 16) * std::max(1, N2 / 8);
    auto kblocks = [&](int zc) { return per * ((g.P3 + zc - 1) / zc) * g.nrhs; };
    while (g.KZC > 4 && kblocks(g.KZC) < 2LL * 148 * 2) g.KZC /= 2;
  }
  return UNO_OK;
}

// Device workspace of a handle: every buffer the library owns, carved from one arena (caller-
// provided or allocated here) at 256-byte aligned offsets.  Order = WS_* below.
enum { WS_R, WS_D, WS_P, WS_U, WS_SPEC, WS_GTAB, WS_KEL, WS_TWX, WS_TWXP, WS_TWY, WS_TWZ, WS_TWZ2, WS_RT, WS_TWX2,
       WS_TWY2, WS_ST, WS_PARTS, WS_CNT, WS_RES, WS_SCR, WS_LOOP, WS_D2, WS_N };

// Paired u updates (kernels.cuh Ctx::d2): 3D whole-grid handles with the UNO preconditioner (set per
// handle), periodic or Dirichlet-z storage; the x^-1 passes (xinv_kernel, xinv512_kernel) and the
// 3D K kernels follow the two direction buffers.
#ifndef UNO_PAIRED_U
#define UNO_PAIRED_U 1  // 0: one direction buffer, u updated every iteration (A/B builds only)
#endif
static bool paired_u_ok(const Geo& g) { return UNO_PAIRED_U && g.dim == 3 && !g.dmask && !g.halo; }

static size_t scratch_doubles(const Geo& g) {
  return (size_t)std::max<long long>((long long)(kMaxRhs * kMaxRhs + 1) * (148 * 4 + 1) * 2 + 64,
                                     (long long)g.nrhs * g.c * 148 * 2 + g.nrhs * g.c + 64);
}

static size_t ws_layout(const Geo& g, size_t off[WS_N]) {
  const size_t vec = (size_t)g.nrhs * g.c * g.n * 8;
  const size_t sz[WS_N] = {
      vec, vec, vec, vec, (size_t)g.nrhs * g.c * g.nspec * 16, (size_t)g.C * g.nspec * 8, 2 * 576 * 8,
      (size_t)g.M * 16, (size_t)(g.M + 1) * 16, (size_t)g.N2 * 16, (size_t)g.N3 * 16, (size_t)2 * g.N3 * 16,
      g.dmask ? vec : 8, g.dmask ? (size_t)2 * g.N1 * 16 : 16, g.dmask ? (size_t)2 * g.N2 * 16 : 16,
      kMaxRhs * sizeof(LoadState), (size_t)RED_NSLOT * kMaxRhs * blocks_needed_max(g) * 8,
      RED_NSLOT * kMaxRhs * sizeof(unsigned), RED_NSLOT * kMaxRhs * 8, scratch_doubles(g) * 8, 64,
      paired_u_ok(g) ? vec : 8};
  size_t t = 0;
  for (int i = 0; i < WS_N; ++i) {
    if (off) off[i] = t;
    t += (sz[i] + 255) & ~(size_t)255;
  }
  return t;
}

extern "C" uno_status uno_cg_workspace_size(const uno_cg_desc* desc, size_t* bytes) {
  if (!desc || !bytes) return fail(UNO_ERR_ARG, "null argument");
  Geo g;
  const uno_status st = make_geo(*desc, g);
  if (st != UNO_OK) return st;
  *bytes = ws_layout(g, nullptr);
  return UNO_OK;
}

// ------------------------------------------------------------------------------ create/destroy
extern "C" uno_status uno_cg_create(const uno_cg_desc* desc, const uint8_t* d_phase, void* d_workspace,
                                    uno_cg_handle** out) {
  NvtxRange nvtx_("uno_cg_create");
  if (!desc || !d_phase || !out) return fail(UNO_ERR_ARG, "null argument");
  *out = nullptr;
  if (((uintptr_t)d_workspace & 255) != 0) return fail(UNO_ERR_ARG, "d_workspace must be 256-byte aligned");
  const uno_cg_desc& D = *desc;
  Geo g0;
  const uno_status gs = make_geo(D, g0);
  if (gs != UNO_OK) return gs;

  uno_cg_handle* h = new uno_cg_handle();  // value-initialised: all members zero
  h->desc = D;
  h->stream = (cudaStream_t)D.stream;
  h->phase = d_phase;
  h->g = g0;
  const Geo& g = h->g;
  cudaStream_t s = h->stream;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && !g_pool_cfg[dev]) {  // keep freed pool memory cached on this device
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = ~0ULL;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    g_pool_cfg[dev] = true;
  }
  size_t off[WS_N];
  const size_t total = ws_layout(g, off);
  h->scratch_len = scratch_doubles(g);
  h->hist_stride = 0;
  cudaError_t e = cudaSuccess;
  if (d_workspace) {
    h->arena = (char*)d_workspace;
    h->own_arena = false;
  } else if ((e = cudaMallocAsync((void**)&h->arena, total, s)) != cudaSuccess) {
    h->arena = nullptr;
    free_all(h);
    return fail(UNO_ERR_CUDA, std::string("workspace allocation: ") + cudaGetErrorString(e));
  } else {
    h->own_arena = true;
  }
  char* A = h->arena;
  h->r = (double*)(A + off[WS_R]);
  h->d = (double*)(A + off[WS_D]);
  h->p = (double*)(A + off[WS_P]);
  h->u = (double*)(A + off[WS_U]);
  h->spec = (double2*)(A + off[WS_SPEC]);
  h->gtab = (double*)(A + off[WS_GTAB]);
  h->kel = (double*)(A + off[WS_KEL]);
  h->twx = (double2*)(A + off[WS_TWX]);
  h->twxp = (double2*)(A + off[WS_TWXP]);
  h->twy = (double2*)(A + off[WS_TWY]);
  h->twz = (double2*)(A + off[WS_TWZ]);
  h->twz2 = (double2*)(A + off[WS_TWZ2]);
  h->rt = (double*)(A + off[WS_RT]);
  h->twx2 = (double2*)(A + off[WS_TWX2]);
  h->twy2 = (double2*)(A + off[WS_TWY2]);
  h->st = (LoadState*)(A + off[WS_ST]);
  h->partials = (double*)(A + off[WS_PARTS]);
  h->counters = (unsigned*)(A + off[WS_CNT]);
  h->results = (double*)(A + off[WS_RES]);
  h->scratch = (double*)(A + off[WS_SCR]);
  h->loopctr = (int*)(A + off[WS_LOOP]);
  h->d2 = paired_u_ok(g) ? (double*)(A + off[WS_D2]) : nullptr;
  if ((e = cudaMallocHost((void**)&h->h_st, kMaxRhs * sizeof(LoadState))) ||
      (e = cudaMallocHost((void**)&h->h_small, 4096 * 8)) || (e = cudaEventCreate(&h->e0)) ||
      (e = cudaEventCreate(&h->e1))) {
    free_all(h);
    return fail(UNO_ERR_CUDA, std::string("allocation: ") + cudaGetErrorString(e));
  }
  cudaMemsetAsync(h->counters, 0, RED_NSLOT * kMaxRhs * sizeof(unsigned), s);
  cudaMemsetAsync(h->st, 0, kMaxRhs * sizeof(LoadState), s);
  cudaMemsetAsync(h->loopctr, 0, 64, s);
  // twiddles (long double on the host)
  const int N1 = g.N1, N2 = g.N2, N3 = g.N3;
  std::vector<double2> t;
  auto up = [&](double2* dst, int L, int denom) {
    twiddles(L, denom, t);
    cudaMemcpyAsync(dst, t.data(), (size_t)L * 16, cudaMemcpyHostToDevice, s);
    cudaStreamSynchronize(s);
  };
  up(h->twx, g.M, g.M);
  up(h->twxp, g.M + 1, N1);
  up(h->twy, N2, N2);
  up(h->twz, N3, N3);
  up(h->twz2, 2 * N3, 2 * N3);
  if (g.dmask) {
    up(h->twx2, 2 * N1, 2 * N1);
    up(h->twy2, 2 * N2, 2 * N2);
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) {
    free_all(h);
    return fail(UNO_ERR_CUDA, std::string("create: ") + cudaGetErrorString(e));
  }
  const uno_status st0 = setup_problem(h);
  if (st0 != UNO_OK) {
    free_all(h);
    return st0;
  }
  *out = h;
  return UNO_OK;
}

extern "C" uno_status uno_cg_destroy(uno_cg_handle* h) {
  if (!h) return fail(UNO_ERR_ARG, "null handle");
  cudaStreamSynchronize(h->stream);
  free_all(h);
  return UNO_OK;
}

extern "C" uno_status uno_cg_update(uno_cg_handle* h, const uno_cg_desc* desc, const uint8_t* d_phase) {
  NvtxRange nvtx_("uno_cg_update");
  if (!h || !desc || !d_phase) return fail(UNO_ERR_ARG, "null argument");
  const uno_cg_desc& D = *desc;
  const uno_cg_desc& O = h->desc;
  if (D.dim != O.dim || D.physics != O.physics || D.nrhs != O.nrhs || D.n[0] != O.n[0] || D.n[1] != O.n[1] ||
      (D.dim == 3 && D.n[2] != O.n[2]) || D.h != O.h)
    return fail(UNO_ERR_ARG, "update: grid, physics, h and nrhs must match the handle");
  for (int i = 0; i < D.dim; ++i)
    if (D.bc[i] != O.bc[i]) return fail(UNO_ERR_ARG, "update: boundary conditions must match the handle");
  if (D.physics == UNO_THERMAL) {
    if (!(D.mat[0][0] > 0) || !(D.mat[1][0] > 0)) return fail(UNO_ERR_ARG, "conductivities must be > 0");
  } else {
    for (int p = 0; p < 2; ++p)
      if (!(D.mat[p][1] > 0) || !(D.mat[p][0] >= 0)) return fail(UNO_ERR_ARG, "need mu > 0, lambda >= 0");
  }
  if (D.seed != 0 && !(D.amp >= 0 && D.amp < 1)) return fail(UNO_ERR_ARG, "amp must be in [0, 1)");
  void* keep_stream = O.stream;
  h->desc = D;
  h->desc.stream = keep_stream;  // the handle stays on its creation stream
  h->phase = d_phase;
  return setup_problem(h);
}

extern "C" uno_status uno_cg_set_preconditioner(uno_cg_handle* h, int32_t kind) {
  if (!h) return fail(UNO_ERR_ARG, "null handle");
  if (kind < UNO_PRECOND_UNO || kind > UNO_PRECOND_JACOBI) return fail(UNO_ERR_ARG, "kind must be 0, 1 or 2");
  if (kind == UNO_PRECOND_JACOBI && !h->dinv) CK(cudaMallocAsync((void**)&h->dinv, (size_t)h->g.n * 8, h->stream));
  h->precond = kind;
  h->cx = make_ctx(h);  // the paired u updates apply to the UNO preconditioner only
  if (kind == UNO_PRECOND_JACOBI) launch_jacobi_dinv(h->cx, h->dinv, h->stream);
  if (h->gexec) {  // the iteration body changes: re-capture on the next solve
    cudaGraphExecDestroy(h->gexec);
    h->gexec = nullptr;
  }
  CK(cudaGetLastError());
  return UNO_OK;
}

// ------------------------------------------------------------------------------ training (Alg 4)
static uno_status train_check(const uno_cg_handle* h) {
  const Geo& g = h->g;
  if (g.dim != 3 || g.dirz || g.dmask)
    return fail(UNO_ERR_UNSUPPORTED, "training: 3D periodic grids with the 5-pass transforms");
  return UNO_OK;
}

extern "C" uno_status uno_cg_train_features(uno_cg_handle* h, const double* d_r, const double* d_s, double scale,
                                            double* d_feat) {
  if (!h || !d_r || !d_s || !d_feat) return fail(UNO_ERR_ARG, "null argument");
  uno_status st = train_check(h);
  if (st != UNO_OK) return st;
  const Geo& g = h->g;
  cudaStream_t s = h->stream;
  long long launches = 0;
  if (!h->tspec) CK(cudaMallocAsync((void**)&h->tspec, (size_t)g.nrhs * g.c * g.nspec * 16, s));
  auto fwd = [&](const double* x) -> uno_status {  // r_hat = T x (unnormalised: x, y, z passes)
    KL(launch_xfwd(h->cx, STANDALONE, x, s), KC_XF);
    KL(launch_ypass(h->cx, STANDALONE, false, s), KC_Y);
    KL(launch_gpass(h->cx, FWDZ, s), KC_G);
    return UNO_OK;
  };
  if ((st = fwd(d_r)) != UNO_OK) return st;
  CK(cudaMemcpyAsync(h->tspec, h->spec, (size_t)g.nrhs * g.c * g.nspec * 16, cudaMemcpyDeviceToDevice, s));
  if ((st = fwd(d_s)) != UNO_OK) return st;
  // unitary T = FFT / sqrt(n): products of two transforms carry 1/n
  KL(launch_train_feat(h->cx, h->tspec, h->spec, scale / (double)g.n, d_feat, s), KC_OTHER);
  CK(cudaGetLastError());
  return UNO_OK;
}

extern "C" uno_status uno_cg_train_pairs(uno_cg_handle* h, int32_t M, int64_t* npair, int32_t* h_bins) {
  if (!h || !npair) return fail(UNO_ERR_ARG, "null argument");
  uno_status st = train_check(h);
  if (st != UNO_OK) return st;
  if (M < 0) return fail(UNO_ERR_ARG, "M >= 0");
  std::vector<int> pbin, binpair;
  train_build_pairs(h->g, M, pbin, binpair);
  *npair = (int64_t)(pbin.size() / 2);
  if (h_bins) std::memcpy(h_bins, pbin.data(), pbin.size() * 4);
  return UNO_OK;
}

extern "C" uno_status uno_cg_train_newton(uno_cg_handle* h, const double* d_feat, int32_t M, int32_t epochs,
                                          double* h_theta0, double* d_thetas, double* h_loss) {
  if (!h || !d_feat || !h_theta0 || epochs < 0) return fail(UNO_ERR_ARG, "null argument / epochs");
  uno_status st = train_check(h);
  if (st != UNO_OK) return st;
  std::vector<int> pbin, binpair;
  train_build_pairs(h->g, M, pbin, binpair);
  if (!d_thetas && !pbin.empty()) return fail(UNO_ERR_ARG, "d_thetas required when K is not empty");
  std::string err;
  if (train_newton_run(h->cx, d_feat, pbin, binpair, epochs, h_theta0, d_thetas, h_loss, h->stream, err) < 0)
    return fail(UNO_ERR_CUDA, "training: " + err);
  return UNO_OK;
}

extern "C" uno_status uno_cg_train_install(uno_cg_handle* h, int32_t M, const double* h_theta0, const double* d_thetas) {
  if (!h || !h_theta0) return fail(UNO_ERR_ARG, "null argument");
  uno_status st = train_check(h);
  if (st != UNO_OK) return st;
  std::vector<int> pbin, binpair;
  train_build_pairs(h->g, M, pbin, binpair);
  if (train_install_run(h->cx, pbin, binpair, h_theta0, d_thetas, h->gtab, h->stream) < 0)
    return fail(UNO_ERR_CUDA, "training install");
  if (h->gexec) {
    cudaGraphExecDestroy(h->gexec);
    h->gexec = nullptr;
  }
  int nblk = 0;  // Eq 55 on the learned symbol; psi makes it SPD by construction
  launch_eq55(h->cx, h->gtab, h->scratch, &nblk, h->stream);
  std::vector<double> mm(2 * nblk);
  CK(cudaMemcpyAsync(mm.data(), h->scratch, 2 * nblk * 8, cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  double lo = 1e300;
  for (int i = 0; i < nblk; ++i) lo = std::min(lo, mm[i]);
  if (!(lo > 1e-14)) return fail(UNO_ERR_NOT_SPD, "Eq 55 safety check failed on the trained symbol");
  return UNO_OK;
}

static void fill_loads(const uno_cg_handle* h, const double* h_loads, LoadParams& lp) {
  std::memset(&lp, 0, sizeof(lp));
  const int nv = h->g.c == 1 ? h->g.dim : (h->g.dim == 3 ? 6 : 3);
  for (int l = 0; l < h->g.nrhs; ++l)
    for (int j = 0; j < nv; ++j) lp.v[l][j] = h_loads[l * nv + j];
}

extern "C" uno_status uno_cg_rhs(uno_cg_handle* h, const double* h_loads, double* d_f) {
  NvtxRange nvtx_("uno_cg_rhs");
  if (!h || !h_loads || !d_f) return fail(UNO_ERR_ARG, "null argument");
  LoadParams lp;
  fill_loads(h, h_loads, lp);
  launch_rhs(h->cx, lp, d_f, h->stream);
  CK(cudaGetLastError());
  return UNO_OK;
}

extern "C" uno_status uno_cg_apply_K(uno_cg_handle* h, const double* d_u, double* d_Au, double* h_uAu) {
  NvtxRange nvtx_("uno_cg_apply_K");
  if (!h || !d_u || !d_Au) return fail(UNO_ERR_ARG, "null argument");
  if (d_u == d_Au) return fail(UNO_ERR_ARG, "apply_K: input and output must not alias");
  long long launches = 0;
  KL(launch_kapply(h->cx, STANDALONE, d_u, d_Au, h->stream), KC_K);
  KL(launch_scalar(h->cx, RED_DP, STANDALONE, h->stream), KC_OTHER);
  CK(cudaGetLastError());
  if (h_uAu) {
    CK(cudaMemcpyAsync(h->h_small, h->results + RED_DP * kMaxRhs, h->g.nrhs * 8, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    for (int l = 0; l < h->g.nrhs; ++l) h_uAu[l] = h->h_small[l];
  }
  return UNO_OK;
}

extern "C" uno_status uno_cg_apply_precond(uno_cg_handle* h, const double* d_r, double* d_z, double* h_rz) {
  NvtxRange nvtx_("uno_cg_apply_precond");
  if (!h || !d_r || !d_z) return fail(UNO_ERR_ARG, "null argument");
  long long launches = 0;
  cudaStream_t s = h->stream;
  if (h->precond != 0) {  // z = P r (identity / Jacobi) and r.z
    KL(launch_jac_r(h->cx, h->precond, STANDALONE, h->dinv, d_r, d_z, s), KC_XF);
    KL(launch_scalar_n(h->cx, RED_GAMMA, STANDALONE, jacobi_nblk(h->g), s), KC_OTHER);
  } else if (h->g.dmask) {  // all-Dirichlet / 2D mixed: DST-I axes (dirichlet.cu)
    const double2* tw2[3] = {h->twx2, h->twy2, h->twz2};
    KL(launch_d3_precond(h->cx, d_r, d_z, tw2, s), KC_G);
    KL(launch_d3_dot(h->cx, d_r, d_z, STANDALONE, s), KC_OTHER);
    KL(launch_scalar_n(h->cx, RED_GAMMA, STANDALONE, jacobi_nblk(h->g), s), KC_OTHER);
  } else {  // periodic, or mixed BC (Dirichlet z: the z DST-I . G . DST-I stage on the spectrum)
    KL(launch_xfwd(h->cx, STANDALONE, d_r, s), KC_XF);
    if (h->g.dim == 3) KL(launch_ypass(h->cx, STANDALONE, false, s), KC_Y);
    if (h->g.dirz)
      KL(launch_pencil_dst_green(h->cx, h->spec, STANDALONE, s), KC_G);
    else
      KL(launch_gpass(h->cx, STANDALONE, s), KC_G);
    if (h->g.dim == 3) KL(launch_ypass(h->cx, STANDALONE, true, s), KC_Y);
    KL(launch_xinv(h->cx, STANDALONE, d_z, s), KC_XI);
    KL(launch_scalar(h->cx, RED_GAMMA, STANDALONE, s), KC_OTHER);
  }
  CK(cudaGetLastError());
  if (h_rz) {
    CK(cudaMemcpyAsync(h->h_small, h->results + RED_GAMMA * kMaxRhs, h->g.nrhs * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    for (int l = 0; l < h->g.nrhs; ++l) h_rz[l] = h->h_small[l];
  }
  return UNO_OK;
}

// one PCG iteration (Alg 2 body) as kernel launches.  When `ev` is given, an event pair
// brackets every launch: slots 0..5 = xfwd, yfwd, gpass, yinv, xinv, K.
static const int kSlotClass[6] = {KC_XF, KC_Y, KC_G, KC_Y, KC_XI, KC_K};
static int enqueue_iteration(uno_cg_handle* h, cudaStream_t s, cudaEvent_t* ev /* [6][2] or null */) {
  const Ctx& cx = h->cx;
  int n = 0;
  auto run = [&](int slot, auto&& launch) -> bool {
    // external event-record nodes (plain cudaEventRecord under capture is graph-internal)
    if (ev) cudaEventRecordWithFlags(ev[2 * slot], s, cudaEventRecordExternal);
    const int r = launch();
    if (ev) cudaEventRecordWithFlags(ev[2 * slot + 1], s, cudaEventRecordExternal);
    if (r < 0) return false;
    n += r;
    return true;
  };
  if (h->precond != 0) {  // baselines (precond.cu): r pass | scalars | d pass, then K
    const int nb = jacobi_nblk(h->g);
    if (!run(0, [&] { return launch_jac_r(cx, h->precond, CG, h->dinv, nullptr, nullptr, s); })) return -1;
    n += launch_scalar_n(cx, RED_RNORM, CG, nb, s);
    n += launch_scalar_n(cx, RED_GAMMA, CG, nb, s);
    if (!run(4, [&] { return launch_jac_d(cx, h->precond, h->dinv, s); })) return -1;
  } else if (h->g.dmask) {  // all-Dirichlet / 2D mixed: r pass | s = P r | r.s | d pass
    const int nb = jacobi_nblk(h->g);
    const double2* tw2[3] = {h->twx2, h->twy2, h->twz2};
    if (!run(0, [&] { return launch_jac_r(cx, 1, CG, nullptr, nullptr, nullptr, s); })) return -1;
    n += launch_scalar_n(cx, RED_RNORM, CG, nb, s);
    if (!run(2, [&] { return launch_d3_precond(cx, cx.r, h->rt, tw2, s); })) return -1;
    n += launch_d3_dot(cx, cx.r, h->rt, CG, s);
    n += launch_scalar_n(cx, RED_GAMMA, CG, nb, s);
    if (!run(4, [&] { return launch_jac_d_ext(cx, h->rt, s); })) return -1;
  } else {  // 5-pass: x | y | z.G.z^-1 (mixed BC: DST_z . G . DST_z on the spectrum) | y^-1 | x^-1, K
    const bool d3 = h->g.dim == 3;
    if (!run(0, [&] { return launch_xfwd(cx, CG, cx.r, s); })) return -1;
    n += launch_scalar(cx, RED_RNORM, CG, s);
    if (d3 && !run(1, [&] { return launch_ypass(cx, CG, false, s); })) return -1;
    if (!run(2, [&] { return h->g.dirz ? launch_pencil_dst_green(cx, cx.spec, CG, s) : launch_gpass(cx, CG, s); }))
      return -1;
    n += launch_scalar(cx, RED_GAMMA, CG, s);
    if (d3 && !run(3, [&] { return launch_ypass(cx, CG, true, s); })) return -1;
    if (!run(4, [&] { return launch_xinv(cx, CG, nullptr, s); })) return -1;
  }
  if (!run(5, [&] { return launch_kapply(cx, CG, cx.d, cx.p, s); })) return -1;
  n += launch_scalar(cx, RED_DP, CG, s);
  return n;
}

// The solve loop as one CUDA graph.  Untimed: a WHILE conditional node whose body holds
// `chunk` PCG iterations plus the loop-control kernel, so the whole solve runs device-side
// with a single host launch.  Timed: `chunk` iterations bracketed by event-record nodes,
// relaunched from the host (events inside a device loop could not be read per iteration).
static uno_status build_graph(uno_cg_handle* h, int chunk, bool timed, int cap) {
  if (h->gexec && h->gchunk == chunk && h->gtimed == timed && h->gcap == cap) return UNO_OK;
  if (h->gexec) {
    cudaGraphExecDestroy(h->gexec);
    h->gexec = nullptr;
  }
  if (timed) {
    const size_t need = (size_t)chunk * 6 * 2;
    while (h->tev.size() < need) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      h->tev.push_back(e);
    }
  }
  cudaStream_t cs;
  CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  cudaGraph_t graph;
  if (timed) {
    CK(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
    for (int i = 0; i < chunk; ++i) {
      if (enqueue_iteration(h, cs, &h->tev[(size_t)i * 6 * 2]) < 0) {
        cudaStreamEndCapture(cs, &graph);
        cudaStreamDestroy(cs);
        return fail(UNO_ERR_SHAPE, "no kernel instance for this grid size");
      }
    }
    CK(cudaStreamEndCapture(cs, &graph));
  } else {
    CK(cudaGraphCreate(&graph, 0));
    cudaGraphConditionalHandle ch;
    CK(cudaGraphConditionalHandleCreate(&ch, graph, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = ch;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t node;
    CK(cudaGraphAddNode(&node, graph, nullptr, 0, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    CK(cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    for (int i = 0; i < chunk; ++i) {
      if (enqueue_iteration(h, cs, nullptr) < 0) {
        cudaStreamEndCapture(cs, &body);
        cudaStreamDestroy(cs);
        cudaGraphDestroy(graph);
        return fail(UNO_ERR_SHAPE, "no kernel instance for this grid size");
      }
    }
    launch_loop_ctl(ch, h->st, h->g.nrhs, h->loopctr, cap, cs);
    CK(cudaStreamEndCapture(cs, &body));
  }
  CK(cudaGraphInstantiate(&h->gexec, graph, 0));
  cudaGraphDestroy(graph);
  cudaStreamDestroy(cs);
  h->gchunk = chunk;
  h->gtimed = timed;
  h->gcap = cap;
  return UNO_OK;
}

static double zero_floor(const uno_cg_handle* h, const double* load, int nv) {
  double mod;
  if (h->g.c == 1)
    mod = std::max(std::fabs(h->desc.mat[0][0]), std::fabs(h->desc.mat[1][0]));
  else
    mod = std::max(h->desc.mat[0][0] + 2 * h->desc.mat[0][1], h->desc.mat[1][0] + 2 * h->desc.mat[1][1]);
  double lm = 0;
  for (int j = 0; j < nv; ++j) lm = std::max(lm, std::fabs(load[j]));
  return 1e-13 * mod * std::pow(h->g.h, h->g.dim - 1) * lm;
}

extern "C" uno_status uno_cg_solve(uno_cg_handle* h, const double* h_loads, double rel_tol, int32_t max_iter,
                                   int32_t fixed_iters, double* d_u, uno_cg_report* rep, double* h_hist) {
  NvtxRange nvtx_("uno_cg_solve");
  if (!h || !h_loads || !d_u) return fail(UNO_ERR_ARG, "null argument");
  if (!(rel_tol >= 0) || max_iter < 0) return fail(UNO_ERR_ARG, "rel_tol >= 0, max_iter >= 0 required");
  const Geo& g = h->g;
  cudaStream_t s = h->stream;
  long long launches = 0;
  const int cap = fixed_iters > 0 ? fixed_iters : max_iter;
  // per-iteration record: residual history, gamma_1, alpha (planes of kMaxRhs x (cap + 1))
  if (h->hist_stride < cap + 1) {
    if (h->hist) cudaFreeAsync(h->hist, s);
    h->hist = nullptr;
    CK(cudaMallocAsync(&h->hist, (size_t)3 * kMaxRhs * (cap + 1) * 8, s));
    h->hist_stride = cap + 1;
    h->cx = make_ctx(h);
    if (h->gexec) {
      cudaGraphExecDestroy(h->gexec);
      h->gexec = nullptr;
    }
  }
  const int nv = g.c == 1 ? g.dim : (g.dim == 3 ? 6 : 3);
  LoadParams lp;
  fill_loads(h, h_loads, lp);
  CK(cudaEventRecord(h->e0, s));
  // a1: r = f ; u = 0 ; d = 0 (first F5 overwrites)
  KL(launch_rhs(h->cx, lp, h->r, s), KC_OTHER);
  KL(launch_zero(h->u, (long long)g.nrhs * g.c * g.n, s), KC_OTHER);
  for (int l = 0; l < g.nrhs; ++l) {
    LoadState& st = h->h_st[l];
    std::memset(&st, 0, sizeof(st));
    st.active = 1;
    st.rel_tol = rel_tol;
    st.fixed_iters = fixed_iters;
    st.max_iter = max_iter;
    st.gamma1 = 1.0;
    st.zero_floor = zero_floor(h, h_loads + l * nv, nv);
  }
  CK(cudaMemcpyAsync(h->st, h->h_st, g.nrhs * sizeof(LoadState), cudaMemcpyHostToDevice, s));
  const long long work = (long long)g.nrhs * g.c * g.n;
  // passes + 3 scalar kernels (mixed: 6 too)
  const int per_iter = h->precond != 0 ? 6 : g.dmask ? 15 : (g.dim == 3 ? (g.dirz ? 8 : 6) : 4) + 3;
  if (!h->timing && h->precond == 0 && tiny_supported(g)) {
    // small 2D grid (config 0): the whole of Alg 2 in one persistent CTA per load (tiny.cu)
    KL(launch_tiny_pcg(h->cx, s), KC_OTHER);
  } else if (!h->timing) {
    // whole solve device-side: WHILE node over bodies of `chunk` iterations
    const int chunk = work >= (1LL << 22) ? 2 : 4;
    const int cap_body = (cap + 1 + chunk - 1) / chunk + 1;
    uno_status bs = build_graph(h, chunk, false, cap_body);
    if (bs != UNO_OK) return bs;
    CK(cudaGraphLaunch(h->gexec, s));
    CK(cudaMemcpyAsync(h->h_st, h->st, g.nrhs * sizeof(LoadState), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    int it = 0;
    for (int l = 0; l < g.nrhs; ++l) it = std::max(it, h->h_st[l].iters);
    launches += (long long)(it / chunk + 1) * (chunk * per_iter + 1);  // bodies executed (>= iters/chunk)
  } else {
    const int chunk = work >= (1LL << 22) ? 4 : (work >= (1LL << 18) ? 8 : 16);
    uno_status bs = build_graph(h, chunk, true, 0);
    if (bs != UNO_OK) return bs;
    int done = 0;
    bool any = true;
    while (any) {
      if (done > cap + 1) break;  // safety: the device stops itself at cap
      CK(cudaGraphLaunch(h->gexec, s));
      launches += (long long)chunk * per_iter;
      int before = 0;
      for (int l = 0; l < g.nrhs; ++l) before = std::max(before, h->h_st[l].iters);
      CK(cudaMemcpyAsync(h->h_st, h->st, g.nrhs * sizeof(LoadState), cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      done += chunk;
      any = false;
      int after = 0;
      for (int l = 0; l < g.nrhs; ++l) {
        any = any || h->h_st[l].active;
        after = std::max(after, h->h_st[l].iters);
      }
      const int worked = std::min(chunk, std::max(0, after - before));
      for (int i = 0; i < worked; ++i)
        for (int slot = 0; slot < 6; ++slot) {
          if (g.dim == 2 && (slot == 1 || slot == 3)) continue;
          float ms = 0.f;
          if (cudaEventElapsedTime(&ms, h->tev[((size_t)i * 6 + slot) * 2], h->tev[((size_t)i * 6 + slot) * 2 + 1]) ==
              cudaSuccess) {
            h->kms[kSlotClass[slot]] += ms;
            h->kcnt[kSlotClass[slot]] += 1;
          } else {
            (void)cudaGetLastError();  // clear the non-sticky error of a failed query
          }
        }
    }
  }
  KL(launch_finalize(h->cx, s), KC_OTHER);
  if (g.dirz || g.dmask)  // Dirichlet faces: no null space, the fluctuation is not mean-free
    CK(cudaMemcpyAsync(d_u, h->u, (size_t)g.nrhs * g.c * g.n * 8, cudaMemcpyDeviceToDevice, s));
  else
    KL(launch_mean_removal(h->cx, h->u, d_u, h->scratch, s), KC_OTHER);
  CK(cudaEventRecord(h->e1, s));
  CK(cudaMemcpyAsync(h->h_st, h->st, g.nrhs * sizeof(LoadState), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  CK(cudaGetLastError());
  float ms = 0.f;
  cudaEventElapsedTime(&ms, h->e0, h->e1);
  h->last_ms = ms;
  h->last_launches = launches;
  uno_status worst = UNO_OK;
  for (int l = 0; l < g.nrhs; ++l) {
    const LoadState& st = h->h_st[l];
    if (rep) {
      rep[l].iterations = st.iters;
      rep[l].converged = st.converged;
      rep[l].status = st.status;
      rep[l].pad_ = 0;
      rep[l].r0_inf = st.r0;
      rep[l].rel_res = st.r0 > 0 ? st.rn / st.r0 : 0.0;
      rep[l].gamma_last = st.gamma1;
    }
    if (st.status != 0 && worst == UNO_OK) worst = (uno_status)st.status;
  }
  if (h_hist && h->hist) {  // rows of this solve's cap + 1 entries (the device stride may be longer)
    CK(cudaMemcpy2DAsync(h_hist, (size_t)(cap + 1) * 8, h->hist, (size_t)h->hist_stride * 8, (size_t)(cap + 1) * 8,
                         g.nrhs, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
  }
  if (worst != UNO_OK) return fail(worst, "PCG breakdown or non-finite residual (see per-load report)");
  return UNO_OK;
}

extern "C" uno_status uno_cg_effective_property(uno_cg_handle* h, const double* d_u, const double* h_loads,
                                                double* h_out) {
  NvtxRange nvtx_("uno_cg_effective_property");
  if (!h || !d_u || !h_loads || !h_out) return fail(UNO_ERR_ARG, "null argument");
  const Geo& g = h->g;
  LoadParams lp;
  fill_loads(h, h_loads, lp);
  int nblk = 0;
  launch_effective(h->cx, lp, d_u, h->scratch, &nblk, h->stream);
  const int nl = g.nrhs, nacc = nl * nl + 1;
  CK(cudaMemcpyAsync(h->h_small, h->scratch + (long long)nacc * nblk, nacc * 8, cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  CK(cudaGetLastError());
  const double nvox = (double)g.N1 * g.N2 * g.N3;
  const double vf = h->h_small[nl * nl] / nvox;
  const double vol = nvox * std::pow(g.h, g.dim);
  const int nv = g.c == 1 ? g.dim : (g.dim == 3 ? 6 : 3);
  for (int i = 0; i < nl; ++i)
    for (int j = 0; j < nl; ++j) {
      double base;
      const double* li = h_loads + i * nv;
      const double* lj = h_loads + j * nv;
      if (g.c == 1) {
        const double km = (1 - vf) * h->desc.mat[0][0] + vf * h->desc.mat[1][0];
        double dot = 0;
        for (int k = 0; k < nv; ++k) dot += li[k] * lj[k];
        base = km * dot;
      } else {  // B_i : <D> : B_j  with D = lam m m^T + 2 mu I (Mandel)
        const double lam = (1 - vf) * h->desc.mat[0][0] + vf * h->desc.mat[1][0];
        const double mu = (1 - vf) * h->desc.mat[0][1] + vf * h->desc.mat[1][1];
        double tri = 0, trj = 0, dot = 0;
        for (int k = 0; k < g.dim; ++k) {
          tri += li[k];
          trj += lj[k];
        }
        for (int k = 0; k < nv; ++k) dot += li[k] * lj[k];
        base = lam * tri * trj + 2 * mu * dot;
      }
      h_out[i * nl + j] = base - h->h_small[i * nl + j] / vol;
    }
  return UNO_OK;
}

// ------------------------------------------------------------------ PCG coefficients / spectrum
static uno_status read_coefficients(uno_cg_handle* h, int load, std::vector<double>& gam, std::vector<double>& alp) {
  const int m = h->hist ? std::min(h->h_st[load].iters, h->hist_stride) : 0;
  gam.assign(m, 0.0);
  alp.assign(m, 0.0);
  if (m > 0) {
    CK(cudaMemcpyAsync(gam.data(), h->hist + ((long long)1 * kMaxRhs + load) * h->hist_stride, (size_t)m * 8,
                       cudaMemcpyDeviceToHost, h->stream));
    CK(cudaMemcpyAsync(alp.data(), h->hist + ((long long)2 * kMaxRhs + load) * h->hist_stride, (size_t)m * 8,
                       cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
  }
  return UNO_OK;
}

extern "C" uno_status uno_cg_last_coefficients(uno_cg_handle* h, int32_t load, int32_t cap, double* h_gamma,
                                               double* h_alpha, int32_t* m_out) {
  if (!h || !m_out || load < 0 || load >= h->g.nrhs || cap < 0 || (cap > 0 && (!h_gamma || !h_alpha)))
    return fail(UNO_ERR_ARG, "null pointer, load out of range or cap < 0");
  std::vector<double> gam, alp;
  const uno_status e = read_coefficients(h, load, gam, alp);
  if (e != UNO_OK) return e;
  *m_out = (int32_t)gam.size();
  for (int i = 0; i < (int)gam.size() && i < cap; ++i) {
    h_gamma[i] = gam[i];
    h_alpha[i] = alp[i];
  }
  return UNO_OK;
}

// number of eigenvalues of the symmetric tridiagonal (d, e) below x (Sturm sequence of the LDL^T
// pivots; a zero pivot is replaced by -pivmin)
static int sturm_count(const std::vector<double>& d, const std::vector<double>& e, double x, double pivmin) {
  int c = 0;
  double q = 1.0;
  for (size_t i = 0; i < d.size(); ++i) {
    q = (d[i] - x) - (i > 0 ? e[i - 1] * e[i - 1] / q : 0.0);
    if (std::fabs(q) < pivmin) q = -pivmin;
    if (q < 0) ++c;
  }
  return c;
}

// k-th smallest eigenvalue (k = 1 .. n) by bisection inside the Gershgorin interval
static double tridiag_eig(const std::vector<double>& d, const std::vector<double>& e, int k) {
  const int n = (int)d.size();
  double lo = d[0], hi = d[0], scale = 0.0;
  for (int i = 0; i < n; ++i) {
    const double r = (i > 0 ? std::fabs(e[i - 1]) : 0.0) + (i + 1 < n ? std::fabs(e[i]) : 0.0);
    lo = std::min(lo, d[i] - r);
    hi = std::max(hi, d[i] + r);
    scale = std::max(scale, std::fabs(d[i]) + r);
  }
  const double pivmin = std::numeric_limits<double>::min() * std::max(1.0, scale * scale);
  lo -= 1e-15 * scale;
  hi += 1e-15 * scale;
  for (int it = 0; it < 200 && hi - lo > 2e-16 * std::max(std::fabs(lo), std::fabs(hi)); ++it) {
    const double mid = 0.5 * (lo + hi);
    if (sturm_count(d, e, mid, pivmin) >= k) hi = mid;
    else lo = mid;
  }
  return 0.5 * (lo + hi);
}

extern "C" uno_status uno_cg_spectrum(uno_cg_handle* h, int32_t load, double tol, double* h_out, int32_t* m_out) {
  if (!h || !h_out || !m_out || load < 0 || load >= h->g.nrhs || !(tol > 0 && tol < 1))
    return fail(UNO_ERR_ARG, "null pointer, load out of range or tol outside (0, 1)");
  std::vector<double> gam, alp;
  const uno_status e = read_coefficients(h, load, gam, alp);
  if (e != UNO_OK) return e;
  const int m = (int)gam.size();
  *m_out = m;
  if (m == 0) return fail(UNO_ERR_ARG, "no PCG iteration recorded for this load");
  // Lanczos tridiagonal of P A from the CG coefficients
  std::vector<double> d(m), off(m > 1 ? m - 1 : 0);
  for (int j = 0; j < m; ++j) {
    d[j] = 1.0 / alp[j];
    if (j > 0) d[j] += (gam[j] / gam[j - 1]) / alp[j - 1];
    if (j + 1 < m) off[j] = std::sqrt(gam[j + 1] / gam[j]) / alp[j];
  }
  const double lmin = tridiag_eig(d, off, 1), lmax = tridiag_eig(d, off, m);
  const double cond = lmax / lmin;
  const double sq = std::sqrt(cond);
  const double C = (sq - 1.0) / (sq + 1.0);
  h_out[0] = lmin;
  h_out[1] = lmax;
  h_out[2] = cond;
  h_out[3] = C;
  h_out[4] = C > 0 ? std::log(tol / 2.0) / std::log(C) : 1.0;
  return UNO_OK;
}

extern "C" uno_status uno_cg_last_solve_stats(uno_cg_handle* h, double* ms, int64_t* kernel_launches) {
  if (!h) return fail(UNO_ERR_ARG, "null handle");
  if (ms) *ms = h->last_ms;
  if (kernel_launches) *kernel_launches = h->last_launches;
  return UNO_OK;
}

extern "C" uno_status uno_cg_kernel_timing(uno_cg_handle* h, int32_t enable, int32_t reset, double* ms6,
                                           int64_t* count6) {
  if (!h) return fail(UNO_ERR_ARG, "null handle");
  if (reset) {
    for (int i = 0; i < KC_N; ++i) {
      h->kms[i] = 0;
      h->kcnt[i] = 0;
    }
  }
  if (enable >= 0) h->timing = enable != 0;
  if (ms6)
    for (int i = 0; i < KC_N; ++i) ms6[i] = h->kms[i];
  if (count6)
    for (int i = 0; i < KC_N; ++i) count6[i] = h->kcnt[i];
  return UNO_OK;
}

extern "C" const char* uno_cg_last_error(void) { return g_err.c_str(); }
extern "C" const char* uno_cg_version(void) { return "libunocg 0.1 (sm_100a, fp64)"; }
