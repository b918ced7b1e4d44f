// kernels.cuh — host-visible launch interface of the libunocg kernels.
#pragma once
#include <string>
#include <vector>

#include "common.cuh"

namespace uno {

struct Tw {                 // device twiddle tables (host-computed in long double)
  const double2* x;         // length M:   e^{-2 pi i m / M}
  const double2* xpost;     // length M+1: e^{-2 pi i k / N1}
  const double2* y;         // length N2
  const double2* z;         // length N3
  const double2* z2;        // length 2 N3 (DST-I via odd extension, mixed BC)
};

struct Ctx {
  Geo g;
  Tw tw;
  LoadState* st;            // [nrhs] device CG state
  Scratch sc;
  const uint8_t* phase;     // [N3][N2][N1]
  double mat[2][2];         // thermal {k,-}; elastic {lam, mu} per phase
  const double* gtab;       // [C][H1][N3][N2]  G_hat(k)/n, unique entries (Eq 51, B7 order)
  const double* kel;        // elastic: per-phase element matrices [2][(c 2^d)^2] (lam K_lam + mu K_mu)
  double2* spec;            // [nrhs][c][H1][N3][N2]
  double* r;                // [nrhs][c][n]
  double* d;
  double* d2;               // paired u updates: direction j lives in (j & 1) ? d2 : d, and the x^-1
                            // pass adds two terms to u every other iteration (null: one buffer,
                            // u += alpha d_old every iteration)
  double* p;
  double* u;
  double* hist;             // [nrhs][hist_stride] residual history (device) or null
  int hist_stride;
  const double* hlo;        // slab mode (g.halo): node plane zlo-1 of d, [nrhs][c][N2][N1]
  const double* hhi;        // slab mode: node plane zlo+P3 of d
  // slab peer-memory forward (ypass256 PEER instance): bin k of row `row` goes to
  // peer[k / peer_yc] + peer_off + row * peer_yc + k % peer_yc (receivers' a2a buffers)
  double2* peer[8];
  long long peer_off;
  int peer_yc;
  // slab peer-memory green (gpass_z PEER instance): pencil element (lk, z, y) goes to
  // peer[z / peer_z] + ((peer_rank * peer_nlckx + lk) * peer_z + z % peer_z) * N2 + y
  int peer_rank, peer_z;
  long long peer_nlckx;
};

struct LoadParams {         // macroscopic loads for the RHS / effective-property kernels
  double v[kMaxRhs][6];
};

enum Mode { STANDALONE = 0, CG = 1, PLAIN = 2, FWDZ = 3 };  // PLAIN: skips inactive loads, no CG fusions;
                                                           // FWDZ: forward z FFT only (G pass, training)

// pass launchers; return number of kernels launched (or -1 on unsupported size)
// b0/nb: launch only blocks [b0, b0+nb) of 8 x-rows (nb = 0: all) — z-chunks of the pipelined schedule
int launch_xfwd(const Ctx& cx, int mode, const double* src, cudaStream_t s, int b0 = 0, int nb = 0);
int launch_xinv(const Ctx& cx, int mode, double* dst, cudaStream_t s, int b0 = 0, int nb = 0);
// z0/zc: only z in [z0, z0+zc) of every (comp, kx) plane (zc = 0: all; multiples of 8)
int launch_ypass(const Ctx& cx, int mode, bool inverse, cudaStream_t s, int z0 = 0, int zc = 0);
// slab forward y pass storing straight into the peers' receive buffers (N2 = 256 only; -1 otherwise)
int launch_ypass_peer(const Ctx& cx, cudaStream_t s);
// slab green stage storing the z^-1 output straight into the peers' receive buffers (generic
// tiled z pass; -1 where a specialised G pass is the production kernel)
int launch_gpass_peer(const Ctx& cx, cudaStream_t s);
int launch_gpass(const Ctx& cx, int mode, cudaStream_t s);
// persistent elastic G pass at N3 = 512 (gpass512e.cu); same per-tile gamma partials as the tiled z pass
bool gpass512e_supported(const Geo& g);
int gpass512e_nblk(const Geo& g);
int launch_gpass512e(const Ctx& cx, int mode, cudaStream_t s);
// TMA-streamed thermal G pass at N3 = 256 (gpass256t.cu); -1 if the tensor maps cannot be encoded
bool gpass256t_supported(const Geo& g);
int launch_gpass256t(const Ctx& cx, int mode, cudaStream_t s);
int gpass_nblk(const Geo& g);  // CTAs (gamma partials per load) of the CG-mode G pass
// zc0/nzl: 3D thermal only, z-chunks [zc0, zc0+nzl) of g.KZC planes (nzl = 0: all)
int launch_kapply(const Ctx& cx, int mode, const double* src, double* dst, cudaStream_t s, int zc0 = 0, int nzl = 0);
int launch_rhs(const Ctx& cx, const LoadParams& lp, double* f, cudaStream_t s);
int launch_finalize(const Ctx& cx, cudaStream_t s);
// CG-mode direction vector of `load` for the K pass (paired u updates: the buffer of direction iters)
__device__ __forceinline__ const double* cg_dir(const Ctx& cx, int mode, const double* src, int load) {
  return (mode == CG && cx.d2) ? ((cx.st[load].iters & 1) ? cx.d2 : cx.d) : src;
}
int launch_mean_removal(const Ctx& cx, const double* u, double* out, double* scratch_means, cudaStream_t s);
int launch_effective(const Ctx& cx, const LoadParams& lp, const double* u, double* partials, int* nblocks_out,
                     cudaStream_t s);
int launch_build_symbol(const Ctx& cx, double* gtab, double ref0, double ref1, unsigned long long seed, double amp,
                        cudaStream_t s);
int launch_eq55(const Ctx& cx, const double* gtab, double* minmax_partials, int* nblocks_out, cudaStream_t s);
int launch_zero(double* x, long long n, cudaStream_t s);
int launch_loop_ctl(cudaGraphConditionalHandle h, const LoadState* st, int nrhs, int* counter, int cap, cudaStream_t s);

int blocks_needed_max(const Geo& g);
int launch_scalar(const Ctx& cx, int slot, int mode, cudaStream_t s);  // combine partials + CG scalars  // max CTAs per load of any reducing kernel

// Dirichlet z (whole-grid mixed BC, or slab pencils on padded storage Geo::zpad): DST-I . G . DST-I
// on the spectrum in place, 3 launches (dst.cu)
int launch_pencil_dst_green(const Ctx& cx, double2* spec, int mode, cudaStream_t s);
int pencil_gmul_nblk();

// whole Alg 2 in one CTA per load for small 2D periodic thermal grids (tiny.cu)
bool tiny_supported(const Geo& g);
int launch_tiny_pcg(const Ctx& cx, cudaStream_t s);

// elastic K.u in the Walsh-Hadamard modal basis, kp_elastic.cu
int launch_kp_elastic_modal(const Ctx& cx, int mode, const double* src, double* dst, cudaStream_t s);
int kp_elastic_modal_nblk(const Geo& g);

// baseline preconditioners P = I / Jacobi (Eq 25), precond.cu; kind 1 = identity, 2 = Jacobi
int launch_jacobi_dinv(const Ctx& cx, double* dinv, cudaStream_t s);
int launch_jac_r(const Ctx& cx, int kind, int mode, const double* dinv, const double* src, double* z, cudaStream_t s);
int launch_jac_d(const Ctx& cx, int kind, const double* dinv, cudaStream_t s);
int jacobi_nblk(const Geo& g);
int launch_scalar_n(const Ctx& cx, int slot, int mode, int nblk, cudaStream_t s);  // explicit partial count

// all-Dirichlet (dirichlet.cu): s = P r (DST-I on every axis, 7 passes), r.s partials, symbol
int launch_d3_precond(const Ctx& cx, const double* r, double* sbuf, const double2* const tw2[3], cudaStream_t s);
int launch_d3_dot(const Ctx& cx, const double* a, const double* b, int mode, cudaStream_t s);
int launch_d3_symbol(const Ctx& cx, double* gtab, double ref0, double ref1, unsigned long long seed, double amp,
                     cudaStream_t s);
int launch_jac_d_ext(const Ctx& cx, const double* sbuf, cudaStream_t s);  // d = s + beta d from a buffer

// second-order UNO training (train.cu, Alg 4)
int launch_train_feat(const Ctx& cx, const double2* sr, const double2* ss, double scale, double* feat, cudaStream_t s);
void train_build_pairs(const Geo& g, int M, std::vector<int>& pbin, std::vector<int>& binpair);
int train_newton_run(const Ctx& cx, const double* feat, const std::vector<int>& pbin, const std::vector<int>& binpair,
                     int epochs, double* th0_host, double* d_ths, double* loss_hist, cudaStream_t s, std::string& err);
int train_install_run(const Ctx& cx, const std::vector<int>& pbin, const std::vector<int>& binpair,
                      const double* th0_host, const double* d_ths, double* gtab, cudaStream_t s);

// mixed BC (Dirichlet on z), dst.cu

}  // namespace uno
