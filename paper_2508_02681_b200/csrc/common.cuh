// common.cuh — shared device/host definitions of libunocg (B200, sm_100a).
// Nothing here is shared with oracle/ (the CPU reference); see DESIGN.md.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace uno {

constexpr int kMaxRhs = 8;
constexpr int kTile = 8;  // columns per FFT smem tile (conflict-free with the XOR swizzle)

// Geometry of one handle (periodic grid, cubic voxels).
struct Geo {
  int dim, c, nrhs;
  int N1, N2, N3;       // voxels; N3 = 1 in 2D
  int M, H1;            // M = N1/2 (complex length of the x R2C), H1 = M + 1 half-spectrum planes
  long long n;          // N1*N2*N3 nodes
  long long nspec;      // H1*N2*N3 complex bins per component
  double h;             // voxel edge
  int C;                // unique symbol entries per bin: c(c+1)/2 (Eq 51)
  int dirz;             // 1: Dirichlet on z (mixed BC; DST-I along z), node planes 1..N3-1 stored
  int P3;               // stored node planes along z: N3 (periodic) or N3 - 1 (dirz); 1 in 2D
  int KZC;              // z planes per CTA of the 3D thermal K kernel
  // z-slab decomposition (slab.cu; all 0 for a whole-grid handle):
  int zlo;              // global z of the first stored node plane of this slab
  int halo;             // 1: K reads node planes zlo-1 / zlo+P3 from Ctx::hlo / Ctx::hhi
  int Ny, ky0;          // symbol of a y-chunk pencil: global N2 and the chunk's first k_y (Ny = 0: N2)
  int dir3;             // 1: Dirichlet on every axis (dirichlet.cu): periodic storage, index-0 nodes held at 0
  int dmask;            // Dirichlet axes kept in that padded periodic storage (bit i = axis i): 7 (3D
                        // all-Dirichlet), 3 (2D Dirichlet), 2 (2D mixed: periodic x, Dirichlet y)
  int zpad;             // slab mode, Dirichlet z on padded storage: node plane z = 0 (and sine mode 0
                        // of the pencil) held at 0, planes 1..N3-1 the unknowns (wrap = plane N3 = 0)
};

// Per-load CG state (device resident; Alg 2 scalars).
struct LoadState {
  double alpha;      // alpha of the last K step (alpha_m)
  double gamma0, gamma1, beta;
  double r0, rn, tol_abs, zero_floor;
  double dp;
  int active;        // 1 while iterating
  int iters;         // completed iterations (K applications)
  int status;        // 0 ok, 6 breakdown, 7 nonfinite
  int converged;
  int pending_u;     // u += alpha d still owed (deferred to the x-inverse pass / finalize)
  int fixed_iters, max_iter;
  int u_done;        // paired u updates (Ctx::d2): direction terms 0 .. u_done-1 are in u
  double rel_tol;
  double alpha_prev; // alpha of the K step before the last one (paired u updates)
};

// Reduction slots: one per (kernel class, load).
enum RedSlot { RED_RNORM = 0, RED_GAMMA = 1, RED_DP = 2, RED_AUX = 3, RED_NSLOT = 4 };

struct Scratch {
  double* partials;      // [RED_NSLOT][kMaxRhs][max_blocks]
  unsigned* counters;    // [RED_NSLOT][kMaxRhs]
  double* results;       // [RED_NSLOT][kMaxRhs] (standalone mode results)
  int max_blocks;
};

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
__device__ __forceinline__ double2 mul_mi(double2 a) { return make_double2(a.y, -a.x); }  // -i a
__device__ __forceinline__ double2 mul_pi(double2 a) { return make_double2(-a.y, a.x); }  // +i a

// SplitMix64 counter-based generator — independent device implementation.
__host__ __device__ __forceinline__ uint64_t sm64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ double u01(uint64_t seed, uint64_t stream, uint64_t i) {
  return (double)(sm64(seed ^ sm64(stream ^ sm64(i))) >> 11) * (1.0 / 9007199254740992.0);
}

// ---------------------------------------------------------------------------------------
// Deterministic block + grid reductions.  Each CTA writes its partial; the last CTA to
// finish (atomic ticket) combines all partials in a FIXED order, so the result is
// bitwise independent of CTA scheduling.
// ---------------------------------------------------------------------------------------
template <bool MAX>
__device__ __forceinline__ double red_op(double a, double b) {
  return MAX ? fmax(a, b) : a + b;
}

template <bool MAX>
__device__ double block_reduce(double v, double* sh /* >= 32 doubles */) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = red_op<MAX>(v, __shfl_down_sync(0xffffffffu, v, o));
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double r = MAX ? 0.0 : 0.0;
  if (threadIdx.x == 0) {
    r = sh[0];
    for (int w = 1; w < nw; ++w) r = red_op<MAX>(r, sh[w]);
  }
  return r;  // valid in thread 0
}

// Returns true in exactly one CTA (the last), with *total valid in its thread 0.
template <bool MAX>
__device__ bool grid_reduce(double v, double* partials, unsigned* counter, int nblocks, int my,
                            double* total, double* sh) {
  double b = block_reduce<MAX>(v, sh);
  __shared__ unsigned s_ticket;
  if (threadIdx.x == 0) {
    partials[my] = b;
    __threadfence();
    s_ticket = atomicAdd(counter, 1u);
  }
  __syncthreads();
  if (s_ticket != (unsigned)(nblocks - 1)) return false;
  __threadfence();
  // fixed-order combine: thread t sums partials t, t+T, t+2T, ... then a fixed tree.
  double acc = 0.0;
  for (int i = threadIdx.x; i < nblocks; i += blockDim.x) {
    double pv = *((volatile double*)&partials[i]);
    acc = (i == (int)threadIdx.x) ? pv : red_op<MAX>(acc, pv);
  }
  double t = block_reduce<MAX>(acc, sh);
  if (threadIdx.x == 0) {
    *total = t;
    *counter = 0u;  // re-arm for the next launch
  }
  return true;
}

}  // namespace uno
