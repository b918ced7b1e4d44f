/*
 * uno_cg_slab.h — z-slab decomposition of one UNO-CG problem over several GPUs
 * (SURVEY.md §8(e) "Config 4 (one 512^3 grid): one exchange step per stage").
 *
 * One handle per rank.  Rank r owns the node planes z in [r Z, (r+1) Z), Z = N3 / nranks,
 * of every CG vector (layout [nrhs][c][Z][N2][N1], the whole-grid convention of uno_cg.h
 * restricted to the slab) and the whole phase field.  One PCG iteration (Alg 2,
 * P:518-533) is a fixed sequence of local stages separated by exchanges that the CALLER
 * performs (NCCL / torch.distributed over NVLink, or plain copies when the ranks are
 * emulated in one process); every arithmetic step runs in this library's kernels:
 *
 *   forward   r -= alpha p, ||r||_inf partial, x R2C + y FFT of the slab,
 *             pack the spectrum by destination rank                          (l.11, l.3, l.4)
 *   [all-to-all: slab spectrum (all k_y, own z) -> pencils (own k_y chunk, all z)]
 *   green     z FFT, s_hat = G_hat r_hat (+ Parseval partial of gamma), z^-1, pack back (l.4-7)
 *   [all-to-all back]
 *   inverse   y^-1, x^-1 -> s, d = s + beta d, u += alpha_prev d_old; copy the slab's two
 *             boundary node planes of d to the halo send buffer                (l.6, 8, 12)
 *   [halo exchange: my first plane -> rank-1, my last plane -> rank+1 (periodic in z)]
 *   kapply    p = A d with the neighbours' planes, d.p partial                 (l.9-10)
 *
 * and three scalar reductions per iteration: each rank reduces its per-CTA partials
 * (uno_slab_reduce), the caller all-reduces them across ranks (max for ||r||_inf, sum
 * for gamma and d.p) and hands the totals back (uno_slab_apply), which runs the CG
 * scalar logic (alpha, beta, convergence) identically on every rank.
 *
 * Buffers (all device, caller-owned, sizes from uno_slab_sizes):
 *   a2a send/recv: complex fp64 [nranks][nrhs][c][H1][Z][Yc], Yc = N2 / nranks; block q
 *     of the send buffer goes to rank q, block q of the receive buffer came from rank q.
 *   halo send/recv: fp64 [2][nrhs][c][N2][N1]; send[0] = my first plane (to rank-1),
 *     send[1] = my last plane (to rank+1); recv[0] = plane zlo-1 (from rank-1),
 *     recv[1] = plane zlo+Z (from rank+1).
 * Scope: 3D, thermal (N1 >= 32, N2 >= 16) and elastic (N1 >= 16), the 5-pass transforms;
 * N3 % nranks == 0 and N2 % nranks == 0 with Yc = N2 / nranks >= 8.  Boundary conditions:
 * periodic, or the mixed case of Eq 82 / §6.4 (bc = {0,0,1}: periodic x, y, Dirichlet faces on
 * z, U = F_x F_y DST-I_z).  Dirichlet z uses PADDED slab storage: the vectors keep
 * N3 node planes, plane z = 0 is the fixed Dirichlet face (held at 0 on input and output; rank
 * 0's first plane), planes 1..N3-1 are the unknowns (the whole-grid handle stores only those
 * N3-1), so the slabs stay equal; the pencil stage applies the z DST-I after the all-to-all.
 * Errors as in uno_cg.h (uno_cg_last_error()).
 */
#ifndef UNO_CG_SLAB_H
#define UNO_CG_SLAB_H

#include "uno_cg.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct uno_slab_handle uno_slab_handle; /* opaque */

enum { UNO_SLAB_RNORM = 0, UNO_SLAB_GAMMA = 1, UNO_SLAB_DP = 2 };

/* desc describes the WHOLE grid (n = global N1, N2, N3); d_phase is the whole phase field
 * [N3][N2][N1] (caller-owned, outlives the handle).  Tabulates G_hat on this rank's pencil
 * (k_y in [rank Yc, (rank+1) Yc)) and runs the Eq 55 check on it.                        */
UNO_API uno_status uno_slab_create(const uno_cg_desc* desc, int32_t rank, int32_t nranks, const uint8_t* d_phase,
                                   uno_slab_handle** out);
UNO_API uno_status uno_slab_destroy(uno_slab_handle* h);

/* Re-target the handle's launches to another stream (e.g. the capture stream of a CUDA graph
 * that records a chunk of iterations, exchanges included, so the iteration loop runs without a
 * host synchronisation per iteration).  The caller orders it against earlier work.          */
UNO_API uno_status uno_slab_set_stream(uno_slab_handle* h, void* stream);

/* out[0] = slab vector elements (nrhs*c*Z*N2*N1), out[1] = complex elements per a2a block
 * (nrhs*c*H1*Z*Yc), out[2] = fp64 elements per halo side (nrhs*c*N2*N1), out[3] = Z.    */
UNO_API uno_status uno_slab_sizes(uno_slab_handle* h, int64_t out[4]);

/* Alg 2 l.1-2 on the slab: r = f (Eq 76/81 RHS of this slab's nodes), u = 0, CG state
 * reset; loads / rel_tol / max_iter / fixed_iters as uno_cg_solve.                     */
UNO_API uno_status uno_slab_begin(uno_slab_handle* h, const double* h_loads, double rel_tol, int32_t max_iter,
                                  int32_t fixed_iters);

UNO_API uno_status uno_slab_forward(uno_slab_handle* h, double* d_send /* complex as 2 doubles */);
UNO_API uno_status uno_slab_green(uno_slab_handle* h, const double* d_recv, double* d_send);
UNO_API uno_status uno_slab_inverse(uno_slab_handle* h, const double* d_recv, double* d_halo_send);
UNO_API uno_status uno_slab_kapply(uno_slab_handle* h, const double* d_halo_recv);

/* Peer-memory variants of forward / green (BASELINE north star (e), SURVEY §8(e) "v2"): the
 * pack kernel stores each destination's block straight into that rank's receive buffer over
 * NVLink (P2P / CUDA IPC / symmetric-memory mappings), so the exchange is done by this kernel
 * and no send buffer or separate all-to-all exists.  h_peer_recv: HOST array [nranks] of
 * DEVICE pointers, entry q = rank q's receive buffer as addressable from this device (entry
 * `rank` = the local one); this rank writes block `rank` of each.  Use two receive buffer sets,
 * A for forward and B for green: green_peer reads the local A (d_recv) and writes the peers' B,
 * uno_slab_inverse then reads the local B.  Ordering (caller): every rank's forward_peer /
 * green_peer must complete before any rank reads the written buffers — the ||r||_inf and gamma
 * all-reduces that follow these stages (stream-ordered) provide exactly that; each pack kernel
 * ends with a system-scope fence.  UNO_ERR_NCCL: the peer table is NULL, has a NULL entry or
 * nranks exceeds the supported 8 peers.                                                   */
UNO_API uno_status uno_slab_forward_peer(uno_slab_handle* h, double* const* h_peer_recv);
UNO_API uno_status uno_slab_green_peer(uno_slab_handle* h, const double* d_recv, double* const* h_peer_recv);
/* Peer variant of inverse: the two boundary node planes of d go straight into the neighbours'
 * halo receive buffers (h_peer_halo_recv: HOST array [nranks] of DEVICE pointers to every rank's
 * halo receive buffer; my first plane -> recv[1] of rank-1, my last plane -> recv[0] of rank+1).
 * Ordering as above (barrier before the neighbours' uno_slab_kapply).                      */
UNO_API uno_status uno_slab_inverse_peer(uno_slab_handle* h, const double* d_recv, double* const* h_peer_halo_recv);

/* Per-rank partial of a CG scalar (slot UNO_SLAB_*), written to d_out[nrhs] (device);
 * uno_slab_apply takes the cross-rank totals d_in[nrhs] and updates the CG state.       */
UNO_API uno_status uno_slab_reduce(uno_slab_handle* h, int32_t slot, double* d_out);
UNO_API uno_status uno_slab_apply(uno_slab_handle* h, int32_t slot, const double* d_in);

/* Host copy of the CG state (synchronises the stream): *any_active, per-load reports.  */
UNO_API uno_status uno_slab_state(uno_slab_handle* h, int32_t* any_active, uno_cg_report* rep);

/* Apply the deferred u update and copy this slab's u to d_u [nrhs][c][Z][N2][N1].      */
UNO_API uno_status uno_slab_finish(uno_slab_handle* h, double* d_u);
/* Per (load, component) mean of d_u over this slab -> d_means[nrhs*c].  subtract_means takes
 * the SUM over ranks of those slab means (slabs are equal, so the grid mean is that sum / nranks)
 * and removes the grid mean per component.                                      */
UNO_API uno_status uno_slab_local_means(uno_slab_handle* h, const double* d_u, double* d_means);
UNO_API uno_status uno_slab_subtract_means(uno_slab_handle* h, double* d_u, const double* d_means);

#ifdef __cplusplus
}
#endif
#endif /* UNO_CG_SLAB_H */
