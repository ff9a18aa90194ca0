/*
 * sb200.h -- C ABI of libsb200.so, the B200 (sm_100a) implementation of the
 * seven Benchmark Streaming operations (BS1-BS7) of arXiv 2009.10917 and the
 * gather/scatter operator builders they consume.
 *
 * The reference (`streambench`, pure Python + numpy) has no FFI of its own;
 * its drop-in boundary is the Python function API re-exported by
 * pkg/src/streambench/__init__.py:3-13.  Each entry point below names the
 * reference function it replaces; INTEGRATION.md shows the ctypes binding a
 * streambench maintainer would add.
 *
 * Conventions
 *   - Every function returns SB_OK (0) or an SB_E_* code and never throws.
 *     sb_last_error() returns a thread-local message for the last failure.
 *   - Array arguments are DEVICE pointers (cudaMalloc / torch CUDA storage)
 *     unless stated otherwise.  Sizes are int64; mesh ids are int32, exactly
 *     like the reference's INDEX_DTYPE (mesh.py:15).
 *   - All work is enqueued on `stream` (a cudaStream_t; NULL = legacy default
 *     stream) and is asynchronous; results written through device pointers
 *     are valid once the stream is synchronised.
 *   - Reductions take a caller-owned zero-initialised workspace of
 *     sb_reduce_workspace_bytes(block_size, n_blocks) bytes.  Calls sharing a
 *     workspace must be ordered on one stream (the kernel leaves the workspace
 *     zeroed for the next call).
 *   - fp64 arithmetic is rounded exactly as the reference's numpy code: no
 *     FMA contraction, every product and sum rounded separately.
 */
#ifndef SB200_H
#define SB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void *sb_stream_t; /* cudaStream_t */

enum {
    SB_OK = 0,
    SB_E_INVALID = 1, /* bad argument (length, config, alignment of ids, ...) */
    SB_E_CUDA = 2,    /* CUDA runtime / launch failure */
    SB_E_RANGE = 3,   /* id or size outside the int32 id space */
};

/* ---- library ----------------------------------------------------------- */
int sb_version(void);                 /* 100*major + minor */
const char *sb_last_error(void);      /* thread-local, "" if none */
int sb_device_info(int device, int *sm_count, int *cc_major, int *cc_minor,
                   int64_t *l2_bytes);

/* ---- BS1 / BS2: elementwise streams (kernels.py:90-103) ----------------- */

/* kernels.py:90-93 bs1_copy(x, y): y[i] = x[i].  16 B/element. */
int sb_bs1_copy(const double *x, double *y, int64_t n, sb_stream_t stream);

/* kernels.py:96-103 bs2_axpy(alpha, x, beta, y): y = (alpha*x) + (beta*y),
 * two rounded products and one rounded add.  24 B/element.  x == y allowed. */
int sb_bs2_axpy(double alpha, const double *x, double beta, double *y, int64_t n,
                sb_stream_t stream);

/* ---- BS3 / BS4 / BS5: lattice reductions (kernels.py:19-132) ------------
 * The scalar equals kernels._reduce_product bit for bit for the same
 * ReductionConfig(block_size, n_blocks) (kernels.py:38-87): slot
 * s = b*block_size + t accumulates u[s + c*S]*v[s + c*S] (S = block_size *
 * n_blocks) in c order from +0.0, then a power-of-two tree per block, then
 * one block of block_size slots over the n_blocks partials.
 * block_size: power of two >= 2; n_blocks >= 1.  `result` is a device
 * double written when the kernel completes (single launch for
 * block_size <= 1024). */
size_t sb_reduce_workspace_bytes(int64_t block_size, int64_t n_blocks);

/* kernels.py:106-108 bs3_norm2(x, cfg).  8 B/element. */
int sb_bs3_norm2(const double *x, int64_t n, int64_t block_size, int64_t n_blocks,
                 void *workspace, double *result, sb_stream_t stream);

/* kernels.py:111-114 bs4_dot(x, y, cfg).  16 B/element. */
int sb_bs4_dot(const double *x, const double *y, int64_t n, int64_t block_size,
               int64_t n_blocks, void *workspace, double *result, sb_stream_t stream);

/* kernels.py:117-132 bs5_fused_cg_update(alpha, p, ap, x, r, cfg):
 * x += alpha*p; r -= alpha*ap; result = norm2(r_new) on the same lattice.
 * ONE pass: 48 B/element (the reference re-reads r). */
int sb_bs5_fused_cg_update(double alpha, const double *p, const double *ap, double *x,
                           double *r, int64_t n, int64_t block_size, int64_t n_blocks,
                           void *workspace, double *result, sb_stream_t stream);

/* Deterministic rank-order sum of `count` device doubles from +0.0
 * (multi-GPU combine of per-rank BS3/BS4/BS5 scalars after an all-gather). */
int sb_sum_ordered(const double *values, int64_t count, double *result, sb_stream_t stream);

/* ---- BS6 / BS7: gather / scatter (gs.py:10-61) ---------------------------- */

/* gs.py:10-39 bs6_gather(op, q_local): out[r] = sum of q_local[col_ids[c]],
 * c ascending over row r, from +0.0 -- or from carry_in[r] for r < n_carry
 * (multi-GPU carry halo; pass NULL/0 otherwise).  Rows are processed in the
 * operator's row blocks (block_starts, <= nodes_per_block nonzeros each).
 * 12*nl + 8*ng + 4*(ng+1) B per call (core.py:73). */
int sb_bs6_gather(const int32_t *block_starts, int64_t n_blocks, const int32_t *row_starts,
                  const int32_t *col_ids, int64_t ng, int64_t nl, int64_t nodes_per_block,
                  const double *q_local, double *out, const double *carry_in, int64_t n_carry,
                  sb_stream_t stream);

/* Pipelined BS6 (the fast path): a per-operator "plan" of super-blocks
 * (G = max(1, 512 / nodes_per_block) consecutive row blocks each) lets a
 * persistent kernel keep index tiles, value gathers and row sums of three
 * super-blocks in flight.  sb_bs6_plan_size returns the number of int32
 * plan entries (0 if nodes_per_block > 512: use sb_bs6_gather);
 * sb_bs6_make_plan fills it once per operator and synchronises its stream
 * once: the plan's trailer word flags a super-block with more than 512 rows
 * or entries (empty rows or a hand-built block_starts), and such a plan is
 * remembered by address so sb_bs6_gather_planned sums its rows straight from
 * global memory (still bitwise).  row_starts and col_ids must
 * be 16-byte aligned.  Results are bitwise those of sb_bs6_gather. */
int64_t sb_bs6_plan_size(int64_t n_blocks, int64_t nodes_per_block);
int sb_bs6_make_plan(const int32_t *block_starts, int64_t n_blocks, const int32_t *row_starts,
                     int64_t nodes_per_block, int32_t *plan, sb_stream_t stream);
/* Name of the kernel sb_bs6_gather_planned launches for this operator shape
 * (written into name[cap]; tests and the bench report it). */
int sb_bs6_planned_kernel(int64_t n_blocks, int64_t nodes_per_block, int64_t ng, int64_t nl,
                          char *name, size_t cap);
int sb_bs6_gather_planned(const int32_t *plan, int64_t n_blocks, int64_t nodes_per_block,
                          const int32_t *row_starts, const int32_t *col_ids, int64_t ng,
                          int64_t nl, const double *q_local, double *out,
                          const double *carry_in, int64_t n_carry, sb_stream_t stream);

/* BS6 over a z-slab WITH its carry halo in one launch (multi-GPU, dist.py
 * DistGather): the send operator's rows (this rank's top
 * interface plane) are summed straight into rank r+1's carry buffer
 * send_out[e & 1] (an NVLink-mapped address), the own operator's rows are
 * seeded from carry[e & 1] for rows < n_carry once rank r-1's partials have
 * landed.  `sync` (8 uint64, zeroed once, in this rank's symmetric window) holds
 * [0] ready (written by rank r-1), [1] ack (written by rank r+1), [2] the call
 * count e (device-side: CUDA-graph replays stay correct), [3..4] counters;
 * peer_ready = rank r+1's sync[0], peer_ack = rank r-1's sync[1] (NULL at
 * the ends; send_plan NULL on the last rank).  Plans from sb_bs6_make_plan
 * with the same nodes_per_block.  Results bitwise sb_bs6_gather's. */
int sb_bs6_gather_halo(const int32_t *send_plan, int64_t send_nblk, const int32_t *send_rs,
                       const int32_t *send_ci, double *const send_out[2], const int32_t *own_plan,
                       int64_t own_nblk, const int32_t *own_rs, const int32_t *own_ci, int64_t own_ng,
                       double *own_out, const double *const carry[2], int64_t n_carry, int64_t npb,
                       const double *q, uint64_t *sync, uint64_t *peer_ready, uint64_t *peer_ack,
                       sb_stream_t stream);


/* z-sweep BS6 for structured operators of order p <= 2 (the fast path
 * there; csrc/sb_gs_sweep.cu).  The operator's rows must be the lattice rows
 * of planes [c_lo, c_hi) of the slab z0..z1 of a K^3 order-p build_mesh
 * numbering (the sb_build_gather_csr geometry; whole mesh: 0, K, 0, K*p+1),
 * so ng = (c_hi-c_lo)*(K*p+1)^2 and nl = K*K*(z1-z0)*(p+1)^3.  A persistent
 * kernel sweeps columns of 32 x 8 rows along z, staging each element plane
 * under a column in shared memory once (cp.async.bulk) and reading the
 * entries from there (p = 2: one lane per row, its column ids checked against
 * the closed form; SB200_BS6_SWEEP_ROW2=0 selects the p = 1 value-tile
 * consumer).  Columns outside the staged element runs are read from global
 * memory, so ANY CSR with these rows gives the right answer: results are
 * bitwise those of sb_bs6_gather.  No plan; q_local 16-byte aligned. */
int sb_bs6_gather_sweep(int32_t K, int32_t p, int32_t z0, int32_t z1, int32_t c_lo, int32_t c_hi,
                        const int32_t *row_starts, const int32_t *col_ids, int64_t ng, int64_t nl,
                        const double *q_local, double *out, const double *carry_in, int64_t n_carry,
                        sb_stream_t stream);
/* Row-line-tiled BS6 for structured operators of order p = 1 (the fast path
 * there; csrc/sb_gs_tile.cu).  Same operator geometry contract as
 * sb_bs6_gather_sweep.  A CTA takes <= 128 consecutive rows of one lattice
 * row line and loads q in structure order (one 16 B node pair per element
 * and run); those values are used only when the tile's row starts and column
 * ids equal the closed form, otherwise the same kernel gathers in CSR order,
 * so ANY CSR with these rows gives sb_bs6_gather's result bit for bit. */
int sb_bs6_gather_tiled(int32_t K, int32_t p, int32_t z0, int32_t z1, int32_t c_lo, int32_t c_hi,
                        const int32_t *row_starts, const int32_t *col_ids, int64_t ng, int64_t nl,
                        const double *q_local, double *out, const double *carry_in, int64_t n_carry,
                        sb_stream_t stream);
/* Process-wide knobs of sb_bs6_gather_sweep for A/B runs (not thread-safe;
 * 0 / -1 restore the measured defaults): shared-memory ring slots (3..8,
 * default 4), L2 prefetch distance in element planes (-1: 0 = off; measured slower), work
 * items per resident CTA (default 8), value-tile swizzle (-1: for p = 1),
 * row lines per column = consumer warps per CTA (7, 8 or 16; 0: 8). */
int sb_bs6_sweep_tune(int32_t slots, int32_t l2_prefetch_planes, int32_t waves, int32_t swizzle,
                      int32_t row_lines);

/* gs.py:42-61 bs7_scatter(ids, q_global, q_local): q_local[n] =
 * q_global[ids[n]] where ids[n] >= 0 (masked entries untouched).  The caller
 * validates max(ids) < ng once per operator (sb_ids_minmax) instead of per
 * call.  12*nl + 8*ng B per call (core.py:79). */
int sb_bs7_scatter(const int32_t *ids, int64_t nl, const double *q_global, int64_t ng,
                   double *q_local, int has_mask, sb_stream_t stream);

/* gs.py:42-61 with q_global in two pieces: ids < n_own read q_own[id], ids
 * >= n_own read q_halo[id - n_own] (a multi-GPU slab's own rows and the halo
 * plane another rank wrote over NVLink; dist.py).  Ids must be < n_own +
 * n_halo (not re-checked). */
int sb_bs7_scatter_split(const int32_t *ids, int64_t nl, const double *q_own, int64_t n_own,
                         const double *q_halo, int64_t n_halo, double *q_local, int has_mask,
                         sb_stream_t stream);
/* The same with two alternating halo buffers: q_halo0 or q_halo1 by the parity
 * of (*call_count - 1), a device-side call counter that
 * sb_lsa_barrier_advance advanced just before (so captured CUDA graphs
 * alternate correctly on replay).  sb_bs7_halo_put copies n doubles of src
 * into dst0 or dst1 by the parity of *call_count (before the barrier): the
 * rank above's bottom plane into this rank's halo buffer (dist.py). */
int sb_bs7_scatter_split_pair(const int32_t *ids, int64_t nl, const double *q_own, int64_t n_own,
                              const double *q_halo0, const double *q_halo1, int64_t n_halo,
                              const unsigned long long *call_count, double *q_local, int has_mask,
                              sb_stream_t stream);
int sb_bs7_halo_put(const double *src, double *dst0, double *dst1, int64_t n,
                    const unsigned long long *call_count, sb_stream_t stream);

/* ---- operator construction (mesh.py:73-153) ------------------------------
 * Slab form: elements with ez in [z0, z1) of the K^3 order-p mesh; the
 * single-GPU operator is z0 = 0, z1 = K.  Local indices are relative to the
 * slab's first element ((ez - z0)*K^2 + ey*K + ex)*(p+1)^3 + node. */

/* mesh.py:73-97 build_mesh: local_to_global of the slab (global lattice ids).
 * l2g has K*K*(z1-z0)*(p+1)^3 entries.  SB_E_RANGE if (K*p+1)^3 > INT32_MAX. */
int sb_build_l2g(int64_t K, int64_t p, int64_t z0, int64_t z1, int32_t *l2g,
                 sb_stream_t stream);

/* mesh.py:113-134 build_gather rows and columns, closed form: rows are the
 * global lattice ids of planes c in [c_lo, c_hi) renumbered from 0;
 * row_starts (rows+1) and col_ids (nl of the slab) equal the reference's
 * bincount/cumsum and stable argsort bit for bit. */
int sb_build_gather_csr(int64_t K, int64_t p, int64_t z0, int64_t z1, int64_t c_lo,
                        int64_t c_hi, int32_t *row_starts, int32_t *col_ids,
                        sb_stream_t stream);

/* mesh.py:136-143 greedy block packing over row_starts (ng+1 entries).
 * block_starts needs room for max_blocks+1 entries (ng+1 always suffices);
 * *n_blocks_out (DEVICE int64) receives the block count, or -1 if a row is
 * longer than nodes_per_block, or -2 if more than max_blocks are needed.
 * Rows must be non-empty (the reference rejects empty rows, mesh.py:124). */
int sb_build_block_starts(const int32_t *row_starts, int64_t ng, int64_t nodes_per_block,
                          int32_t *block_starts, int64_t max_blocks, int64_t *n_blocks_out,
                          sb_stream_t stream);

/* mesh.py:150-153 multiplicity over the rows of planes [c_lo, c_hi) of the
 * slab (== row lengths), as doubles. */
int sb_multiplicity(int64_t K, int64_t p, int64_t z0, int64_t z1, int64_t c_lo,
                    int64_t c_hi, double *out, sb_stream_t stream);

/* mesh.py:100-110 build_scatter_ids: ids[n] = mask[l2g[n]] ? -1 : l2g[n].
 * mask_gids (DEVICE int64) lists n_mask global ids in [0, ng);
 * `scratch` is a device byte buffer of ng bytes. */
int sb_build_scatter_ids(const int32_t *l2g, int64_t nl, const int64_t *mask_gids,
                         int64_t n_mask, int64_t ng, uint8_t *scratch, int32_t *ids,
                         sb_stream_t stream);

/* mesh.py:113-134 for an ARBITRARY local_to_global map (meshes not made by
 * sb_build_l2g): col_ids = stable argsort(l2g) (CUB radix sort), row_starts =
 * [0, cumsum(bincount(l2g))].  `temp` is a device buffer of
 * sb_build_gather_general_temp_bytes(nl) bytes; stats (DEVICE, 2 x u64)
 * receives [min row length, max row length] so the caller can apply the
 * reference's coverage / nodes_per_block checks (mesh.py:124-129). */
size_t sb_build_gather_general_temp_bytes(int64_t nl);
int sb_build_gather_general(const int32_t *l2g, int64_t nl, int64_t ng, int32_t *row_starts,
                            int32_t *col_ids, void *temp, size_t temp_bytes,
                            unsigned long long *stats, sb_stream_t stream);

/* mesh.py:150-153 multiplicity for an arbitrary id map: out[g] = count of g
 * in ids (exact integer counts in doubles). */
int sb_histogram(const int32_t *ids, int64_t n, int64_t ng, double *out, sb_stream_t stream);

/* min and max of an int32 id array (out[0] = min, out[1] = max; DEVICE). */
int sb_ids_minmax(const int32_t *ids, int64_t n, int32_t *out, sb_stream_t stream);

/* ---- validators (the GPU counterpart of reference.py) -------------------- */

/* reference.py:25-30: sum(u[i]*v[i]) with each product rounded (as numpy
 * forms x*y) and accumulated in double-double; result rounded once.
 * workspace: sb_reduce_workspace_bytes(256, 592) bytes. */
int sb_dot_compensated(const double *u, const double *v, int64_t n, void *workspace,
                       double *result, sb_stream_t stream);


/* ---- device-resident CG (cg.py:27-72) -----------------
 * The solver's scalars live in device memory: alpha = rr / pAp and
 * beta = rr_new / rr are formed by one-thread control kernels (IEEE
 * division, exactly as Python's) and read by the streaming kernels, so no
 * host sync is needed per iteration.  All kernels are gated
 * on `active`; launching more iterations than needed is harmless.  One
 * iteration, given ap = A p computed by the caller on the same stream:
 *     sb_cg_pap(p, ap, ...); sb_cg_update(fused, p, ap, x, r, ...);
 *     sb_cg_direction(r, p, ...);
 * Iterates, iteration count and final r.r are bitwise those of cg_solve with
 * host scalars for the same ReductionConfig. */
enum { SB_CG_RUNNING = 0, SB_CG_CONVERGED = 1, SB_CG_EXHAUSTED = 2, SB_CG_NOT_SPD = 3 };
typedef struct sb_cg_state {
    double rr;          /* r.r of the current iterate */
    double rr_new;      /* r.r after the update */
    double pap;         /* p.Ap of the current direction */
    double tol;         /* eps, or eps * b.b for a relative tolerance */
    double fail_pap;    /* p.Ap that stopped the solve (SB_CG_NOT_SPD) */
    double alpha;       /* rr / pAp of the current iteration */
    double beta;        /* rr_new / rr of the current iteration */
    int64_t iterations; /* completed iterations */
    int64_t max_iter;
    int32_t active;     /* 1 while iterating */
    int32_t status;     /* SB_CG_* */
} sb_cg_state;

/* rr0 = r0.r0 (device), bb = b.b (device) for a relative tolerance or NULL. */
int sb_cg_begin(sb_cg_state *state, const double *rr0, const double *bb, double eps,
                int64_t max_iter, sb_stream_t stream);
/* kernels.py:111 bs4_dot(p, ap) -> state->pap, then the cg.py:61-64 SPD check. */
int sb_cg_pap(const double *p, const double *ap, int64_t n, int64_t block_size,
              int64_t n_blocks, void *workspace, sb_cg_state *state, sb_stream_t stream);
/* cg.py:65-70: fused (BS5) or unfused (BS2, BS2, BS3) update of x and r. */
int sb_cg_update(int fused, const double *p, const double *ap, double *x, double *r,
                 int64_t n, int64_t block_size, int64_t n_blocks, void *workspace,
                 sb_cg_state *state, sb_stream_t stream);
/* cg.py:71-74: p = r + beta p, then advance the iteration. */
int sb_cg_direction(const double *r, double *p, int64_t n, sb_cg_state *state,
                    sb_stream_t stream);


/* ---- fused multi-GPU reductions -----------------------
 * BS3/BS4/BS5 whose CTA 0 also combines the per-rank scalars over NVLink
 * peer memory (NCCL 2.28 device API, LSA windows): the rank's value is
 * stored into every peer's symmetric window, the ranks meet at an LSA
 * barrier, and each sums the values in rank order from +0.0 -- bitwise the
 * all-gather + sb_sum_ordered result, in a single launch.  Collective: every
 * rank of the context must make the same sequence of calls, one stream per
 * context.  Needs libnccl.so.2 >= 2.28 in the process (torch's) and every
 * rank NVLink-reachable; otherwise sb_lsa_create returns SB_E_INVALID. */
typedef struct sb_lsa sb_lsa_t;
/* SB_OK when this process can attempt the fused path (libnccl.so.2 >= 2.28
 * with the host symbols loadable); local, non-collective, no side effects --
 * ranks agree on it before the collective sb_lsa_create. */
int sb_lsa_available(void);
int sb_lsa_unique_id(void *out, size_t bytes);  /* rank 0; bytes >= 128 */
int sb_lsa_create(const void *unique_id, size_t bytes, int nranks, int rank, sb_lsa_t **out);
int sb_lsa_destroy(sb_lsa_t *ctx);  /* collective (every rank of the context) */
/* Local, non-collective teardown (ncclCommAbort) for a context whose peers
 * did not all finish sb_lsa_create. */
int sb_lsa_abort(sb_lsa_t *ctx);
/* BS6 carry halo over NVLink (dist.py DistGather): a symmetric window per
 * context (collective); sb_lsa_halo_pointers returns this rank's local
 * address of `offset` and peer `peer`'s NVLink-mapped address of it, so the
 * send-plane gather (sb_bs6_gather_planned) writes its partials straight
 * into rank+1's carry buffer; sb_lsa_barrier (collective, one thread)
 * orders those stores before rank+1's own gather reads them. */
int sb_lsa_halo_window(sb_lsa_t *ctx, size_t bytes);
int sb_lsa_halo_pointers(sb_lsa_t *ctx, size_t offset, int peer, void **local, void **remote);
int sb_lsa_barrier(sb_lsa_t *ctx, sb_stream_t stream);
/* The barrier, then *call_count += 1 (one thread; the BS7 halo parity). */
int sb_lsa_barrier_advance(sb_lsa_t *ctx, unsigned long long *call_count, sb_stream_t stream);
/* Multi-GPU device-resident CG: sb_cg_pap / sb_cg_update whose reductions
 * (pAp, r.r) combine over the ranks in the same launch, so every rank's
 * sb_cg_state holds the global scalars and the ranks gate identically;
 * sb_cg_begin / sb_cg_direction are used unchanged (with rr0 / b.b from
 * sb_lsa_bs3_norm2).  Vectors are the rank's chunks. */
int sb_lsa_cg_pap(const double *p, const double *ap, int64_t n, int64_t block_size,
                  int64_t n_blocks, void *workspace, sb_cg_state *state, sb_lsa_t *ctx,
                  sb_stream_t stream);
int sb_lsa_cg_update(int fused, const double *p, const double *ap, double *x, double *r,
                     int64_t n, int64_t block_size, int64_t n_blocks, void *workspace,
                     sb_cg_state *state, sb_lsa_t *ctx, sb_stream_t stream);
int sb_lsa_bs3_norm2(const double *x, int64_t n, int64_t block_size, int64_t n_blocks,
                     void *workspace, double *result, sb_lsa_t *ctx, sb_stream_t stream);
int sb_lsa_bs4_dot(const double *x, const double *y, int64_t n, int64_t block_size,
                   int64_t n_blocks, void *workspace, double *result, sb_lsa_t *ctx,
                   sb_stream_t stream);
int sb_lsa_bs5_fused_cg_update(double alpha, const double *p, const double *ap, double *x,
                               double *r, int64_t n, int64_t block_size, int64_t n_blocks,
                               void *workspace, double *result, sb_lsa_t *ctx,
                               sb_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* SB200_H */
