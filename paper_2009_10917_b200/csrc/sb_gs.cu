// sb_gs.cu -- BS6 gather (Z^T) and BS7 scatter (Z) (gs.py:10-61).
//
// BS6 follows the paper's Listing 4 structure, B200-sized: a CTA owns G
// consecutive row blocks of the operator (block_starts from build_gather,
// <= nodes_per_block nonzeros each, so <= CAP = G*npb entries), loads that
// contiguous col_ids / row_starts window with coalesced streaming loads,
// gathers q_local[col_ids] into shared memory (all loads in flight before the
// first use), then one thread per row sums its entries in ascending column
// order from +0.0 (or from the carry-in partial of a lower rank) and writes
// out[r] -- bitwise the reference's per-row sequential sum (gs.py:34-36).
//
// BS7 (sb_gs_pipe.cu) streams ids and q_local (evict-first) and gathers
// q_global with an L2 evict_last policy: every global node is re-read by up
// to 8 elements, the furthest one a whole element layer later (SURVEY
// Appendix A.6), so q_global must survive the streams in L2.
#include <stdlib.h>

#include <algorithm>

#include "sb_common.cuh"

namespace sb {

constexpr int kGsThreads = 256;
constexpr int kGatherCap = 2048;  // entries staged per CTA (16 KB of q)

template <int T, int CAP>
__global__ void __launch_bounds__(T) k_bs6_smem(const int32_t *__restrict__ bst, int64_t nblk, int G,
                                               const int32_t *__restrict__ rs,
                                               const int32_t *__restrict__ ci,
                                               const double *__restrict__ q, double *__restrict__ out,
                                               const double *__restrict__ carry, int64_t ncarry) {
    __shared__ double qs[CAP];
    __shared__ int32_t rss[CAP + 1];
    const int64_t b0 = (int64_t)blockIdx.x * G;
    const int64_t b1 = b0 + G < nblk ? b0 + G : nblk;
    const int32_t r0 = __ldg(bst + b0), r1 = __ldg(bst + b1);
    const int nrows = r1 - r0;
    const int32_t e0 = __ldg(rs + r0);
    const int ne = __ldg(rs + r1) - e0;
    constexpr int M = CAP / T;
    if (ne > CAP || nrows > CAP) {
        // blocks that do not fit the tile (empty rows padding a block past CAP
        // rows, or block_starts not packed to nodes_per_block): rows straight
        // from global memory, same ascending order
        for (int k = threadIdx.x; k < nrows; k += T) {
            const int64_t r = (int64_t)r0 + k;
            double acc = r < ncarry ? carry[r] : 0.0;
            for (int32_t c = rs[r], e = rs[r + 1]; c < e; c++) acc = add(acc, __ldg(q + ci[c]));
            st_stream(out + r, acc);
        }
        return;
    }
    int32_t cols[M];
#pragma unroll
    for (int m = 0; m < M; m++) {
        const int k = threadIdx.x + m * T;
        if (k < ne) cols[m] = ld_stream(ci + e0 + k);
    }
    for (int k = threadIdx.x; k <= nrows; k += T) rss[k] = ld_stream(rs + r0 + k);
#pragma unroll
    for (int m = 0; m < M; m++) {
        const int k = threadIdx.x + m * T;
        if (k < ne) qs[k] = __ldg(q + cols[m]);
    }
    __syncthreads();
    for (int k = threadIdx.x; k < nrows; k += T) {
        const int s = rss[k] - e0, e = rss[k + 1] - e0;
        const int64_t r = (int64_t)r0 + k;
        double acc = r < ncarry ? carry[r] : 0.0;
        for (int c = s; c < e; c++) acc = add(acc, qs[c]);
        st_stream(out + r, acc);
    }
}

// Rows straight from global memory (operators whose blocks exceed CAP).
__global__ void __launch_bounds__(256) k_bs6_rows(const int32_t *__restrict__ rs, const int32_t *__restrict__ ci,
                                                 int64_t ng, const double *__restrict__ q,
                                                 double *__restrict__ out, const double *__restrict__ carry,
                                                 int64_t ncarry) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < ng;
         r += (int64_t)gridDim.x * blockDim.x) {
        double acc = r < ncarry ? carry[r] : 0.0;
        const int32_t s = rs[r], e = rs[r + 1];
        for (int32_t c = s; c < e; c++) acc = add(acc, __ldg(q + ci[c]));
        out[r] = acc;
    }
}

int bs7_lanes_launch(const int32_t *ids, int64_t nl, const double *qg, double *ql, int has_mask,
                     cudaStream_t st);  // sb_gs_pipe.cu
int bs7_split_launch(const int32_t *ids, int64_t nl, const double *qg, int32_t split, const double *qh,
                     const double *qh1, const unsigned long long *cnt, double *ql, int has_mask,
                     cudaStream_t st);  // sb_gs_pipe.cu
int halo_put_launch(const double *src, double *dst0, double *dst1, int64_t n, const unsigned long long *cnt,
                    cudaStream_t st);  // sb_gs_pipe.cu

// rows straight from global memory for every operator (A/B reference point)
int bs6_rows_launch(const int32_t *rs, const int32_t *ci, int64_t ng, const double *q, double *out,
                    const double *carry, int64_t ncarry, cudaStream_t st) {
    const int64_t grid = std::min<int64_t>((ng + 255) / 256, (int64_t)sm_count() * 32);
    k_bs6_rows<<<(unsigned)grid, 256, 0, st>>>(rs, ci, ng, q, out, carry, ncarry);
    return launch_check("sb_bs6_gather");
}

}  // namespace sb

using namespace sb;

extern "C" {

int sb_bs6_gather(const int32_t *bst, int64_t nblk, const int32_t *rs, const int32_t *ci, int64_t ng,
                  int64_t nl, int64_t npb, const double *q, double *out, const double *carry,
                  int64_t ncarry, sb_stream_t s) {
    clear_error();
    if (ng < 0 || nl < 0 || nblk < 0 || npb < 1 || ncarry < 0 || (ncarry > 0 && !carry) ||
        (ng > 0 && (!rs || !out || !bst || nblk < 1)) || (nl > 0 && (!ci || !q))) {
        set_error("sb_bs6_gather: invalid arguments");
        return SB_E_INVALID;
    }
    if (ng == 0) return SB_OK;
    if (ncarry > ng) ncarry = ng;
    cudaStream_t st = as_stream(s);
    if (npb <= kGatherCap) {
        const int G = (int)std::max<int64_t>(1, kGatherCap / npb);
        const int64_t grid = (nblk + G - 1) / G;
        k_bs6_smem<kGsThreads, kGatherCap><<<(unsigned)grid, kGsThreads, 0, st>>>(bst, nblk, G, rs, ci, q,
                                                                               out, carry, ncarry);
    } else {
        const int64_t grid = std::min<int64_t>((ng + 255) / 256, (int64_t)sm_count() * 32);
        k_bs6_rows<<<(unsigned)grid, 256, 0, st>>>(rs, ci, ng, q, out, carry, ncarry);
    }
    return launch_check("sb_bs6_gather");
}

int sb_bs7_scatter(const int32_t *ids, int64_t nl, const double *qg, int64_t ng, double *ql,
                   int has_mask, sb_stream_t s) {
    clear_error();
    if (nl < 0 || ng < 0 || (nl > 0 && (!ids || !ql || (!qg && ng > 0)))) {
        set_error("sb_bs7_scatter: invalid arguments");
        return SB_E_INVALID;
    }
    if (nl == 0) return SB_OK;
    return bs7_lanes_launch(ids, nl, qg, ql, has_mask, as_stream(s));
}

int sb_bs7_scatter_split(const int32_t *ids, int64_t nl, const double *q_own, int64_t n_own,
                         const double *q_halo, int64_t n_halo, double *ql, int has_mask, sb_stream_t s) {
    clear_error();
    if (nl < 0 || n_own < 0 || n_halo < 0 || n_own > 0x7fffffffLL ||
        (nl > 0 && (!ids || !ql || (n_own > 0 && !q_own) || (n_halo > 0 && !q_halo)))) {
        set_error("sb_bs7_scatter_split: invalid arguments");
        return SB_E_INVALID;
    }
    if (nl == 0) return SB_OK;
    return bs7_split_launch(ids, nl, q_own, (int32_t)n_own, q_halo, nullptr, nullptr, ql, has_mask, as_stream(s));
}

int sb_bs7_scatter_split_pair(const int32_t *ids, int64_t nl, const double *q_own, int64_t n_own,
                              const double *q_halo0, const double *q_halo1, int64_t n_halo,
                              const unsigned long long *call_count, double *ql, int has_mask, sb_stream_t s) {
    clear_error();
    if (nl < 0 || n_own < 0 || n_halo < 0 || n_own > 0x7fffffffLL || !call_count ||
        (nl > 0 && (!ids || !ql || (n_own > 0 && !q_own) || (n_halo > 0 && (!q_halo0 || !q_halo1))))) {
        set_error("sb_bs7_scatter_split_pair: invalid arguments");
        return SB_E_INVALID;
    }
    if (nl == 0) return SB_OK;
    return bs7_split_launch(ids, nl, q_own, (int32_t)n_own, q_halo0, q_halo1, call_count, ql, has_mask,
                            as_stream(s));
}

int sb_bs7_halo_put(const double *src, double *dst0, double *dst1, int64_t n, const unsigned long long *call_count,
                    sb_stream_t s) {
    clear_error();
    if (n < 0 || (n > 0 && (!src || !dst0 || !dst1 || !call_count))) {
        set_error("sb_bs7_halo_put: invalid arguments");
        return SB_E_INVALID;
    }
    if (n == 0) return SB_OK;
    return halo_put_launch(src, dst0, dst1, n, call_count, as_stream(s));
}

}  // extern "C"
