// sb_build.cu -- gather/scatter operator construction on the GPU (mesh.py:73-153).
//
// The reference builds Z^T with bincount + stable argsort + cumsum + a greedy
// searchsorted loop (mesh.py:113-147) -- O(NG * n_blocks) on the host
// (SURVEY Appendix B.1).  The structured K^3 order-p numbering has a closed
// form that gives the same arrays bit for bit:
//   * per axis, lattice coordinate c belongs to element c/p (local c%p) and,
//     when c%p == 0, also to element c/p-1 (local p) -- so a row (global id
//     (c*g+b)*g+a) has cx*cy*cz entries, and ascending local index is the
//     lexicographic (ez, ey, ex) order of those candidates;
//   * the exclusive prefix of row lengths factorises per axis, so
//     row_starts[r] is O(1) per row (no scan);
//   * block_starts is the reference's greedy packing, walked by one warp over
//     row_starts staged in shared memory (a 32-way ballot search per block).
// Everything is generalised to a z-slab of element layers [z0, z1) and a
// plane range [c_lo, c_hi) of rows, which is what the multi-GPU partition
// needs; z0 = 0, z1 = K, c_lo = 0, c_hi = K*p+1 is the reference operator.
#include <algorithm>
#include <climits>

#include "sb_common.cuh"

namespace sb {

struct Axis {
    int64_t e_lo, e_hi, p;
};

// F(c) = number of (element, local) pairs along this axis with coordinate < c
//      = sum_{e in [e_lo, e_hi)} clamp(c - e*p, 0, p+1).
__device__ __forceinline__ int64_t axis_prefix(int64_t c, const Axis &A) {
    if (c <= A.e_lo * A.p) return 0;
    int64_t full_end = c >= A.p + 1 ? (c - A.p - 1) / A.p + 1 : 0;
    full_end = full_end < A.e_lo ? A.e_lo : (full_end > A.e_hi ? A.e_hi : full_end);
    int64_t sum = (full_end - A.e_lo) * (A.p + 1);
    for (int64_t e = full_end; e < A.e_hi && e * A.p < c; e++) sum += c - e * A.p;
    return sum;
}

// Candidate (element, local) pairs containing coordinate c, ascending element.
__device__ __forceinline__ int axis_cands(int64_t c, const Axis &A, int64_t e[2], int64_t l[2]) {
    int n = 0;
    const int64_t q = c / A.p, m = c % A.p;
    if (m == 0 && q - 1 >= A.e_lo && q - 1 < A.e_hi) { e[n] = q - 1; l[n] = A.p; n++; }
    if (q >= A.e_lo && q < A.e_hi) { e[n] = q; l[n] = m; n++; }
    return n;
}

// mesh.py:85-97: node (i,j,k) of element (ex,ey,ez) -> lattice (ex*p+i, ey*p+j, ez*p+k)
__global__ void k_l2g(int64_t K, int64_t p, int64_t z0, int64_t nl, int32_t *l2g) {
    const int64_t npe = p + 1, npe3 = npe * npe * npe, g = K * p + 1;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < nl;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = idx / npe3, nd = idx - e * npe3;
        const int64_t ex = e % K, ey = (e / K) % K, ez = z0 + e / (K * K);
        const int64_t i = nd % npe, j = (nd / npe) % npe, k = nd / (npe * npe);
        l2g[idx] = (int32_t)(((ez * p + k) * g + (ey * p + j)) * g + (ex * p + i));
    }
}

struct CsrArgs {
    int64_t K, p, z0, z1, c_lo, c_hi, g, nrows;
    int64_t SX, SY, Fz_lo;
};

__global__ void k_csr(CsrArgs a, int32_t *rs, int32_t *ci) {
    const Axis AX{0, a.K, a.p}, AZ{a.z0, a.z1, a.p};
    const int64_t npe = a.p + 1, npe3 = npe * npe * npe;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < a.nrows;
         r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t ai = r % a.g, bi = (r / a.g) % a.g, ci_ = a.c_lo + r / (a.g * a.g);
        const int64_t Fx = axis_prefix(ai, AX), cx = axis_prefix(ai + 1, AX) - Fx;
        const int64_t Fy = axis_prefix(bi, AX), cy = axis_prefix(bi + 1, AX) - Fy;
        const int64_t Fz = axis_prefix(ci_, AZ), cz = axis_prefix(ci_ + 1, AZ) - Fz;
        const int64_t start = (Fz - a.Fz_lo) * a.SY * a.SX + cz * Fy * a.SX + cz * cy * Fx;
        rs[r] = (int32_t)start;
        if (r == a.nrows - 1) rs[a.nrows] = (int32_t)(start + cx * cy * cz);
        int64_t ex[2], lx[2], ey[2], ly[2], ez[2], lz[2];
        const int nx = axis_cands(ai, AX, ex, lx);
        const int ny = axis_cands(bi, AX, ey, ly);
        const int nz = axis_cands(ci_, AZ, ez, lz);
        int64_t o = start;
        for (int z = 0; z < nz; z++)
            for (int y = 0; y < ny; y++)
                for (int x = 0; x < nx; x++) {
                    const int64_t elem = ((ez[z] - a.z0) * a.K + ey[y]) * a.K + ex[x];
                    ci[o++] = (int32_t)(elem * npe3 + (lz[z] * npe + ly[y]) * npe + lx[x]);
                }
    }
}

__global__ void k_mult(CsrArgs a, double *out) {
    const Axis AX{0, a.K, a.p}, AZ{a.z0, a.z1, a.p};
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < a.nrows;
         r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t ai = r % a.g, bi = (r / a.g) % a.g, ci_ = a.c_lo + r / (a.g * a.g);
        const int64_t cx = axis_prefix(ai + 1, AX) - axis_prefix(ai, AX);
        const int64_t cy = axis_prefix(bi + 1, AX) - axis_prefix(bi, AX);
        const int64_t cz = axis_prefix(ci_ + 1, AZ) - axis_prefix(ci_, AZ);
        out[r] = (double)(cx * cy * cz);
    }
}

// mesh.py:136-143 greedy packing: nxt = searchsorted(rs, rs[row]+npb, 'right')-1,
// clamped to [row+1, ng].  One CTA; row_starts staged CH rows at a time; warp 0
// walks the chain with a 32-way ballot search (rows are non-empty, so the
// answer lies in [row+1, row+npb]).
constexpr int kChunk = 12000;

template <bool SMEM>
__global__ void __launch_bounds__(1024) k_block_starts(const int32_t *rs, int64_t ng, int64_t npb,
                                                       int32_t *bst, int64_t maxb, int64_t *nblk_out) {
    __shared__ int32_t sh[SMEM ? kChunk + 1 : 1];
    __shared__ long long s_row, s_nb;
    __shared__ int s_err;
    const int lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        s_row = 0;
        s_nb = 0;
        s_err = 0;
        bst[0] = 0;
    }
    __syncthreads();
    while (true) {
        int64_t row = s_row;
        if (row >= ng || s_err) break;
        const int64_t base = row;
        const int64_t cnt = SMEM ? std::min<int64_t>(kChunk, ng - base) + 1 : ng - base + 1;
        if (SMEM)
            for (int64_t k = threadIdx.x; k < cnt; k += blockDim.x) sh[k] = rs[base + k];
        __syncthreads();
        const int32_t *R = SMEM ? sh : rs + base;  // R[j - base] == rs[j]
        if (threadIdx.x < 32) {
            int64_t nb = s_nb;
            const int64_t last = base + cnt - 1;  // last row index whose start is loaded
            int err = 0;
            while (row < ng) {
                const int64_t limit = (int64_t)R[row - base] + npb;
                int64_t hi = std::min<int64_t>(row + npb, ng);
                if (hi > last) break;  // reload a chunk starting at `row`
                int64_t lo = row + 1;
                if ((int64_t)R[lo - base] > limit) { err = 1; break; }  // row longer than npb
                while (hi > lo) {
                    const int64_t step = (hi - lo + 31) / 32;
                    const int64_t pos = std::min<int64_t>(lo + step * (lane + 1), hi);
                    const bool ok = (int64_t)R[pos - base] <= limit;
                    const int c = __popc(__ballot_sync(0xffffffffu, ok));
                    const int64_t plo = c > 0 ? std::min<int64_t>(lo + step * c, hi) : lo;
                    const int64_t phi = c < 32 ? std::min<int64_t>(lo + step * (c + 1), hi) - 1 : hi;
                    lo = plo;
                    hi = phi;
                }
                if (++nb > maxb) { err = 2; break; }
                if (lane == 0) bst[nb] = (int32_t)lo;
                row = lo;
            }
            if (lane == 0) {
                s_row = row;
                s_nb = nb;
                if (err) s_err = err;
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) *nblk_out = s_err ? -(int64_t)s_err : (int64_t)s_nb;
}

__global__ void k_fill_u8(uint8_t *p, int64_t n, uint8_t v) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        p[i] = v;
}

__global__ void k_mark(const int64_t *gids, int64_t n, uint8_t *m) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        m[gids[i]] = 1;
}

__global__ void k_apply_mask(const int32_t *l2g, int64_t nl, const uint8_t *m, int32_t *ids) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nl;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t g = l2g[i];
        ids[i] = (m && m[g]) ? -1 : g;
    }
}

__global__ void k_minmax_init(int32_t *out) {
    out[0] = INT_MAX;
    out[1] = INT_MIN;
}

__global__ void __launch_bounds__(256) k_minmax(const int32_t *ids, int64_t n, int32_t *out) {
    int32_t lo = INT_MAX, hi = INT_MIN;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = ids[i];
        lo = min(lo, v);
        hi = max(hi, v);
    }
    for (int o = 16; o; o >>= 1) {
        lo = min(lo, __shfl_down_sync(0xffffffffu, lo, o));
        hi = max(hi, __shfl_down_sync(0xffffffffu, hi, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(out, lo);
        atomicMax(out + 1, hi);
    }
}

static int grid_for(int64_t n) {
    return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)sm_count() * 32));
}

static int slab_args(int64_t K, int64_t p, int64_t z0, int64_t z1, int64_t c_lo, int64_t c_hi,
                     CsrArgs &a, const char *name) {
    if (K < 1 || p < 1 || z0 < 0 || z1 > K || z0 >= z1 || c_lo < z0 * p || c_hi > z1 * p + 1 ||
        c_lo >= c_hi) {
        set_error("%s: invalid slab (K=%lld p=%lld z=[%lld,%lld) c=[%lld,%lld))", name, (long long)K,
                  (long long)p, (long long)z0, (long long)z1, (long long)c_lo, (long long)c_hi);
        return SB_E_INVALID;
    }
    const int64_t g = K * p + 1;
    if (g * g * g > INT32_MAX) {
        set_error("%s: global id space (K*p+1)^3 = %lld overflows int32", name, (long long)(g * g * g));
        return SB_E_RANGE;
    }
    a.K = K; a.p = p; a.z0 = z0; a.z1 = z1; a.c_lo = c_lo; a.c_hi = c_hi; a.g = g;
    a.nrows = (c_hi - c_lo) * g * g;
    a.SX = K * (p + 1);
    a.SY = K * (p + 1);
    // Fz(c_lo) on the host: same formula as axis_prefix
    int64_t F = 0;
    for (int64_t e = z0; e < z1; e++) F += std::max<int64_t>(0, std::min<int64_t>(c_lo - e * p, p + 1));
    a.Fz_lo = F;
    // entries of the slab rows must fit int32
    int64_t Fhi = 0;
    for (int64_t e = z0; e < z1; e++) Fhi += std::max<int64_t>(0, std::min<int64_t>(c_hi - e * p, p + 1));
    if ((Fhi - F) * a.SX * a.SY > INT32_MAX) {
        set_error("%s: %lld local DOFs overflow the int32 id space", name,
                  (long long)((Fhi - F) * a.SX * a.SY));
        return SB_E_RANGE;
    }
    return SB_OK;
}

}  // namespace sb

using namespace sb;

extern "C" {

int sb_build_l2g(int64_t K, int64_t p, int64_t z0, int64_t z1, int32_t *l2g, sb_stream_t s) {
    clear_error();
    CsrArgs a;
    if (int rc = slab_args(K, p, z0, z1, z0 * p, z1 * p + 1, a, "sb_build_l2g")) return rc;
    const int64_t nl = K * K * (z1 - z0) * (p + 1) * (p + 1) * (p + 1);
    if (nl > INT32_MAX) {
        set_error("sb_build_l2g: NL = %lld overflows int32 local indices", (long long)nl);
        return SB_E_RANGE;
    }
    if (!l2g) { set_error("sb_build_l2g: null output"); return SB_E_INVALID; }
    k_l2g<<<grid_for(nl), 256, 0, as_stream(s)>>>(K, p, z0, nl, l2g);
    return launch_check("sb_build_l2g");
}

int sb_build_gather_csr(int64_t K, int64_t p, int64_t z0, int64_t z1, int64_t c_lo, int64_t c_hi,
                        int32_t *rs, int32_t *ci, sb_stream_t s) {
    clear_error();
    CsrArgs a;
    if (int rc = slab_args(K, p, z0, z1, c_lo, c_hi, a, "sb_build_gather_csr")) return rc;
    if (!rs || !ci) { set_error("sb_build_gather_csr: null output"); return SB_E_INVALID; }
    k_csr<<<grid_for(a.nrows), 256, 0, as_stream(s)>>>(a, rs, ci);
    return launch_check("sb_build_gather_csr");
}

int sb_multiplicity(int64_t K, int64_t p, int64_t z0, int64_t z1, int64_t c_lo, int64_t c_hi,
                    double *out, sb_stream_t s) {
    clear_error();
    CsrArgs a;
    if (int rc = slab_args(K, p, z0, z1, c_lo, c_hi, a, "sb_multiplicity")) return rc;
    if (!out) { set_error("sb_multiplicity: null output"); return SB_E_INVALID; }
    k_mult<<<grid_for(a.nrows), 256, 0, as_stream(s)>>>(a, out);
    return launch_check("sb_multiplicity");
}

int sb_build_block_starts(const int32_t *rs, int64_t ng, int64_t npb, int32_t *bst, int64_t maxb,
                          int64_t *nblk_out, sb_stream_t s) {
    clear_error();
    if (ng < 0 || npb < 1 || maxb < 0 || !bst || !nblk_out || (ng > 0 && !rs)) {
        set_error("sb_build_block_starts: invalid arguments");
        return SB_E_INVALID;
    }
    if (npb + 1 <= kChunk)
        k_block_starts<true><<<1, 1024, 0, as_stream(s)>>>(rs, ng, npb, bst, maxb, nblk_out);
    else
        k_block_starts<false><<<1, 1024, 0, as_stream(s)>>>(rs, ng, npb, bst, maxb, nblk_out);
    return launch_check("sb_build_block_starts");
}

int sb_build_scatter_ids(const int32_t *l2g, int64_t nl, const int64_t *mask_gids, int64_t n_mask,
                         int64_t ng, uint8_t *scratch, int32_t *ids, sb_stream_t s) {
    clear_error();
    if (nl < 0 || n_mask < 0 || (nl > 0 && (!l2g || !ids)) || (n_mask > 0 && (!mask_gids || !scratch))) {
        set_error("sb_build_scatter_ids: invalid arguments");
        return SB_E_INVALID;
    }
    cudaStream_t st = as_stream(s);
    const uint8_t *m = nullptr;
    if (n_mask > 0) {
        k_fill_u8<<<grid_for(ng), 256, 0, st>>>(scratch, ng, 0);
        k_mark<<<grid_for(n_mask), 256, 0, st>>>(mask_gids, n_mask, scratch);
        m = scratch;
    }
    if (nl > 0) k_apply_mask<<<grid_for(nl), 256, 0, st>>>(l2g, nl, m, ids);
    return launch_check("sb_build_scatter_ids");
}

int sb_ids_minmax(const int32_t *ids, int64_t n, int32_t *out, sb_stream_t s) {
    clear_error();
    if (n < 0 || !out || (n > 0 && !ids)) {
        set_error("sb_ids_minmax: invalid arguments");
        return SB_E_INVALID;
    }
    cudaStream_t st = as_stream(s);
    k_minmax_init<<<1, 1, 0, st>>>(out);
    if (n > 0) k_minmax<<<grid_for(n), 256, 0, st>>>(ids, n, out);
    return launch_check("sb_ids_minmax");
}

}  // extern "C"

// ---- general (unstructured) operator construction -------------------------
// mesh.py:113-134 for an arbitrary local_to_global map: col_ids = stable
// argsort(l2g) (CUB radix sort of (key=l2g, value=iota) is stable), and
// row_starts[r] = lower_bound(sorted keys, r) (== [0, cumsum(bincount)]).
#include <cub/device/device_radix_sort.cuh>

namespace sb {

__global__ void k_iota(int32_t *v, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        v[i] = (int32_t)i;
}

// row_starts[r] = first index with key >= r; stats: [min row len, max row len]
__global__ void k_row_bounds(const int32_t *keys, int64_t nl, int64_t ng, int32_t *rs,
                             unsigned long long *stats) {
    unsigned long long mn = ~0ull, mx = 0;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r <= ng;
         r += (int64_t)gridDim.x * blockDim.x) {
        int64_t lo = 0, hi = nl;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (keys[mid] < r) lo = mid + 1; else hi = mid;
        }
        rs[r] = (int32_t)lo;
        if (r < ng) {
            int64_t lo2 = lo, hi2 = nl;
            while (lo2 < hi2) {
                const int64_t mid = (lo2 + hi2) >> 1;
                if (keys[mid] < r + 1) lo2 = mid + 1; else hi2 = mid;
            }
            const unsigned long long len = (unsigned long long)(lo2 - lo);
            mn = len < mn ? len : mn;
            mx = len > mx ? len : mx;
        }
    }
    atomicMin(stats, mn);
    atomicMax(stats + 1, mx);
}

__global__ void k_stats_init(unsigned long long *stats) {
    stats[0] = ~0ull;
    stats[1] = 0ull;
}

__global__ void k_histogram(const int32_t *ids, int64_t n, double *out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(out + ids[i], 1.0);
}

static size_t general_layout(int64_t nl, size_t *sort_bytes) {
    size_t sb = 0;
    cub::DeviceRadixSort::SortPairs<int32_t, int32_t>(nullptr, sb, (const int32_t *)nullptr,
                                                      (int32_t *)nullptr, (const int32_t *)nullptr,
                                                      (int32_t *)nullptr, (int)nl);
    *sort_bytes = (sb + 255) & ~(size_t)255;
    const size_t arr = ((size_t)nl * sizeof(int32_t) + 255) & ~(size_t)255;
    return *sort_bytes + 2 * arr + 256;  // sort temp + sorted keys + iota values + stats
}

}  // namespace sb

extern "C" {

size_t sb_build_gather_general_temp_bytes(int64_t nl) {
    size_t sbytes;
    return sb::general_layout(nl, &sbytes);
}

int sb_build_gather_general(const int32_t *l2g, int64_t nl, int64_t ng, int32_t *rs, int32_t *ci,
                            void *temp, size_t temp_bytes, unsigned long long *stats, sb_stream_t s) {
    using namespace sb;
    clear_error();
    if (nl < 0 || ng < 0 || nl > INT32_MAX || ng > INT32_MAX || !rs || !stats ||
        (nl > 0 && (!l2g || !ci || !temp))) {
        set_error("sb_build_gather_general: invalid arguments");
        return SB_E_INVALID;
    }
    size_t sort_bytes;
    const size_t need = general_layout(nl, &sort_bytes);
    if (temp_bytes < need) {
        set_error("sb_build_gather_general: temp too small (%zu < %zu)", temp_bytes, need);
        return SB_E_INVALID;
    }
    cudaStream_t st = as_stream(s);
    char *t = static_cast<char *>(temp);
    const size_t arr = ((size_t)nl * sizeof(int32_t) + 255) & ~(size_t)255;
    int32_t *keys = reinterpret_cast<int32_t *>(t + sort_bytes);
    int32_t *vals = reinterpret_cast<int32_t *>(t + sort_bytes + arr);
    k_iota<<<grid_for(nl), 256, 0, st>>>(vals, nl);
    size_t sb = sort_bytes;
    if (nl > 0 &&
        cuda_check(cub::DeviceRadixSort::SortPairs(t, sb, l2g, keys, vals, ci, (int)nl, 0, 32, st),
                   "sb_build_gather_general: radix sort"))
        return SB_E_CUDA;
    k_stats_init<<<1, 1, 0, st>>>(stats);
    k_row_bounds<<<grid_for(ng + 1), 256, 0, st>>>(keys, nl, ng, rs, stats);
    return launch_check("sb_build_gather_general");
}

int sb_histogram(const int32_t *ids, int64_t n, int64_t ng, double *out, sb_stream_t s) {
    using namespace sb;
    clear_error();
    if (n < 0 || ng < 0 || !out || (n > 0 && !ids)) {
        set_error("sb_histogram: invalid arguments");
        return SB_E_INVALID;
    }
    cudaStream_t st = as_stream(s);
    if (cuda_check(cudaMemsetAsync(out, 0, sizeof(double) * (size_t)ng, st), "sb_histogram")) return SB_E_CUDA;
    if (n > 0) k_histogram<<<grid_for(n), 256, 0, st>>>(ids, n, out);
    return launch_check("sb_histogram");
}

}  // extern "C"
