// sb_gs_tile.cu -- BS6 gather for p = 1 over row-line tiles, with the q
// gathers in structure order (gs.py:10-39; bitwise the reference: every row
// is summed in ascending column order from +0.0, or the carry-in, by one
// thread).
//
// Why.  The super-block kernels (sb_gs_pipe.cu) gather q in CSR order: a
// warp instruction covers 32 consecutive entries = 4 rows x 8 columns, which
// at p = 1 come from 4 element runs x ~5 elements, i.e. ~14 distinct 128 B
// lines -- one L1 tag lookup each.  That L1 work, not HBM, bounds them at
// N = 1 (ncu: l1tex 84%, DRAM 59%; 0.73 of the copy peak).
//
// Here a CTA takes a tile of <= 128 consecutive rows of ONE row line (b, c)
// of the lattice (mesh.py:73-97 numbering).  Those rows read exactly 4
// element runs (ey, ez) in {b-1, b} x {c-1, c}, and from each element of a
// run one aligned 16 B pair of nodes (i = 0, 1): node i=0 is entry j = 2r+1
// of row ex, node i=1 entry j = 2r of row ex+1 (r = run, j = dz*4 + dy*2 + dx).
// So lane u loads the pair of element u>>2 of run u&3 with one 16 B load --
// 8 lines per 64 entries instead of ~28 -- at an address computed from the
// tile alone, i.e. issued before the tile's indices have even arrived.
// Those values are only USED if the tile's row starts and column ids equal
// the closed form (one compare per entry against the coalesced col_ids
// stream, which is read as before); any other operator takes the CSR-order
// gather in the same kernel, so results are right for ANY CSR with these
// rows.  Row sums: the value tile + one thread per row, as in sb_gs_pipe.cu.
#include <limits.h>

#include <algorithm>

#include "sb_common.cuh"

namespace sb {

namespace {

constexpr int kTlT = 128;    // threads = max rows per tile
constexpr int kTlCap = 1024; // max entries per tile (128 rows x 8)
constexpr int kTlE = kTlCap / kTlT;
constexpr int kTlPairs = (4 * (kTlT + 1) + kTlT - 1) / kTlT;  // 16 B loads per thread (4 runs x 129 elements)

struct TlGeom {
    int K, z0, z1, c_lo, c_hi, g;
    int na;            // tiles per row line
    int ch;            // row planes per item (z chunk)
    int n_items;       // columns (ta, b) x z chunks; a CTA walks an item's planes in order
};

struct TlTile {
    int a0, n, b, c;   // rows a in [a0, a0 + n) of row line (b, c)
    int64_t r0;        // first row (operator numbering)
    bool structured;   // interior row line: four element runs present
    bool valid;
};

// A CTA's tile sequence: items blockIdx.x + k * gridDim.x, each a column of
// tiles (ta, b) walked along c -- consecutive tiles of a CTA are z-neighbours
// (the elements of plane c are read at c and again at c+1: the second read
// hits L2), and CTAs with neighbouring item numbers hold the y-neighbours
// at about the same c.
struct TlCursor {
    int item, ta, b, c, c1;
    __device__ __forceinline__ void set(const TlGeom &G, int it) {
        item = it;
        if (it < G.n_items) {
            const int col = it % (G.na * G.g), chunk = it / (G.na * G.g);
            ta = col % G.na;
            b = col / G.na;
            c = G.c_lo + chunk * G.ch;
            c1 = min(G.c_hi, c + G.ch);
        }
    }
    __device__ __forceinline__ void next(const TlGeom &G) {
        if (item >= G.n_items) return;
        if (++c >= c1) set(G, item + (int)gridDim.x);
    }
};

__device__ __forceinline__ TlTile tl_tile(const TlGeom &G, const TlCursor &C) {
    TlTile T;
    T.valid = C.item < G.n_items;
    T.b = C.b;
    T.c = C.c;
    T.a0 = C.ta * kTlT;
    T.n = min(kTlT, G.g - T.a0);
    T.r0 = ((int64_t)(T.c - G.c_lo) * G.g + T.b) * G.g + T.a0;
    T.structured = T.valid && T.b >= 1 && T.b <= G.g - 2 && T.c - 1 >= G.z0 && T.c <= G.z1 - 1;
    return T;
}

// Closed-form position of entry j (0..7) of tile row rho: its offset from the
// tile's first entry and whether the row has all 8 entries (x-edge rows a = 0
// and a = g-1 have the 4 entries dx = 1 resp. dx = 0).
struct TlShape {
    bool first, last;
    int s0, r1, nfull, ne;
    __device__ __forceinline__ TlShape(const TlTile &T, int g) {
        first = T.a0 == 0;
        last = T.a0 + T.n == g;
        s0 = first ? 4 : 0;
        r1 = first ? 1 : 0;
        nfull = T.n - r1 - (last ? 1 : 0);
        ne = s0 + 8 * nfull + (last ? 4 : 0);
    }
    __device__ __forceinline__ int start(int rho) const { return (first && rho == 0) ? 0 : s0 + 8 * (rho - r1); }
};

// column of entry j of row a0 + rho (closed form; B0 = entry 0 of row a0)
__device__ __forceinline__ int tl_col(int B0, int rho, int j, int ystride, int zstride) {
    return B0 + 8 * rho + ((j >> 2) & 1) * (zstride - 4) + ((j >> 1) & 1) * (ystride - 2) + (j & 1) * 7;
}

// Staging layout of one tile: run r (0..3) at r * kTlRun doubles, element e
// of the run (ex = xlo + e) at 2 e: its node pair (i = 0, 1).  Row rho reads
// entry j at run j >> 1, element rho + (j & 1) + sh, node 1 - (j & 1): with
// the lanes of a warp on consecutive rows the addresses step by 2 doubles,
// i.e. 2 wavefronts per warp read (conflict-free).
constexpr int kTlRun = 2 * (kTlT + 1) + 2;  // 260 doubles (+2: runs on distinct 16 B phases)
constexpr int kTlStage = 4 * kTlRun;
constexpr int kTlBufs = 3;                  // staged two tiles ahead

__device__ __forceinline__ void tl_stage(const TlGeom &G, const TlTile &T, const double *__restrict__ q,
                                         double *stg) {
    if (!T.structured) return;
    const int t = threadIdx.x;
    const int ystride = G.K * 8, zstride = G.K * ystride;
    const int xlo = max(T.a0 - 1, 0);
    const int nel = min(T.a0 + T.n - 1, G.K - 1) - xlo + 1;
    const int64_t cbase = ((((int64_t)(T.c - 1 - G.z0) * G.K + (T.b - 1)) * G.K) + xlo) * 8;
#pragma unroll
    for (int i = 0; i < kTlPairs; i++) {
        const int u = t + i * kTlT, r = u & 3, e = u >> 2;
        if (e < nel) {
            // run r = (dz, dy) = (r >> 1, r & 1): element (xlo + e, b-1+dy, c-1+dz),
            // node pair (i = 0, 1) at j = 1-dy, k = 1-dz
            const int64_t off = cbase + (r >> 1) * (int64_t)zstride + (r & 1) * ystride + e * 8 +
                                (1 - (r >> 1)) * 4 + (1 - (r & 1)) * 2;
            cp_async16(stg + r * kTlRun + 2 * e, q + off);
        }
    }
}

template <int MINB>
__global__ void __launch_bounds__(kTlT, MINB)
    k_bs6_tile1(TlGeom G, const int32_t *__restrict__ rs, const int32_t *__restrict__ ci,
                const double *__restrict__ q, double *__restrict__ out, const double *__restrict__ carry,
                int64_t ncarry) {
    extern __shared__ __align__(16) double stg_all[];
    const int t = threadIdx.x;
    const int ystride = G.K * 8, zstride = G.K * ystride;
    if ((int)blockIdx.x >= G.n_items) return;
    // pipeline: q pairs staged two tiles ahead (cp.async), row starts and
    // column ids one tile ahead (registers), entry ranges two tiles ahead
    TlCursor C;
    C.set(G, (int)blockIdx.x);
    TlTile T = tl_tile(G, C);
    C.next(G);
    TlTile T1 = tl_tile(G, C);
    C.next(G);  // C: two tiles ahead of T from here on
    tl_stage(G, T, q, stg_all);
    cp_async_commit();
    if (T1.valid) tl_stage(G, T1, q, stg_all + kTlStage);
    cp_async_commit();
    int e0 = __ldg(rs + T.r0), e1 = __ldg(rs + T.r0 + T.n);
    int f0 = 0, f1 = 0;  // entry range of tile + 1
    if (T1.valid) {
        f0 = __ldg(rs + T1.r0);
        f1 = __ldg(rs + T1.r0 + T1.n);
    }
    int col[kTlE];
#pragma unroll
    for (int j = 0; j < kTlE; j++)
        if (t + j * kTlT < e1 - e0) col[j] = ld_stream(ci + e0 + t + j * kTlT);
    int lo = t <= T.n ? ld_stream(rs + T.r0 + t) : 0;
    int buf = 0;
    while (T.valid) {
        __syncthreads();  // (A) the buffer staged below was last read two tiles ago
        const TlTile T2 = tl_tile(G, C);
        C.next(G);
        if (T2.valid) tl_stage(G, T2, q, stg_all + ((buf + 2) % kTlBufs) * kTlStage);
        cp_async_commit();
        // verify this tile against the closed form (row starts + columns)
        const TlShape S(T, G.g);
        const int ne = e1 - e0;
        const int xlo = max(T.a0 - 1, 0);
        bool ok = T.structured && ne == S.ne && ne <= kTlCap;
        if (ok) {
            const int B0 = (int)(((((int64_t)(T.c - 1 - G.z0) * G.K + (T.b - 1)) * G.K) + T.a0 - 1) * 8 + 7);
            if (t < T.n) ok = ok && lo - e0 == S.start(t);
            // entry k = t + 128 j: row r1 + (k - s0) >> 3, entry (k - s0) & 7 = jl
            // (lane-constant), i.e. column X + 128 j -- except at most one
            // entry per thread: row 0's (k < 4, entries 2k+1) or the last
            // row's (the tile's last 4 entries, entries 2m)
            const int jl = (t - S.s0) & 7;
            const int X = tl_col(B0, S.r1 + ((t - S.s0) >> 3), jl, ystride, zstride);
            int jfix = -1, want_fix = 0;
            if (S.first && t < 4) {
                jfix = 0;
                want_fix = tl_col(B0, 0, 2 * t + 1, ystride, zstride);
            }
            if (S.last) {
                const int m = (t - (ne - 4)) & (kTlT - 1);  // k = ne - 4 + m, k = t (mod 128)
                if (m < 4) {
                    jfix = (ne - 4 + m - t) / kTlT;
                    want_fix = tl_col(B0, S.r1 + S.nfull, 2 * m, ystride, zstride);
                }
            }
#pragma unroll
            for (int j = 0; j < kTlE; j++) {
                const int want = j == jfix ? want_fix : X + kTlT * j;
                if (t + j * kTlT < ne) ok = ok && col[j] == want;
            }
        }
        // this row's end (before lo is replaced by the next tile's)
        int hi = __shfl_down_sync(0xffffffffu, lo, 1);
        if (t < T.n && ((t & 31) == 31 || t == T.n - 1)) hi = __ldg(rs + T.r0 + t + 1);
        const int lo_cur = lo;
        // next tile's columns / row starts (registers freed by the compares),
        // and the entry range of the tile after it
        if (T1.valid) {
#pragma unroll
            for (int j = 0; j < kTlE; j++)
                if (t + j * kTlT < f1 - f0) col[j] = ld_stream(ci + f0 + t + j * kTlT);
            lo = t <= T1.n ? ld_stream(rs + T1.r0 + t) : 0;
        }
        int g0 = 0, g1 = 0;
        if (T2.valid) {
            g0 = __ldg(rs + T2.r0);
            g1 = __ldg(rs + T2.r0 + T2.n);
        }
        cp_async_wait<2>();                      // this tile's pairs (own copies) ...
        const bool fast = __syncthreads_and(ok);  // (B) ... everyone's, and the vote
        if (t < T.n) {
            const int64_t r = T.r0 + t;
            double acc = r < ncarry ? carry[r] : 0.0;
            if (fast) {
                // entry j: run j >> 1, element rho + (j & 1) + sh, node 1 - (j & 1)
                const double *row = stg_all + buf * kTlStage + 2 * (t + (T.a0 - 1 - xlo)) + 1;
                const bool no_dx0 = S.first && t == 0, no_dx1 = S.last && t == T.n - 1;
#pragma unroll
                for (int j = 0; j < 8; j++) {
                    const bool dx = j & 1;
                    if (!(dx ? no_dx1 : no_dx0)) acc = add(acc, row[(j >> 1) * kTlRun + (j & 1)]);
                }
            } else {  // any other CSR (or an oversize tile): straight from global memory
#pragma unroll 1
                for (int k = lo_cur; k < hi; k++) acc = add(acc, __ldg(q + __ldg(ci + k)));
            }
            st_stream(out + r, acc);
        }
        buf = (buf + 1) % kTlBufs;
        T = T1;
        T1 = T2;
        e0 = f0;
        e1 = f1;
        f0 = g0;
        f1 = g1;
    }
}

}  // namespace
}  // namespace sb

using namespace sb;

extern "C" {

int sb_bs6_gather_tiled(int32_t K, int32_t p, int32_t z0, int32_t z1, int32_t c_lo, int32_t c_hi,
                        const int32_t *row_starts, const int32_t *col_ids, int64_t ng, int64_t nl,
                        const double *q_local, double *out, const double *carry_in, int64_t n_carry,
                        sb_stream_t stream) {
    clear_error();
    const int64_t g = (int64_t)K * p + 1;
    if (K < 1 || p != 1 || z0 < 0 || z1 > K || z0 >= z1 || c_lo < 0 || c_hi > g || c_lo >= c_hi) {
        set_error("sb_bs6_gather_tiled: invalid geometry (K=%d p=%d z=[%d,%d) c=[%d,%d); p must be 1)", K, p, z0, z1,
                  c_lo, c_hi);
        return SB_E_INVALID;
    }
    if (ng != (int64_t)(c_hi - c_lo) * g * g || nl != (int64_t)K * K * (z1 - z0) * 8 || nl > INT_MAX ||
        n_carry < 0 || (n_carry > 0 && !carry_in) || !row_starts || !col_ids || !q_local || !out) {
        set_error("sb_bs6_gather_tiled: invalid arguments (ng=%lld nl=%lld do not match the geometry)",
                  (long long)ng, (long long)nl);
        return SB_E_INVALID;
    }
    if (!aligned16(q_local)) {
        set_error("sb_bs6_gather_tiled: q_local must be 16-byte aligned");
        return SB_E_INVALID;
    }
    if (n_carry > ng) n_carry = ng;
    TlGeom G{};
    G.K = K;
    G.z0 = z0;
    G.z1 = z1;
    G.c_lo = c_lo;
    G.c_hi = c_hi;
    G.g = (int)g;
    G.na = (int)((g + kTlT - 1) / kTlT);
    const int64_t ncols = (int64_t)G.na * g, nc = c_hi - c_lo;
    const auto k = k_bs6_tile1<8>;
    const size_t smem = (size_t)kTlBufs * kTlStage * sizeof(double);
    int rc = cuda_check(cudaFuncSetAttribute((const void *)k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                        "sb_bs6_gather_tiled: shared memory");
    if (rc) return rc;
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void *)k, kTlT, smem);
    const int64_t grid_max = (int64_t)sm_count() * std::max(1, per_sm);
    // z chunks: about 8 items per resident CTA (tail balance)
    int64_t nch = std::max<int64_t>(1, std::min<int64_t>(nc, (8 * grid_max + ncols - 1) / ncols));
    G.ch = (int)((nc + nch - 1) / nch);
    nch = (nc + G.ch - 1) / G.ch;
    if (ncols * nch > INT_MAX) {
        set_error("sb_bs6_gather_tiled: too many tiles");
        return SB_E_RANGE;
    }
    G.n_items = (int)(ncols * nch);
    const int64_t grid = std::min<int64_t>(G.n_items, grid_max);
    k<<<(unsigned)grid, kTlT, smem, as_stream(stream)>>>(G, row_starts, col_ids, q_local, out, carry_in, n_carry);
    return launch_check("sb_bs6_gather_tiled");
}

}  // extern "C"
