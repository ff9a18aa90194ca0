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
#include <cuda.h>
#include <cudaTypedefs.h>
#include <limits.h>
#include <stdlib.h>

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

// ---- 32 x 4 tiles: four row lines per CTA (one per warp) ------------------
// Element (ex, ey, ez)'s 64 B are two 32 B sectors, one per k (z) half; each
// sector holds the four (j, i) nodes of that half, j (y) = 0 / 1 going to row
// lines ey / ey+1.  A tile of 4 consecutive row lines b0..b0+3 at plane c
// therefore reads the k = 1 half of plane c-1 and the k = 0 half of plane c
// of element rows ey = b0-1 .. b0+3, and uses the inner three of those rows'
// sectors completely (the one-row tiles above used every sector half, so L2
// delivered 2x the useful bytes).  Staging plane pl = dz*8 + 2*ey3 + jn - 1
// (ey3 = ey - (b0-1); edge rows hold one j half) keeps element e's node pair
// at 2e: warp w (row line b0+w) reads entry j of row a0+lane at plane
// dz*8 + 2w + dy, double 2(lane + sh) + dx + 1 -- consecutive lanes 2
// doubles apart, conflict-free.  Each warp verifies its own row line against
// the closed form (as the z-sweep kernel does) and otherwise sums its rows
// from global memory; one CTA barrier per tile publishes the staged pairs.
constexpr int kT4W = 32;
constexpr int kT4Plane = 2 * (kT4W + 1) + 2;  // 68 doubles: 33 pairs + pad (16 B multiple)
template <int H>
constexpr int t4_stage_d() { return 4 * H * kT4Plane; }  // doubles per stage: 4H planes
constexpr int kT4E = 8;  // column indices per lane (256 per warp-step)

struct T4Geom {
    int K, z0, z1, c_lo, c_hi, g;
    int na, nb;        // tiles along x (32 rows), along y (4 row lines)
    int ch;            // row planes per item
    int n_items;
};

struct T4Cursor {
    int item, ta, tb, c, c1;
    __device__ __forceinline__ void set(const T4Geom &G, int it) {
        item = it;
        if (it < G.n_items) {
            const int col = it % (G.na * G.nb), chunk = it / (G.na * G.nb);
            ta = col % G.na;
            tb = col / G.na;
            c = G.c_lo + chunk * G.ch;
            c1 = min(G.c_hi, c + G.ch);
        }
    }
    __device__ __forceinline__ void next(const T4Geom &G) {
        if (item >= G.n_items) return;
        if (++c >= c1) set(G, item + (int)gridDim.x);
    }
};

struct T4Tile {
    int a0, n, b0, c;
    bool valid;
};

template <int H>
__device__ __forceinline__ T4Tile t4_tile(const T4Geom &G, const T4Cursor &C) {
    T4Tile T;
    T.valid = C.item < G.n_items;
    T.a0 = C.ta * kT4W;
    T.n = min(kT4W, G.g - T.a0);
    T.b0 = C.tb * H;
    T.c = C.c;
    return T;
}

// cp.async the tile's element-row halves into one stage (chunks of 16 B)
template <int H>
__device__ __forceinline__ void t4_stage(const T4Geom &G, const T4Tile &T, const double *__restrict__ q,
                                         double *stg) {
    const int xlo = max(T.a0 - 1, 0);
    const int nel = min(T.a0 + T.n - 1, G.K - 1) - xlo + 1;
    const int zplane = G.K * G.K * 8;  // (nl < 2^31: 32-bit offsets)
    // chunk u: plane pl = u % 4H = dz*2H + 2*ey3 + jn - 1, element e = u / 4H;
    // node pair (i = 0, 1) at j = jn, k = 1 - dz of element (xlo + e, b0-1+ey3, c-1+dz)
    const int base = (T.c - 1 - G.z0) * zplane + ((T.b0 - 1) * G.K + xlo) * 8;
    const bool inner = T.b0 >= 1 && T.b0 + H - 1 <= G.K - 1 && T.c - 1 >= G.z0 && T.c <= G.z1 - 1;
    for (int u = threadIdx.x; u < 4 * H * nel; u += H * 32) {
        const int pl = u % (4 * H), e = u / (4 * H);
        const int dz = pl / (2 * H), pp = pl % (2 * H) + 1, ey3 = pp >> 1, jn = pp & 1;
        if (!inner) {
            const int ey = T.b0 - 1 + ey3, ez = T.c - 1 + dz;
            if (ey < 0 || ey > G.K - 1 || ez < G.z0 || ez > G.z1 - 1) continue;
        }
        const int off = base + dz * zplane + (ey3 * G.K + e) * 8 + (1 - dz) * 4 + jn * 2;
        cp_async16(stg + pl * kT4Plane + 2 * e, q + off);
    }
}

// Warp w reads exactly the four planes dz*8 + 2w + dy (its row line's runs
// ey = b0-1+w+dy with j-half 1-dy), and no other warp reads them: so each
// warp stages its own four planes (local plane lp = dz*2 + dy) into a
// private ring and needs no CTA barrier -- the warps of a CTA run
// independent pipelines.
__device__ __forceinline__ void t4_stage_warp(const T4Geom &G, const T4Tile &T, int w, int lane,
                                              const double *__restrict__ q, double *stg) {
    if (T.b0 + w >= G.g) return;
    const int xlo = max(T.a0 - 1, 0);
    const int nel = min(T.a0 + T.n - 1, G.K - 1) - xlo + 1;
    const int zplane = G.K * G.K * 8;
    const int base = (T.c - 1 - G.z0) * zplane + ((T.b0 - 1) * G.K + xlo) * 8;
    const bool inner = T.b0 + w >= 1 && T.b0 + w + 1 <= G.K - 1 && T.c - 1 >= G.z0 && T.c <= G.z1 - 1;
    for (int u = lane; u < 4 * nel; u += 32) {
        const int lp = u & 3, e = u >> 2;
        const int dz = lp >> 1, dy = lp & 1;
        const int ey3 = w + dy, jn = 1 - dy;
        if (!inner) {
            const int ey = T.b0 - 1 + ey3, ez = T.c - 1 + dz;
            if (ey < 0 || ey > G.K - 1 || ez < G.z0 || ez > G.z1 - 1) continue;
        }
        const int off = base + dz * zplane + (ey3 * G.K + e) * 8 + (1 - dz) * 4 + jn * 2;
        cp_async16(stg + lp * kT4Plane + 2 * e, q + off);
    }
}

// per-warp row data of one tile: column ids (8 per lane), the lane's row
// start, the row line's entry range (e0, end: loaded one tile earlier, so
// the column loads do not wait on them)
struct T4Rows {
    int col[kT4E];
    int lo, end, e0;
};

__device__ __forceinline__ int64_t t4_r0(const T4Geom &G, const T4Tile &T, int w) {
    return ((int64_t)(T.c - G.c_lo) * G.g + (T.b0 + w)) * G.g + T.a0;
}

__device__ __forceinline__ void t4_load_meta(const T4Geom &G, const T4Tile &T, int w,
                                             const int32_t *__restrict__ rs, int &e0, int &end) {
    e0 = end = 0;
    if (!T.valid || T.b0 + w >= G.g) return;
    const int64_t r0 = t4_r0(G, T, w);
    e0 = __ldg(rs + r0);
    end = __ldg(rs + r0 + T.n);
}

__device__ __forceinline__ void t4_load_rows(const T4Geom &G, const T4Tile &T, int w, int lane, int e0, int end,
                                             const int32_t *__restrict__ rs, const int32_t *__restrict__ ci,
                                             T4Rows &R) {
    R.e0 = e0;
    R.end = end;
    R.lo = 0;
    if (!T.valid || T.b0 + w >= G.g) return;
    R.lo = ld_stream(rs + t4_r0(G, T, w) + (lane < T.n ? lane : T.n));
    const int ne = end - e0;
#pragma unroll
    for (int j = 0; j < kT4E; j++)
        if (lane + 32 * j < ne) R.col[j] = ld_stream(ci + e0 + lane + 32 * j);
}

template <int H, int NB, int MINB, bool WS, bool PROBE = false>
__global__ void __launch_bounds__(H * 32, MINB)
    k_bs6_tile4(T4Geom G, const int32_t *__restrict__ rs, const int32_t *__restrict__ ci,
                const double *__restrict__ q, double *__restrict__ out, const double *__restrict__ carry,
                int64_t ncarry) {
    extern __shared__ __align__(16) double stg_all[];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ystride = G.K * 8, zstride = G.K * ystride;
    if ((int)blockIdx.x >= G.n_items) return;
    T4Cursor C;
    C.set(G, (int)blockIdx.x);
    T4Tile T = t4_tile<H>(G, C);
    C.next(G);
    T4Tile T1 = t4_tile<H>(G, C);
    C.next(G);  // C: two tiles ahead of T
    // stage buffers: CTA-shared (NB x 16 planes) or warp-private (per warp NB x 4 planes)
    double *stg = WS ? stg_all + w * (NB * 4 * kT4Plane) : stg_all;
    constexpr int SS = WS ? 4 * kT4Plane : t4_stage_d<H>();  // doubles per stage
    auto stage = [&](const T4Tile &X, double *dst) {
        if (WS)
            t4_stage_warp(G, X, w, lane, q, dst);
        else
            t4_stage<H>(G, X, q, dst);
    };
    stage(T, stg);
    cp_async_commit();
    if (T1.valid) stage(T1, stg + SS);
    cp_async_commit();
    T4Rows R;
    int m0, m1;  // entry range of tile + 1
    {
        int a0_, a1_;
        t4_load_meta(G, T, w, rs, a0_, a1_);
        t4_load_rows(G, T, w, lane, a0_, a1_, rs, ci, R);
    }
    t4_load_meta(G, T1, w, rs, m0, m1);
    int buf = 0;
    while (T.valid) {
        // the buffer staged below was last read NB-2 tiles ago: by this warp
        // only (WS), or -- with 3 buffers -- by any warp of the CTA
        if (WS)
            __syncwarp();
        else if (NB == 3)
            __syncthreads();
        const T4Tile T2 = t4_tile<H>(G, C);
        C.next(G);
        if (T2.valid) stage(T2, stg + ((buf + 2) % NB) * SS);
        cp_async_commit();
        // this warp's row line: verify against the closed form (z-sweep kernel's fast paths)
        const int b = T.b0 + w;
        const int nrows = b < G.g ? T.n : 0;
        const int ne = R.end - R.e0;
        const bool first = T.a0 == 0, last = T.a0 + T.n == G.g;
        const int xlo = max(T.a0 - 1, 0);
        bool ok = !PROBE && nrows > 0 && b >= 1 && b <= G.g - 2 && T.c - 1 >= G.z0 && T.c <= G.z1 - 1 &&
                  ne <= kT4E * 32;
        if (ok) {
            const int s0 = first ? 4 : 0, r1 = first ? 1 : 0;
            const int nfull = nrows - r1 - (last ? 1 : 0);
            ok = ne == s0 + 8 * nfull + (last ? 4 : 0);
            if (lane < nrows) ok = ok && R.lo - R.e0 == (lane == 0 && first ? 0 : s0 + 8 * (lane - r1));
            const int B0 = ((((T.c - 1 - G.z0) * G.K + (b - 1)) * G.K) + T.a0 - 1) * 8 + 7;
            const int jl = (lane - s0) & 7;
            const int X = tl_col(B0, r1 + ((lane - s0) >> 3), jl, ystride, zstride);
            if (!first && !last) {  // (warp-uniform) 32 rows of 8: column X + 32 j
#pragma unroll
                for (int j = 0; j < kT4E; j++) ok = ok && (lane + 32 * j >= ne || R.col[j] == X + 32 * j);
            } else {
#pragma unroll
                for (int j = 0; j < kT4E; j++) {
                    const int k = lane + 32 * j, kp = k - s0;
                    int want = X + 32 * j;
                    if (kp < 0)
                        want = tl_col(B0, 0, 2 * k + 1, ystride, zstride);
                    else if (kp >= 8 * nfull)
                        want = tl_col(B0, r1 + nfull, 2 * (kp - 8 * nfull), ystride, zstride);
                    ok = ok && (k >= ne || R.col[j] == want);
                }
            }
        }
        // (PROBE: an A/B measurement of the staging + row-sum traffic alone --
        // no index streams, results meaningless)
        const bool fast = PROBE ? nrows > 0 : __all_sync(0xffffffffu, ok);
        int hi = __shfl_down_sync(0xffffffffu, R.lo, 1);
        if (lane == nrows - 1) hi = R.end;
        const int lo = R.lo;
        // the next tile's row data (registers free after the compares), the
        // entry range of the tile after it
        if (!PROBE) {
            t4_load_rows(G, T1, w, lane, m0, m1, rs, ci, R);
            t4_load_meta(G, T2, w, rs, m0, m1);
        }
        cp_async_wait<2>();  // this tile's pairs (own copies) ...
        if (WS)
            __syncwarp();  // ... and the warp's
        else
            __syncthreads();  // ... and the CTA's
        if (lane < nrows) {
            const int64_t r = ((int64_t)(T.c - G.c_lo) * G.g + b) * G.g + T.a0 + lane;
            double acc = r < ncarry ? carry[r] : 0.0;
            if (fast) {
                const double *st = stg + buf * SS + (WS ? 0 : 2 * (w * kT4Plane)) + 2 * (lane + T.a0 - 1 - xlo) + 1;
                const bool no_dx0 = first && lane == 0, no_dx1 = last && lane == nrows - 1;
                // entry j = dz*4 + dy*2 + dx: plane dz*8 + 2w + dy, double 2(lane+sh) + dx + 1
#pragma unroll
                for (int j = 0; j < 8; j++) {
                    const int dz = j >> 2, dy = (j >> 1) & 1, dx = j & 1;
                    if (!(dx ? no_dx1 : no_dx0)) acc = add(acc, st[(WS ? dz * 2 + dy : dz * 2 * H + dy) * kT4Plane + dx]);
                }
            } else {  // any other CSR: straight from global memory
#pragma unroll 1
                for (int k = lo; k < hi; k++) acc = add(acc, __ldg(q + __ldg(ci + k)));
            }
            st_stream(out + r, acc);
        }
        buf = (buf + 1) % NB;
        T = T1;
        T1 = T2;
    }
}

// ---- 32 x 4 tiles staged by TMA tensor boxes ---------------------------------
// The cp.async staging above issues one 16 B request per lane, and L2 moves a
// full 32 B sector for each (ncu, probe kernel: 2.7x the useful q bytes L2 ->
// SM, L2 at 68%, DRAM at 54%).  Here one TMA box per k half does it: q seen as
// a 4-D tensor (node 8, ex K, ey K, ez nz), box (4 nodes = one 32 B sector,
// 33 elements, 5 element rows, 1 plane) at (4 kn, a0-1, b0-1, c-1+dz-z0) --
// out-of-range rows / planes / elements are zero-filled by the TMA unit, so
// edges need no special cases.  The box lands as [ey][ex][4 nodes] with the
// 32 B swizzle (16 B chunk bit 4 ^= bit 7): row-lane reads are 4-way
// conflicted (8-way unswizzled), the price of whole-sector transfers.
template <int H>
constexpr int t5_box() { return (H + 1) * 33 * 4; }  // doubles per box (H+1 element rows)
template <int H>
constexpr int t5_box_stride() { return (t5_box<H>() + 31) / 32 * 32; }  // 256 B aligned (the swizzle)
template <int H>
constexpr int t5_stage() { return 2 * t5_box_stride<H>(); }  // two k halves per tile

__device__ __forceinline__ void tma_load_4d(void *dst, const CUtensorMap *map, int c0, int c1, int c2, int c3,
                                            uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
        "[%6];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
        : "memory");
}

template <int NB, int MINB, bool RS_FIRST = false, int H = 4>
__global__ void __launch_bounds__(H * 32, MINB)
    k_bs6_tile4t(const __grid_constant__ CUtensorMap qmap, T4Geom G, const int32_t *__restrict__ rs,
                 const int32_t *__restrict__ ci, const double *__restrict__ q, double *__restrict__ out,
                 const double *__restrict__ carry, int64_t ncarry) {
    constexpr int kT5Box = t5_box<H>(), kT5BoxStride = t5_box_stride<H>(), kT5Stage = t5_stage<H>();
    extern __shared__ __align__(16) unsigned char smem5[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem5);
    // boxes on 256 B boundaries (the 32 B swizzle pattern repeats every 256 B)
    const uint32_t s0 = smem_u32(smem5) + 256;
    double *stg = reinterpret_cast<double *>(smem5 + 256 + ((256 - (s0 & 255)) & 255));
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ystride = G.K * 8, zstride = G.K * ystride;
    if ((int)blockIdx.x >= G.n_items) return;
    if (threadIdx.x == 0) {
        for (int b = 0; b < NB; b++) mbar_init(&full[b], 1);
        fence_mbar_init();
    }
    __syncthreads();
    auto stage = [&](const T4Tile &X, int b) {  // thread 0: both k-half boxes of tile X into buffer b
        mbar_arrive_expect_tx(&full[b], 2u * kT5Box * 8u);
        for (int dz = 0; dz < 2; dz++)
            tma_load_4d(stg + b * kT5Stage + dz * kT5BoxStride, &qmap, 4 * (1 - dz), X.a0 - 1, X.b0 - 1,
                        X.c - 1 + dz - G.z0, &full[b]);
    };
    T4Cursor C;
    C.set(G, (int)blockIdx.x);
    T4Tile T = t4_tile<H>(G, C);
    C.next(G);
    T4Tile T1 = t4_tile<H>(G, C);
    C.next(G);
    if (threadIdx.x == 0) {
        stage(T, 0);
        if (T1.valid) stage(T1, 1);
    }
    T4Rows R;
    int m0, m1;
    {
        int a0_, a1_;
        t4_load_meta(G, T, w, rs, a0_, a1_);
        t4_load_rows(G, T, w, lane, a0_, a1_, rs, ci, R);
    }
    t4_load_meta(G, T1, w, rs, m0, m1);
    int step = 0;
    while (T.valid) {
        const int buf = step % NB;
        const T4Tile T2 = t4_tile<H>(G, C);
        C.next(G);
        // buffer (step+2) % NB was last read at step+2-NB <= step-1: every warp
        // is past those reads (the barrier closing the previous step)
        if (threadIdx.x == 0 && T2.valid) stage(T2, (step + 2) % NB);
        const int b = T.b0 + w;
        const int nrows = b < G.g ? T.n : 0;
        const int ne = R.end - R.e0;
        const bool first = T.a0 == 0, last = T.a0 + T.n == G.g;
        bool ok = nrows > 0 && b >= 1 && b <= G.g - 2 && T.c - 1 >= G.z0 && T.c <= G.z1 - 1 && ne <= kT4E * 32;
        if (ok) {
            const int s0 = first ? 4 : 0, r1 = first ? 1 : 0;
            const int nfull = nrows - r1 - (last ? 1 : 0);
            ok = ne == s0 + 8 * nfull + (last ? 4 : 0);
            if (lane < nrows) ok = ok && R.lo - R.e0 == (lane == 0 && first ? 0 : s0 + 8 * (lane - r1));
            const int B0 = ((((T.c - 1 - G.z0) * G.K + (b - 1)) * G.K) + T.a0 - 1) * 8 + 7;
            const int jl = (lane - s0) & 7;
            const int X = tl_col(B0, r1 + ((lane - s0) >> 3), jl, ystride, zstride);
            if (!first && !last) {
#pragma unroll
                for (int j = 0; j < kT4E; j++) ok = ok && (lane + 32 * j >= ne || R.col[j] == X + 32 * j);
            } else {
#pragma unroll
                for (int j = 0; j < kT4E; j++) {
                    const int k = lane + 32 * j, kp = k - s0;
                    int want = X + 32 * j;
                    if (kp < 0)
                        want = tl_col(B0, 0, 2 * k + 1, ystride, zstride);
                    else if (kp >= 8 * nfull)
                        want = tl_col(B0, r1 + nfull, 2 * (kp - 8 * nfull), ystride, zstride);
                    ok = ok && (k >= ne || R.col[j] == want);
                }
            }
        }
        const bool fast = __all_sync(0xffffffffu, ok);
        int hi = __shfl_down_sync(0xffffffffu, R.lo, 1);
        if (lane == nrows - 1) hi = R.end;
        const int lo = R.lo;
        if (RS_FIRST) {
            // the next tile's row data after this tile's sums (A/B: see below)
        } else {
            t4_load_rows(G, T1, w, lane, m0, m1, rs, ci, R);
            t4_load_meta(G, T2, w, rs, m0, m1);
        }
        mbar_wait(&full[buf], (uint32_t)((step / NB) & 1));  // this tile's boxes have landed
        if (lane < nrows) {
            const int64_t r = ((int64_t)(T.c - G.c_lo) * G.g + b) * G.g + T.a0 + lane;
            double acc = r < ncarry ? carry[r] : 0.0;
            if (fast) {
                // entry j = dz*4 + dy*2 + dx: box dz, element row w+dy, element
                // lane+dx (the box starts at ex = a0-1), node (1-dy)*2 + (1-dx)
                const unsigned char *box = reinterpret_cast<const unsigned char *>(stg + buf * kT5Stage);
                const bool no_dx0 = first && lane == 0, no_dx1 = last && lane == nrows - 1;
                const int base = (w * 33 + lane) * 32;
#pragma unroll
                for (int j = 0; j < 8; j++) {
                    const int dz = j >> 2, dy = (j >> 1) & 1, dx = j & 1;
                    int off = base + dy * 33 * 32 + dx * 32 + ((1 - dy) * 2 + (1 - dx)) * 8;
                    off ^= ((off >> 7) & 1) << 4;  // the 32 B swizzle
                    const double v = *reinterpret_cast<const double *>(box + dz * kT5BoxStride * 8 + off);
                    if (!(dx ? no_dx1 : no_dx0)) acc = add(acc, v);
                }
            } else {
#pragma unroll 1
                for (int k = lo; k < hi; k++) acc = add(acc, __ldg(q + __ldg(ci + k)));
            }
            st_stream(out + r, acc);
        }
        if (RS_FIRST) {
            t4_load_rows(G, T1, w, lane, m0, m1, rs, ci, R);
            t4_load_meta(G, T2, w, rs, m0, m1);
        }
        __syncthreads();  // the buffer read above may be refilled from the next step on
        step++;
        T = T1;
        T1 = T2;
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
    // A/B: "1" = one-row-line tiles, "3b" = 3 stage buffers / 8 CTAs per SM
    // (4 buffers / 6 CTAs per SM by default: measured 4,776 vs 4,593 GB/s at N=1)
    const char *kv = getenv("SB200_BS6_TILE_KERNEL");
    if (!kv || kv[0] == 't') {
        static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
        if (!encode) {
            cudaDriverEntryPointQueryResult qr;
            void *fn = nullptr;
            if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr) != cudaSuccess ||
                qr != cudaDriverEntryPointSuccess || !fn) {
                (void)cudaGetLastError();
                set_error("sb_bs6_gather_tiled: cuTensorMapEncodeTiled unavailable");
                return SB_E_CUDA;
            }
            encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
        }
        CUtensorMap map;
        const cuuint64_t dims[4] = {8, (cuuint64_t)K, (cuuint64_t)K, (cuuint64_t)(z1 - z0)};
        const cuuint64_t strides[3] = {64, 64ull * K, 64ull * K * K};
        // default: 8 row lines per CTA (t8: 9-row boxes, 3 buffers, 3 CTAs/SM) -- measured best
        const bool h16 = kv && kv[1] == '6', h8 = !h16 && !(kv && (kv[1] == '3' || kv[1] == '4' || kv[1] == 's'));
        const int ry = h16 ? 16 : h8 ? 8 : 4;
        const cuuint32_t box[4] = {4, 33, (cuuint32_t)ry + 1, 1}, estr[4] = {1, 1, 1, 1};
        // (L2 promotion none / 64 / 128 / 256 B measured within 2%: 5,627-5,774 GB/s, DRAM 10.42-10.45 GB)
        const CUtensorMapL2promotion promo = CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
        if (encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double *>(q_local), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B, promo,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
            set_error("sb_bs6_gather_tiled: tensor map encoding failed");
            return SB_E_INVALID;
        }
        T4Geom H{};
        H.K = K;
        H.z0 = z0;
        H.z1 = z1;
        H.c_lo = c_lo;
        H.c_hi = c_hi;
        H.g = (int)g;
        H.na = (int)((g + kT4W - 1) / kT4W);
        H.nb = (int)((g + ry - 1) / ry);
        // variants (A/B, SB200_BS6_TILE_KERNEL): t8 (default) 8 row lines per CTA
        // (9-row boxes), 3 buffers / 3 CTAs per SM; t3: 4 row lines, 3 buffers / 6 per SM;
        // t4: 4 buffers / 5 per SM; ts: t3 with the row sums before the next tile's loads
        const bool nb3 = !(kv && kv[1] == '4');
        const bool rsf = kv && kv[1] == 's';
        using K5 = void (*)(const CUtensorMap, T4Geom, const int32_t *, const int32_t *, const double *, double *,
                            const double *, int64_t);
        const K5 k5 = h16 ? k_bs6_tile4t<3, 2, false, 16> : h8 ? k_bs6_tile4t<3, 3, false, 8>
                         : rsf ? k_bs6_tile4t<3, 6, true> : nb3 ? k_bs6_tile4t<3, 6> : k_bs6_tile4t<4, 5>;
        const size_t stage_d = h16 ? t5_stage<16>() : h8 ? t5_stage<8>() : t5_stage<4>();
        const size_t smem5 = 256 + (size_t)(nb3 ? 3 : 4) * stage_d * sizeof(double) + 256;  // (+ alignment slack)
        int rc5 = cuda_check(cudaFuncSetAttribute((const void *)k5, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  (int)smem5), "sb_bs6_gather_tiled: shared memory");
        if (rc5) return rc5;
        int per5 = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per5, (const void *)k5, ry * 32, smem5);
        const int64_t gmax = (int64_t)sm_count() * std::max(1, per5);
        const int64_t ncols5 = (int64_t)H.na * H.nb, nc5 = c_hi - c_lo;
        // z chunks: about 32 work items per resident CTA -- shorter items keep
        // the CTAs' z sweeps closer together (the halo boxes the neighbouring
        // columns re-read stay in L2) and balance the tail: N=1 (K=463)
        // 5,922-5,946 GB/s vs 5,766-5,789 with 8 items, +3-8% at K=200..400
        // (SB200_BS6_TILE_WAVES overrides; A/B)
        const char *we = getenv("SB200_BS6_TILE_WAVES");
        const int64_t waves = we && atoi(we) > 0 ? atoi(we) : 32;
        int64_t nch5 = std::max<int64_t>(1, std::min<int64_t>(nc5, (waves * gmax + ncols5 - 1) / ncols5));
        H.ch = (int)((nc5 + nch5 - 1) / nch5);
        nch5 = (nc5 + H.ch - 1) / H.ch;
        if (ncols5 * nch5 > INT_MAX) {
            set_error("sb_bs6_gather_tiled: too many tiles");
            return SB_E_RANGE;
        }
        H.n_items = (int)(ncols5 * nch5);
        const int64_t grid5 = std::min<int64_t>(H.n_items, gmax);
        k5<<<(unsigned)grid5, ry * 32, smem5, as_stream(stream)>>>(map, H, row_starts, col_ids, q_local, out, carry_in,
                                                              n_carry);
        return launch_check("sb_bs6_gather_tiled");
    }
    if (kv[0] != '1') {
        T4Geom H{};
        H.K = K;
        H.z0 = z0;
        H.z1 = z1;
        H.c_lo = c_lo;
        H.c_hi = c_hi;
        H.g = (int)g;
        H.na = (int)((g + kT4W - 1) / kT4W);
        // variants (A/B): 4b (default) 4 row lines, 4 CTA-shared buffers, 6 CTAs/SM;
        // 3b: 3 buffers, 8/SM; w4 / w3: warp-private buffers; h8: 8 row lines, 3 buffers, 4/SM
        const bool h8 = kv && kv[0] == 'h';
        const bool four = !h8 && !(kv && (kv[0] == '3' || (kv[0] == 'w' && kv[1] == '3')));
        const bool ws = kv && kv[0] == 'w';
        const int rows_y = h8 ? 8 : 4;
        H.nb = (int)((g + rows_y - 1) / rows_y);
        using K4 = void (*)(T4Geom, const int32_t *, const int32_t *, const double *, double *, const double *,
                            int64_t);
        const bool probe = kv && kv[0] == 'p';
        const K4 k4 = probe ? k_bs6_tile4<4, 4, 6, false, true> : h8 ? k_bs6_tile4<8, 3, 4, false>
                         : ws ? (four ? k_bs6_tile4<4, 4, 6, true> : k_bs6_tile4<4, 3, 8, true>)
                              : (four ? k_bs6_tile4<4, 4, 6, false> : k_bs6_tile4<4, 3, 8, false>);
        const size_t smem4 = (size_t)(h8 ? 3 : (four ? 4 : 3)) * 4 * rows_y * kT4Plane * sizeof(double);
        int rc4 = cuda_check(cudaFuncSetAttribute((const void *)k4, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  (int)smem4), "sb_bs6_gather_tiled: shared memory");
        if (rc4) return rc4;
        int per_sm4 = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm4, (const void *)k4, rows_y * 32, smem4);
        const int64_t gmax = (int64_t)sm_count() * std::max(1, per_sm4);
        const int64_t ncols4 = (int64_t)H.na * H.nb, nc4 = c_hi - c_lo;
        int64_t nch4 = std::max<int64_t>(1, std::min<int64_t>(nc4, (8 * gmax + ncols4 - 1) / ncols4));
        H.ch = (int)((nc4 + nch4 - 1) / nch4);
        nch4 = (nc4 + H.ch - 1) / H.ch;
        if (ncols4 * nch4 > INT_MAX) {
            set_error("sb_bs6_gather_tiled: too many tiles");
            return SB_E_RANGE;
        }
        H.n_items = (int)(ncols4 * nch4);
        const int64_t grid4 = std::min<int64_t>(H.n_items, gmax);
        k4<<<(unsigned)grid4, rows_y * 32, smem4, as_stream(stream)>>>(H, row_starts, col_ids, q_local, out, carry_in,
                                                                       n_carry);
        return launch_check("sb_bs6_gather_tiled");
    }
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
