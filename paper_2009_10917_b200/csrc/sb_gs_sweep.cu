// sb_gs_sweep.cu -- BS6 gather for low polynomial orders (p <= 2) as a sweep
// along z over element planes staged in shared memory (gs.py:10-39; bitwise
// the reference: each row is summed in ascending column order from +0.0, or
// from the carry-in, by one thread).
//
// Why.  At p = 1 a row's 8 entries come from 8 different elements, so every
// 32-entry warp gather of the LSU kernels (sb_gs_pipe.cu) touches ~14
// distinct 128 B lines and the L1 tag / data pipe, not HBM, sets the speed
// (ncu at N=1: l1tex 84%, DRAM 59%).  Staging q in shared memory turns the
// gathers into shared-memory reads (2 wavefronts per warp instruction at
// p = 1: the four element runs a row line reads are bank-disjoint), but it
// only pays if the staging stays close to one read of q: the r02 tile kernel
// (removed; profiles/r02_bs6_staged.md) re-read every element run for each 2x2 patch of row lines
// (1.75x the algorithmic bytes through L2) and topped out at 2.9 TB/s.
//
// Here a CTA owns a column of rows -- W = 32 rows along x times H row lines
// along y -- and sweeps it along z.  Element plane ez (the nx x ny elements
// under the column: one contiguous run of q_local per ey) is copied into a
// ring slot ONCE by the producer thread (cp.async.bulk, mbarrier transaction
// count) and serves every row plane c it touches (p+1 of them); the only
// re-read is the one-element halo a column shares with its x / y neighbours
// ((W+1)(H+1)/(W H) ~ 1.16x of q at p = 1, H = 8), which the neighbouring
// CTAs of the same wave load at about the same time (L2 hits).  The producer
// also prefetches planes further ahead into L2 (cp.async.bulk.prefetch.L2)
// so the bytes in flight are not bounded by the ring.
//
// Consumer warp w takes row line b = b0 + w of every row plane c: lane = row
// for the row starts and the sums, lane = entry for the column loads (one
// coalesced 128 B line per 32 entries), software-pipelined: column indices
// one step ahead, row starts two steps ahead.  Each entry's column is matched
// against the <= 4 element runs (ey, ez) its row line can touch; a column
// outside them (an operator that is not the structured one) is read from
// global memory, so the result is right for ANY CSR with these rows -- the
// geometry only decides the speed.  A warp-step with more than 256 entries
// sums its rows straight from global memory.
//
// p = 2 (k_bs6_sweep2, the default there): rows have 1-8 entries, so the
// value tile costs more than it saves; each lane loads its own row's column
// ids, checks them against the closed form and sums straight from the staged
// runs (sw_step2).  SB200_BS6_SWEEP_ROW2=0 selects the p = 1 consumer.
#include <limits.h>
#include <stdlib.h>

#include <algorithm>

#include "sb_common.cuh"

namespace sb {

namespace {

constexpr int kSwW = 32;    // rows along x per column (lane = row)
constexpr int kSwVt = 256;  // value-tile entries per warp-step
constexpr int kSwMaxSlots = 8;
constexpr int kSwHdr = 256;  // bytes of mbarriers before the ring

struct SwGeom {
    int K, z0, z1, c_lo, c_hi, g;
    int na, nb;       // columns along x (W rows) and y (H row lines)
    int ch;           // row planes per item (z chunk)
    int64_t n_items;  // na * nb * ceil((c_hi - c_lo) / ch)
    int nslot;        // ring slots (element planes)
    int rs_d;         // run stride in doubles (multiple of 16: runs start on bank 0)
    int plane_d;      // slot stride in doubles
    int pfd;          // L2 prefetch distance in planes (0: off)
    int64_t nl;
};

// element range of lattice coordinate x (0 .. K*p) along one axis
template <int P>
__device__ __forceinline__ int el_lo(int x, int K) {
    const int e = (x % P == 0 && x > 0) ? x / P - 1 : x / P;
    return e < K - 1 ? e : K - 1;
}
template <int P>
__device__ __forceinline__ int el_hi(int x, int K) {
    const int e = x / P;
    return e < K - 1 ? e : K - 1;
}

template <bool SWZ>
__device__ __forceinline__ int vslot(int k) {
    return SWZ ? (k ^ ((k >> 4) & 15)) : k;
}

// One work item: the column (ta, tb) over the row planes [c0, c1) and the
// element planes [zf, zf + np) (global ez; slab-local numbering on use).
struct SwItem {
    int a0, a1, b0, c0, c1;
    int xlo, nx, ylo, ny, zf, np;
};

template <int P, int H>
__device__ __forceinline__ SwItem sw_item(const SwGeom &G, int64_t it) {
    SwItem I;
    const int ta = (int)(it % G.na);
    const int tb = (int)((it / G.na) % G.nb);
    const int tc = (int)(it / ((int64_t)G.na * G.nb));
    I.a0 = ta * kSwW;
    I.a1 = min(G.g, I.a0 + kSwW);
    I.b0 = tb * H;
    const int b1 = min(G.g, I.b0 + H);
    I.c0 = G.c_lo + tc * G.ch;
    I.c1 = min(G.c_hi, I.c0 + G.ch);
    I.xlo = el_lo<P>(I.a0, G.K);
    I.nx = el_hi<P>(I.a1 - 1, G.K) - I.xlo + 1;
    I.ylo = el_lo<P>(I.b0, G.K);
    I.ny = el_hi<P>(b1 - 1, G.K) - I.ylo + 1;
    I.zf = max(el_lo<P>(I.c0, G.K), G.z0);
    const int zl = min(el_hi<P>(I.c1 - 1, G.K), G.z1 - 1);
    I.np = zl >= I.zf ? zl - I.zf + 1 : 0;
    return I;
}

// q_local column of node 0 of element (ex, ey, ez) (slab-local numbering)
template <int P>
__device__ __forceinline__ int64_t sw_col(const SwGeom &G, int ex, int ey, int ez) {
    constexpr int N3 = (P + 1) * (P + 1) * (P + 1);
    return ((((int64_t)(ez - G.z0) * G.K + ey) * G.K) + ex) * N3;
}

__device__ __forceinline__ void bulk_prefetch_l2(const void *src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s_plain(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// Row geometry of warp w at one (item, c) step, for the look-ahead loads.
struct SwRows {
    int64_t r0;
    int n;  // rows (0: the row line lies past the mesh, or no step)
};

template <int P, int H>
struct SwCursor {
    int64_t it;
    int c, c1, a0, a1, b;
    __device__ __forceinline__ void set(const SwGeom &G, int64_t item, int w) {
        it = item;
        if (it < G.n_items) {
            const int ta = (int)(it % G.na);
            const int tb = (int)((it / G.na) % G.nb);
            const int tc = (int)(it / ((int64_t)G.na * G.nb));
            a0 = ta * kSwW;
            a1 = min(G.g, a0 + kSwW);
            b = tb * H + w;
            c = G.c_lo + tc * G.ch;
            c1 = min(G.c_hi, c + G.ch);
        }
    }
    __device__ __forceinline__ void next(const SwGeom &G, int w) {
        if (it >= G.n_items) return;
        if (++c >= c1) set(G, it + gridDim.x, w);
    }
    __device__ __forceinline__ SwRows rows(const SwGeom &G) const {
        SwRows R{0, 0};
        if (it < G.n_items && b < G.g) {
            R.r0 = ((int64_t)(c - G.c_lo) * G.g + b) * G.g + a0;
            R.n = a1 - a0;
        }
        return R;
    }
};

// Row starts of a warp-step go into the warp's ring of kSwRsSlots slots
// with cp.async (LDGSTS: no register waits on the load), issued three steps
// ahead: slot[l] = row start of row r0 + l (l < n; the end for l >= n),
// slot[32] = the end of the last row.  Every step commits one group.
constexpr int kSwRsSlots = 8, kSwRsStride = 40;

__device__ __forceinline__ void sw_issue_rs(const SwRows &R, const int32_t *__restrict__ rs, int lane, int *slot) {
    if (R.n > 0) {
        cp_async4(slot + lane, rs + R.r0 + (lane < R.n ? lane : R.n));
        if (lane == 0) cp_async4(slot + 32, rs + R.r0 + R.n);
    } else {
        slot[lane] = 0;
        if (lane == 0) slot[32] = 0;
    }
    cp_async_commit();
}

// L2 prefetch of a warp-step's column indices (<= 8 lines of 128 B)
__device__ __forceinline__ void sw_prefetch_cols(const int *slot, const int32_t *__restrict__ ci, int lane) {
    const int e0 = slot[0], ne = slot[32] - e0;
    if (lane * 32 < ne) asm volatile("prefetch.global.L2 [%0];" ::"l"(ci + e0 + lane * 32));
}

template <int E>
__device__ __forceinline__ void sw_load_cols(const int *slot, const int32_t *__restrict__ ci, int lane,
                                             int (&col)[E]) {
    const int e0 = slot[0];
    const int ne = slot[32] - e0;
#pragma unroll
    for (int j = 0; j < E; j++)
        if (lane + 32 * j < ne) col[j] = ld_stream(ci + e0 + lane + 32 * j);
}

// Consumer state of one warp: the current item / row plane and the plane
// sequence numbers it has waited for and released.
template <int P, int H>
struct SwState {
    SwItem I;
    int64_t it;
    int c;
    int base;            // sequence number of the item's first plane
    int waited, wslot;   // planes waited for (count), next slot to wait on
    uint32_t wph;        // its phase
    int released, rslot; // planes released (count), next slot to release
    int step;            // warp-steps done (row-start ring slot)
};

// One step (row plane c of the current item) of consumer warp `warp`.  Row
// starts arrive in the warp's smem ring four steps ahead (cp.async), the
// column indices of step + 2 are prefetched into L2 and those of step + 1
// loaded into colB; colA holds this step's (loaded one step ago).  colA /
// colB alternate between calls, so no load result is moved (and waited for)
// before the step that uses it.  Returns false after the CTA's last step.
template <int P, int H, bool SWZ, int E>
__device__ __forceinline__ bool sw_step(const SwGeom &G, SwState<P, H> &S, SwCursor<P, H> &ahead, int warp,
                                        int lane, int (&colA)[E], int (&colB)[E], int *rsr,
                                        const int32_t *__restrict__ rs, const int32_t *__restrict__ ci,
                                        const double *__restrict__ q, double *__restrict__ out,
                                        const double *__restrict__ carry, int64_t ncarry, uint64_t *full,
                                        uint64_t *empty, const double *ring, double *vt) {
    const int st = S.step;
    sw_issue_rs(ahead.rows(G), rs, lane, rsr + ((st + 4) & (kSwRsSlots - 1)) * kSwRsStride);  // step + 4
    ahead.next(G, warp);
    cp_async_wait<2>();  // row starts of steps + 1 and + 2 have landed (own copies) ...
    __syncwarp();        // ... and the other lanes' too
    sw_load_cols<E>(rsr + ((st + 1) & (kSwRsSlots - 1)) * kSwRsStride, ci, lane, colB);  // step + 1
    sw_prefetch_cols(rsr + ((st + 2) & (kSwRsSlots - 1)) * kSwRsStride, ci, lane);       // step + 2
    const int *cur = rsr + (st & (kSwRsSlots - 1)) * kSwRsStride;
    const int lo0 = cur[lane], end0 = cur[32];
    S.step = st + 1;

    const SwItem &I = S.I;
    const int c = S.c;
    const int nslot = G.nslot;
    // element planes of this row plane: wait for the newest
    const int zlo = max(el_lo<P>(c, G.K), G.z0), zhi = min(el_hi<P>(c, G.K), G.z1 - 1);
    if (zhi >= zlo) {
        const int need = S.base + (zhi - I.zf) + 1;
        for (; S.waited < need; S.waited++) {
            mbar_wait(&full[S.wslot], S.wph);
            if (++S.wslot == nslot) {
                S.wslot = 0;
                S.wph ^= 1u;
            }
        }
    }
    const int bb = I.b0 + warp;
    if (bb < G.g) {
        const int64_t r0 = ((int64_t)(c - G.c_lo) * G.g + bb) * G.g + I.a0;
        const int nrows = I.a1 - I.a0;
        const int e0 = __shfl_sync(0xffffffffu, lo0, 0);
        const int ne = end0 - e0;
        int nxt = __shfl_down_sync(0xffffffffu, lo0, 1);
        if (lane == nrows - 1) nxt = end0;
        double acc = 0.0;
        const int64_t r = r0 + lane;
        if (lane < nrows && r < ncarry) acc = carry[r];
        if (ne <= kSwVt) {
            // the <= 4 element runs (ey, ez) of this row line, ascending
            // columns; a missing run gets cb = INT_MAX (never selected)
            constexpr int N3 = (P + 1) * (P + 1) * (P + 1);
            const int ylo = el_lo<P>(bb, G.K), yhi = el_hi<P>(bb, G.K);
            const int ystride = G.K * N3, zstride = G.K * ystride, len = I.nx * N3;
            const bool zone = zhi >= zlo, y2 = yhi > ylo, z2 = zhi > zlo;
            const int c00 = zone ? ((zlo - G.z0) * G.K + ylo) * ystride + I.xlo * N3 : 0;
            int sl1 = S.rslot + 1;  // planes from zlo on are the unreleased ones: zlo is at rslot
            if (sl1 == nslot) sl1 = 0;
            const int s0 = S.rslot * G.plane_d + (ylo - I.ylo) * G.rs_d, s2 = sl1 * G.plane_d + (ylo - I.ylo) * G.rs_d;
            int cb[4], dd[4];
            cb[0] = zone ? c00 : INT_MAX;
            cb[1] = zone && y2 ? c00 + ystride : INT_MAX;
            cb[2] = z2 ? c00 + zstride : INT_MAX;
            cb[3] = z2 && y2 ? c00 + zstride + ystride : INT_MAX;
            dd[0] = s0 + (cb[0] & 1) - cb[0];
            dd[1] = s0 + G.rs_d + (cb[1] & 1) - cb[1];
            dd[2] = s2 + (cb[2] & 1) - cb[2];
            dd[3] = s2 + G.rs_d + (cb[3] & 1) - cb[3];
            // 0: generic run search; 1: interior fast path; 2: x-edge / partial fast path
            int fast = 0;
            if constexpr (P == 1) {
                // A structured warp-step -- rows in the closed-form order
                // (mesh.py:113-134: entry j = dz*4 + dy*2 + dx of row a is node
                // (1-dx, 1-dy, 1-dz) of element (a-1+dx, b-1+dy, c-1+dz)) -- is
                // verified against the loaded row starts and columns (one
                // compare per entry) and then needs no run search: entry
                // lane + 32 J has run (lane & 7) >> 1 for every J.  Interior
                // row lines only (both element rows in y and z present); the
                // x-edge rows a = 0 (entries dx = 1) and a = g-1 (dx = 0) have
                // 4 entries and shift the pattern (mode 2).
                if (z2 && y2 && ne <= kSwVt) {
                    // column of entry j = 0 of row a0 (element a0-1, node 7)
                    const int B0 = c00 + 8 * (I.a0 - 1 - I.xlo) + 7;
                    const int offl = ((lane >> 2) & 1) * (zstride - 4) + ((lane >> 1) & 1) * (ystride - 2) + (lane & 1) * 7;
                    if (nrows == kSwW && I.a0 >= 1 && I.a0 + kSwW <= G.g - 1 && ne == kSwVt) {
                        const int X = B0 + 8 * (lane >> 3) + offl;
                        bool ok = lo0 == e0 + 8 * lane;
#pragma unroll
                        for (int j = 0; j < E; j++) ok = ok && colA[j] == X + 32 * j;
                        fast = __all_sync(0xffffffffu, ok) ? 1 : 0;
                    } else {
                        const bool first = I.a0 == 0, last = I.a0 + nrows == G.g;
                        const int s0 = first ? 4 : 0, r1 = first ? 1 : 0;
                        const int nfull = nrows - r1 - (last ? 1 : 0);
                        const int ne_exp = s0 + 8 * nfull + (last ? 4 : 0);
                        bool ok = ne == ne_exp && nfull >= 0;
                        if (lane < nrows)
                            ok = ok && lo0 == (lane == 0 && first ? e0 : e0 + s0 + 8 * (lane - r1));
                        const int jl = (lane - s0) & 7;
                        const int X = B0 + 8 * (r1 + ((lane - s0) >> 3)) +
                                      ((jl >> 2) & 1) * (zstride - 4) + ((jl >> 1) & 1) * (ystride - 2) + (jl & 1) * 7;
#pragma unroll
                        for (int j = 0; j < E; j++) {
                            const int k = lane + 32 * j, kp = k - s0;
                            int want = X + 32 * j;
                            if (kp < 0) {  // row 0: entries dx = 1, j = 2k + 1
                                const int jj = 2 * k + 1;
                                want = B0 + ((jj >> 2) & 1) * (zstride - 4) + ((jj >> 1) & 1) * (ystride - 2) + 7;
                            } else if (kp >= 8 * nfull) {  // row g-1: entries dx = 0, j = 2m
                                const int jj = 2 * (kp - 8 * nfull);
                                want = B0 + 8 * (r1 + nfull) + ((jj >> 2) & 1) * (zstride - 4) +
                                       ((jj >> 1) & 1) * (ystride - 2);
                            }
                            ok = ok && (k >= ne || colA[j] == want);
                        }
                        fast = __all_sync(0xffffffffu, ok) ? 2 : 0;
                    }
                }
            }
            if (fast == 1) {
                const int D = (lane & 4) ? ((lane & 2) ? dd[3] : dd[2]) : ((lane & 2) ? dd[1] : dd[0]);
#pragma unroll
                for (int j = 0; j < E; j++) vt[vslot<SWZ>(lane + 32 * j)] = ring[colA[j] + D];
                __syncwarp();
#pragma unroll
                for (int t = 0; t < 8; t++) acc = add(acc, vt[vslot<SWZ>(8 * lane + t)]);
                st_stream(out + r, acc);
                __syncwarp();
            } else if (fast == 2) {
                // verified: every entry's run is its j >> 1 (rows 0 / g-1: 2k+1 / 2m)
                const bool first = I.a0 == 0, last = I.a0 + nrows == G.g;
                const int s0 = first ? 4 : 0, nfull = nrows - (first ? 1 : 0) - (last ? 1 : 0);
                const int jl = (lane - s0) & 7;
#pragma unroll
                for (int j = 0; j < E; j++) {
                    const int k = lane + 32 * j, kp = k - s0;
                    const int run = kp < 0 ? k : (kp >= 8 * nfull ? kp - 8 * nfull : jl >> 1);
                    const int D = (run & 2) ? ((run & 1) ? dd[3] : dd[2]) : ((run & 1) ? dd[1] : dd[0]);
                    if (k < ne) vt[vslot<SWZ>(k)] = ring[colA[j] + D];
                }
                __syncwarp();
                const int t0 = lane < nrows ? lo0 - e0 : 0, n = lane < nrows ? nxt - lo0 : 0;
#pragma unroll
                for (int t = 0; t < 8; t++) {
                    const double v = vt[vslot<SWZ>((t0 + t) & (kSwVt - 1))];
                    const double sum = add(acc, v);
                    acc = t < n ? sum : acc;
                }
                if (lane < nrows) st_stream(out + r, acc);
                __syncwarp();
            } else {
            // branch-free except for columns outside the runs (a warp vote)
#pragma unroll
            for (int j = 0; j < E; j++) {
                const int k = lane + 32 * j;
                const int col = colA[j];
                int csel = cb[0], dsel = dd[0];
#pragma unroll
                for (int t = 1; t < 4; t++) {
                    const bool ge = col >= cb[t];
                    csel = ge ? cb[t] : csel;
                    dsel = ge ? dd[t] : dsel;
                }
                const bool live = k < ne;
                const bool inrun = live && (unsigned)(col - csel) < (unsigned)len;
                double v = ring[inrun ? col + dsel : 0];
                if (__any_sync(0xffffffffu, live && !inrun)) {
                    if (live && !inrun) v = __ldg(q + col);  // a column outside the staged runs
                }
                if (live) vt[vslot<SWZ>(k)] = v;
            }
            __syncwarp();
            {
                // lanes >= nrows run the same (select-guarded) code on t0 = 0
                const int t0 = lane < nrows ? lo0 - e0 : 0, n = lane < nrows ? nxt - lo0 : 0;
#pragma unroll
                for (int t = 0; t < 8; t++) {
                    const double v = vt[vslot<SWZ>((t0 + t) & (kSwVt - 1))];
                    const double sum = add(acc, v);
                    acc = t < n ? sum : acc;
                }
                if (__any_sync(0xffffffffu, n > 8)) {
#pragma unroll 1
                    for (int t = 8; t < n; t++) acc = add(acc, vt[vslot<SWZ>(t0 + t)]);
                }
                if (lane < nrows) st_stream(out + r, acc);
            }
            __syncwarp();
            }
        } else if (lane < nrows) {  // long rows: straight from global memory
#pragma unroll 1
            for (int t = lo0; t < nxt; t++) acc = add(acc, __ldg(q + __ldg(ci + t)));
            st_stream(out + r, acc);
        }
    }

    // release the planes no later step of this item reads; advance
    const int keep = (c + 1 < I.c1) ? S.base + min(max(el_lo<P>(c + 1, G.K), G.z0) - I.zf, I.np)
                                    : S.base + I.np;
    if (keep > S.released) {
        __syncwarp();
        for (; S.released < keep; S.released++) {
            if (lane == 0) mbar_arrive(&empty[S.rslot]);
            if (++S.rslot == nslot) S.rslot = 0;
        }
    }
    if (++S.c >= I.c1) {
        S.base += I.np;
        S.it += gridDim.x;
        if (S.it >= G.n_items) return false;
        S.I = sw_item<P, H>(G, S.it);
        S.c = S.I.c0;
    }
    return true;
}

// The producer warp: lane y < ny copies run y of each element plane of the
// CTA's items into the ring (cp.async.bulk, one transaction count per plane);
// the item geometry is computed once per item, a plane is an address increment.
template <int P, int H>
__device__ __forceinline__ void sw_produce(const SwGeom &G, const double *__restrict__ q, double *ring,
                                           uint64_t *full, uint64_t *empty, int lane) {
    const int nslot = G.nslot;
    const int64_t grid = gridDim.x;
    constexpr int N3 = (P + 1) * (P + 1) * (P + 1);
    const int64_t pstride = (int64_t)G.K * G.K * N3;  // one element plane of q_local
    const int64_t qlim = G.nl & ~int64_t(1);          // bulk copies move whole 16 B units
    int64_t pit = blockIdx.x;                           // L2 prefetch cursor
    SwItem PI{};
    int pj = 0, pseq = 0;
    bool pok = false;
    auto p_load = [&]() {
        for (; pit < G.n_items; pit += grid) {
            PI = sw_item<P, H>(G, pit);
            if (PI.np > 0) {
                pok = true;
                return;
            }
        }
        pok = false;
    };
    if (G.pfd > 0) p_load();
    int seq = 0, slot = 0;
    uint32_t eph = 0;
    for (int64_t it = blockIdx.x; it < G.n_items; it += grid) {
        const SwItem I = sw_item<P, H>(G, it);
        const int64_t len = (int64_t)I.nx * N3;
        int64_t cb = lane < I.ny ? sw_col<P>(G, I.xlo, I.ylo + lane, I.zf) : 0;
        for (int j = 0; j < I.np; j++, seq++, cb += pstride) {
            while (pok && pseq <= seq + G.pfd) {
                if (pseq > seq && lane < PI.ny) {
                    const int64_t pc = sw_col<P>(G, PI.xlo, PI.ylo + lane, PI.zf + pj);
                    const int64_t pa = pc & ~int64_t(1), pe = min((pc + (int64_t)PI.nx * N3 + 1) & ~int64_t(1), qlim);
                    if (pe > pa) bulk_prefetch_l2(q + pa, (uint32_t)(pe - pa) * 8u);
                }
                pseq++;
                if (++pj >= PI.np) {
                    pj = 0;
                    pit += grid;
                    p_load();
                }
            }
            if (seq >= nslot) mbar_wait(&empty[slot], eph);
            double *dst = ring + (size_t)slot * G.plane_d + (size_t)lane * G.rs_d;
            const int64_t qa = cb & ~int64_t(1), qe = (cb + len + 1) & ~int64_t(1);
            const int64_t ce = qe < qlim ? qe : qlim;
            uint32_t bytes = 0;
            if (lane < I.ny) {
                // the odd tail past the last 16 B unit of q_local: plain
                // stores, ordered before lane 0's arrive by the warp sync
                if (qe > qlim)
                    for (int64_t x = qlim > qa ? qlim : qa; x < cb + len; x++) dst[x - qa] = __ldg(q + x);
                if (ce > qa) bytes = (uint32_t)(ce - qa) * 8u;
            }
            const uint32_t total = __reduce_add_sync(0xffffffffu, bytes);
            if (lane == 0) mbar_arrive_expect_tx(&full[slot], total);
            __syncwarp();
            if (bytes) bulk_g2s_plain(dst, q + qa, bytes, &full[slot]);
            if (++slot == nslot) {
                slot = 0;
                if (seq >= nslot) eph ^= 1u;
            }
        }
    }
}

template <int P, int H, bool SWZ, int MB>
__global__ void __launch_bounds__((H + 1) * 32, MB)
    k_bs6_sweep(SwGeom G, const int32_t *__restrict__ rs, const int32_t *__restrict__ ci,
                const double *__restrict__ q, double *__restrict__ out, const double *__restrict__ carry,
                int64_t ncarry) {
    constexpr int E = kSwVt / 32;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem);
    uint64_t *empty = full + kSwMaxSlots;
    double *ring = reinterpret_cast<double *>(smem + kSwHdr);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nslot = G.nslot;
    if (threadIdx.x == 0) {
        for (int s = 0; s < nslot; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], H);
        }
        fence_mbar_init();
    }
    __syncthreads();
    if (warp == H) {
        sw_produce<P, H>(G, q, ring, full, empty, lane);
        return;
    }

    // ------------------------------------------------------------ consumers
    double *vt = ring + (size_t)nslot * G.plane_d + (size_t)warp * kSwVt;
    if ((int64_t)blockIdx.x >= G.n_items) return;
    SwState<P, H> S;
    S.it = blockIdx.x;
    S.I = sw_item<P, H>(G, S.it);
    S.c = S.I.c0;
    S.base = S.waited = S.wslot = S.released = S.rslot = 0;
    S.wph = 0;
    S.step = 0;
    int *rsr = reinterpret_cast<int *>(ring + (size_t)nslot * G.plane_d + (size_t)H * kSwVt) +
               warp * kSwRsSlots * kSwRsStride;
    SwCursor<P, H> ahead;  // four steps ahead of S
    ahead.set(G, S.it, warp);
    for (int k = 0; k < 4; k++) {
        sw_issue_rs(ahead.rows(G), rs, lane, rsr + k * kSwRsStride);
        ahead.next(G, warp);
    }
    cp_async_wait<0>();
    __syncwarp();
    int col0[E], col1[E];
    sw_load_cols<E>(rsr, ci, lane, col0);
    sw_prefetch_cols(rsr + kSwRsStride, ci, lane);
    while (sw_step<P, H, SWZ, E>(G, S, ahead, warp, lane, col0, col1, rsr, rs, ci, q, out, carry, ncarry, full,
                                 empty, ring, vt) &&
           sw_step<P, H, SWZ, E>(G, S, ahead, warp, lane, col1, col0, rsr, rs, ci, q, out, carry, ncarry, full,
                                 empty, ring, vt)) {
    }
}

// ---------------------------------------------------------------- p = 2
// Row-lane consumer for p = 2 (k_bs6_sweep2).  A p = 2 row has 1, 2, 4 or 8
// entries (3.4 on average), so the value tile of the p = 1 path costs more
// than it saves; instead lane = row throughout: each lane loads its own <= 8
// column ids (one step ahead, from the row starts in the cp.async ring),
// checks them against the closed form of its row (mesh.py:113-134 order:
// candidates (ez, ey, ex) lexicographic, x fastest, node (kn, jn, in) =
// lattice - 2 * element), and -- when the whole warp matches -- sums its row
// straight from the staged element runs in ascending column order.  A run is
// 27 doubles per element (odd), so the 32 lanes' reads of 16 + 1 elements
// fall in distinct bank pairs: 2 wavefronts per read, the minimum for 8 B.
// Any mismatch (a CSR that is not the closed form, rows longer than 8) sums
// the warp's rows from global memory in the same order.

__device__ __forceinline__ void sw_load_cols_row(const int *slot, const int32_t *__restrict__ ci, int lane,
                                                 int (&col)[8]) {
    const int lo = slot[lane], n = slot[lane + 1] - lo;
#pragma unroll
    for (int t = 0; t < 8; t++)
        if (t < n) col[t] = __ldg(ci + lo + t);
}

template <int H>
__device__ __forceinline__ bool sw_step2(const SwGeom &G, SwState<2, H> &S, SwCursor<2, H> &ahead, int warp,
                                         int lane, int (&colA)[8], int (&colB)[8], int *rsr,
                                         const int32_t *__restrict__ rs, const int32_t *__restrict__ ci,
                                         const double *__restrict__ q, double *__restrict__ out,
                                         const double *__restrict__ carry, int64_t ncarry, uint64_t *full,
                                         uint64_t *empty, const double *ring) {
    constexpr int P = 2, N3 = 27;
    const int st = S.step;
    sw_issue_rs(ahead.rows(G), rs, lane, rsr + ((st + 4) & (kSwRsSlots - 1)) * kSwRsStride);  // step + 4
    ahead.next(G, warp);
    cp_async_wait<2>();
    __syncwarp();
    sw_load_cols_row(rsr + ((st + 1) & (kSwRsSlots - 1)) * kSwRsStride, ci, lane, colB);  // step + 1
    sw_prefetch_cols(rsr + ((st + 2) & (kSwRsSlots - 1)) * kSwRsStride, ci, lane);       // step + 2
    const int *cur = rsr + (st & (kSwRsSlots - 1)) * kSwRsStride;
    const int lo0 = cur[lane], n0 = cur[lane + 1] - lo0;
    S.step = st + 1;

    const SwItem &I = S.I;
    const int c = S.c;
    const int nslot = G.nslot;
    const int zlo = max(el_lo<P>(c, G.K), G.z0), zhi = min(el_hi<P>(c, G.K), G.z1 - 1);
    if (zhi >= zlo) {
        const int need = S.base + (zhi - I.zf) + 1;
        for (; S.waited < need; S.waited++) {
            mbar_wait(&full[S.wslot], S.wph);
            if (++S.wslot == nslot) {
                S.wslot = 0;
                S.wph ^= 1u;
            }
        }
    }
    const int bb = I.b0 + warp;
    if (bb < G.g) {
        const int nrows = I.a1 - I.a0;
        const int64_t r = ((int64_t)(c - G.c_lo) * G.g + bb) * G.g + I.a0 + lane;
        double acc = 0.0;
        if (lane < nrows && r < ncarry) acc = carry[r];
        // candidates: z, y per warp (groups g = (iz, iy), m of them), x per
        // lane (one or two); entry t of the row is group t / nx, x t % nx
        const int ylo = el_lo<P>(bb, G.K), yhi = el_hi<P>(bb, G.K);
        const int a = I.a0 + lane;
        const int xlo = el_lo<P>(a, G.K), xhi = el_hi<P>(a, G.K);
        const bool z2 = zhi > zlo, y2 = yhi > ylo, x2 = xhi > xlo;
        const int m = zhi < zlo ? 0 : (z2 ? 2 : 1) * (y2 ? 2 : 1);
        const int ystride = G.K * N3, zstride = G.K * ystride;
        // column of (g, x) = Y[g] + X{0,1}; staged index = column + D[g]
        const int cb0 = ((zlo - G.z0) * G.K + ylo) * ystride + I.xlo * N3;
        const int y00 = cb0 + (c - 2 * zlo) * 9 + (bb - 2 * ylo) * 3;
        const int dz = zstride - 18, dy = ystride - 6;
        const int X0 = (xlo - I.xlo) * N3 + (a - 2 * xlo), X1 = (xhi - I.xlo) * N3 + (a - 2 * xhi);
        int Y[4];
        Y[0] = y00;
        Y[1] = y00 + (y2 ? dy : dz);
        Y[2] = y00 + dz;
        Y[3] = y00 + dz + dy;
        bool ok = lane >= nrows || n0 == (x2 ? 2 * m : m);
#pragma unroll
        for (int g = 0; g < 4; g++) {
            const bool e0 = x2 ? colA[2 * g] == Y[g] + X0 : colA[g] == Y[g] + X0;
            const bool e1 = !x2 || colA[2 * g + 1] == Y[g] + X1;
            ok = ok && (g >= m || lane >= nrows || (e0 && e1));
        }
        if (m > 0 && __all_sync(0xffffffffu, ok)) {
            // staged byte address of group g's run: ring slot of its z plane,
            // run of its y, the run's 16 B-alignment shift, minus its first column
            int sl1 = S.rslot + 1;
            if (sl1 == nslot) sl1 = 0;
            const uint32_t rb = smem_u32(ring);
            const int s0 = S.rslot * G.plane_d + (ylo - I.ylo) * G.rs_d, s2 = sl1 * G.plane_d + (ylo - I.ylo) * G.rs_d;
            const int cy = cb0 + ystride, cz = cb0 + zstride, czy = cz + ystride;
            uint32_t E[4];
            E[0] = rb + 8u * (uint32_t)(s0 + (cb0 & 1) - cb0 + Y[0]);
            E[1] = y2 ? rb + 8u * (uint32_t)(s0 + G.rs_d + (cy & 1) - cy + Y[1])
                      : rb + 8u * (uint32_t)(s2 + (cz & 1) - cz + Y[1]);
            E[2] = rb + 8u * (uint32_t)(s2 + (cz & 1) - cz + Y[2]);
            E[3] = rb + 8u * (uint32_t)(s2 + G.rs_d + (czy & 1) - czy + Y[3]);
            const uint32_t x0 = 8u * (uint32_t)X0, x1 = 8u * (uint32_t)X1;
            if (lane < nrows) {
#pragma unroll
                for (int g = 0; g < 4; g++) {
                    if (g < m) {
                        acc = add(acc, lds_f64(E[g] + x0));
                        if (x2) acc = add(acc, lds_f64(E[g] + x1));
                    }
                }
                st_stream(out + r, acc);
            }
        } else if (lane < nrows) {  // not the closed form: from global memory
#pragma unroll 1
            for (int t = lo0; t < lo0 + n0; t++) acc = add(acc, __ldg(q + __ldg(ci + t)));
            st_stream(out + r, acc);
        }
    }

    const int keep = (c + 1 < I.c1) ? S.base + min(max(el_lo<P>(c + 1, G.K), G.z0) - I.zf, I.np)
                                    : S.base + I.np;
    if (keep > S.released) {
        __syncwarp();
        for (; S.released < keep; S.released++) {
            if (lane == 0) mbar_arrive(&empty[S.rslot]);
            if (++S.rslot == nslot) S.rslot = 0;
        }
    }
    if (++S.c >= I.c1) {
        S.base += I.np;
        S.it += gridDim.x;
        if (S.it >= G.n_items) return false;
        S.I = sw_item<P, H>(G, S.it);
        S.c = S.I.c0;
    }
    return true;
}

template <int H, int MB>
__global__ void __launch_bounds__((H + 1) * 32, MB)
    k_bs6_sweep2(SwGeom G, const int32_t *__restrict__ rs, const int32_t *__restrict__ ci,
                 const double *__restrict__ q, double *__restrict__ out, const double *__restrict__ carry,
                 int64_t ncarry) {
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem);
    uint64_t *empty = full + kSwMaxSlots;
    double *ring = reinterpret_cast<double *>(smem + kSwHdr);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nslot = G.nslot;
    if (threadIdx.x == 0) {
        for (int s = 0; s < nslot; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], H);
        }
        fence_mbar_init();
    }
    __syncthreads();
    if (warp == H) {
        sw_produce<2, H>(G, q, ring, full, empty, lane);
        return;
    }
    if ((int64_t)blockIdx.x >= G.n_items) return;
    SwState<2, H> S;
    S.it = blockIdx.x;
    S.I = sw_item<2, H>(G, S.it);
    S.c = S.I.c0;
    S.base = S.waited = S.wslot = S.released = S.rslot = 0;
    S.wph = 0;
    S.step = 0;
    int *rsr = reinterpret_cast<int *>(ring + (size_t)nslot * G.plane_d) + warp * kSwRsSlots * kSwRsStride;
    SwCursor<2, H> ahead;
    ahead.set(G, S.it, warp);
    for (int k = 0; k < 4; k++) {
        sw_issue_rs(ahead.rows(G), rs, lane, rsr + k * kSwRsStride);
        ahead.next(G, warp);
    }
    cp_async_wait<0>();
    __syncwarp();
    int col0[8], col1[8];
    sw_load_cols_row(rsr, ci, lane, col0);
    sw_prefetch_cols(rsr + kSwRsStride, ci, lane);
    while (sw_step2<H>(G, S, ahead, warp, lane, col0, col1, rsr, rs, ci, q, out, carry, ncarry, full, empty, ring) &&
           sw_step2<H>(G, S, ahead, warp, lane, col1, col0, rsr, rs, ci, q, out, carry, ncarry, full, empty, ring)) {
    }
}

// tuning knobs (sb_bs6_sweep_tune; A/B runs and tests): <= 0 / < 0 = default
int g_sw_slots = 0, g_sw_pfd = -1, g_sw_waves = 0, g_sw_swz = -1, g_sw_h = 0;

template <int P, int H, int MB>
int sweep_launch(const SwGeom &G0, const int32_t *rs, const int32_t *ci, const double *q, double *out,
                 const double *carry, int64_t ncarry, bool swz, bool row2, cudaStream_t st) {
    SwGeom G = G0;
    G.nb = (G.g + H - 1) / H;
    constexpr int N3 = (P + 1) * (P + 1) * (P + 1);
    const int nx_max = (kSwW - 1) / P + 2, ny_max = (H - 1) / P + 2;
    G.rs_d = (nx_max * N3 + 2 + 15) / 16 * 16;  // + the odd-start shift and 16 B rounding
    G.plane_d = ny_max * G.rs_d;
    auto smem_for = [&](int ns) {
        return kSwHdr + (size_t)ns * G.plane_d * 8 + (row2 ? 0 : (size_t)H * kSwVt * 8) +
               (size_t)H * kSwRsSlots * kSwRsStride * 4;
    };
    while (G.nslot > 3 && smem_for(G.nslot) > 227 * 1024) G.nslot--;  // large columns: a shallower ring
    const size_t smem = smem_for(G.nslot);
    using KernT = void (*)(SwGeom, const int32_t *, const int32_t *, const double *, double *, const double *,
                           int64_t);
    KernT k = swz ? k_bs6_sweep<P, H, true, MB> : k_bs6_sweep<P, H, false, MB>;
    if constexpr (P == 2)
        if (row2) k = k_bs6_sweep2<H, MB>;
    int rc = cuda_check(cudaFuncSetAttribute((const void *)k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                        "sb_bs6_gather_sweep: shared memory");
    if (rc) return rc;
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void *)k, (H + 1) * 32, smem);
    per_sm = std::max(1, per_sm);
    const int64_t grid_max = (int64_t)sm_count() * per_sm;
    // z chunks: about 8 items per resident CTA (tail balance) without cutting
    // the sweep shorter than needed (each chunk re-reads one element plane)
    const int64_t ncols = (int64_t)G.na * G.nb, nc = G.c_hi - G.c_lo;
    const int64_t want = grid_max * (g_sw_waves > 0 ? g_sw_waves : 8);
    int64_t nch = std::max<int64_t>(1, std::min<int64_t>(nc, (want + ncols - 1) / ncols));
    G.ch = (int)((nc + nch - 1) / nch);
    nch = (nc + G.ch - 1) / G.ch;
    G.n_items = ncols * nch;
    const int64_t grid = std::min<int64_t>(G.n_items, grid_max);
    k<<<(unsigned)grid, (H + 1) * 32, smem, st>>>(G, rs, ci, q, out, carry, ncarry);
    return launch_check("sb_bs6_gather_sweep");
}

}  // namespace
}  // namespace sb

using namespace sb;

extern "C" {

int sb_bs6_gather_sweep(int32_t K, int32_t p, int32_t z0, int32_t z1, int32_t c_lo, int32_t c_hi,
                        const int32_t *row_starts, const int32_t *col_ids, int64_t ng, int64_t nl,
                        const double *q_local, double *out, const double *carry_in, int64_t n_carry,
                        sb_stream_t stream) {
    clear_error();
    const int64_t g = (int64_t)K * p + 1, n3 = (int64_t)(p + 1) * (p + 1) * (p + 1);
    if (K < 1 || p < 1 || p > 2 || z0 < 0 || z1 > K || z0 >= z1 || c_lo < 0 || c_hi > g || c_lo >= c_hi) {
        set_error("sb_bs6_gather_sweep: invalid geometry (K=%d p=%d z=[%d,%d) c=[%d,%d); p must be 1 or 2)", K, p,
                  z0, z1, c_lo, c_hi);
        return SB_E_INVALID;
    }
    if (ng != (int64_t)(c_hi - c_lo) * g * g || nl != (int64_t)K * K * (z1 - z0) * n3 || nl > INT_MAX ||
        n_carry < 0 || (n_carry > 0 && !carry_in) || !row_starts || !col_ids || !q_local || !out) {
        set_error("sb_bs6_gather_sweep: invalid arguments (ng=%lld nl=%lld do not match the geometry)",
                  (long long)ng, (long long)nl);
        return SB_E_INVALID;
    }
    if (!aligned16(q_local)) {
        set_error("sb_bs6_gather_sweep: q_local must be 16-byte aligned");
        return SB_E_INVALID;
    }
    if (n_carry > ng) n_carry = ng;
    SwGeom G{};
    G.K = K;
    G.z0 = z0;
    G.z1 = z1;
    G.c_lo = c_lo;
    G.c_hi = c_hi;
    G.g = (int)g;
    G.na = (int)((g + kSwW - 1) / kSwW);
    G.nl = nl;
    G.nslot = g_sw_slots > 0 ? g_sw_slots : 4;
    G.pfd = g_sw_pfd >= 0 ? g_sw_pfd : 0;  // L2 prefetch measured slower (profiles/r02_bs6_sweep.md)
    const bool swz = g_sw_swz >= 0 ? g_sw_swz == 1 : p == 1;
    // p = 2: the row-lane consumer (k_bs6_sweep2) unless SB200_BS6_SWEEP_ROW2=0
    const char *r2env = getenv("SB200_BS6_SWEEP_ROW2");
    const bool row2 = p == 2 && !(r2env && r2env[0] == '0');
    const cudaStream_t st = as_stream(stream);
    // row lines per column (one consumer warp each) and CTAs per SM: 8 / 2 by
    // default; 7 / 3 and 16 / 1 for A/B runs
    const int h = g_sw_h > 0 ? g_sw_h : 8;
#define SB_SW(P_) (h == 7 ? sweep_launch<P_, 7, 3>(G, row_starts, col_ids, q_local, out, carry_in, n_carry, swz, row2, st) \
                  : h == 16 ? sweep_launch<P_, 16, 1>(G, row_starts, col_ids, q_local, out, carry_in, n_carry, swz, row2, st) \
                            : sweep_launch<P_, 8, 2>(G, row_starts, col_ids, q_local, out, carry_in, n_carry, swz, row2, st))
    const int rc = p == 1 ? SB_SW(1) : SB_SW(2);
#undef SB_SW
    return rc;
}

int sb_bs6_sweep_tune(int32_t slots, int32_t l2_prefetch_planes, int32_t waves, int32_t swizzle,
                      int32_t row_lines) {
    clear_error();
    if (slots > kSwMaxSlots || (slots > 0 && slots < 3)) {
        set_error("sb_bs6_sweep_tune: slots must be 3..%d (0: default)", kSwMaxSlots);
        return SB_E_INVALID;
    }
    g_sw_slots = slots;
    g_sw_pfd = l2_prefetch_planes;
    g_sw_waves = waves;
    g_sw_swz = swizzle;
    g_sw_h = (row_lines == 7 || row_lines == 8 || row_lines == 16) ? row_lines : 0;
    return SB_OK;
}

}  // extern "C"
