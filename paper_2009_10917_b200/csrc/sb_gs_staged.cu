// sb_gs_staged.cu -- BS6 gather for low polynomial orders with TMA-staged
// value runs (gs.py:10-39; bitwise the reference: every row is summed in
// ascending column order from +0.0, or from the carry-in, by one thread).
//
// Why a second BS6 kernel.  At p = 1 (and 2) a row's 8 (1-8) entries come
// from 8 different elements, so the LSU-gather kernels of sb_gs_pipe.cu pay
// about one L1 tag lookup per 8-byte entry: ncu at N=1 shows the L1 data
// pipe at 86% of peak with DRAM at 55% (profiles/r01_bs6_variants.md).  Here
// the q gathers never touch the LSU/L1 tag path: a tile is a patch of
// ey*p x ez*p row lines (y, z) times w rows along x, and every element row
// ((ey+1)(ez+1) of them) that the patch reads is a CONTIGUOUS run of q_local
// (element-major numbering, mesh.py:73-97).  A producer warp copies those
// runs and the patch's col_ids / row_starts slices -- nothing else -- into a
// shared-memory stage with cp.async.bulk (TMA; mbarrier transaction counts),
// three stages deep; eight consumer warps then take chunks of 32 rows:
//   1. each entry of the chunk's rows: column (staged col_ids) -> staged slot
//      (compare chain over the <= 4 runs the row line can touch) -> value
//      tile, in CSR order (a column outside the staged runs is read from
//      global memory: any CSR gives the right answer, the plan only decides
//      speed);
//   2. each row (one lane): sum of its value-tile entries, ascending.
//
// The tile plan is operator metadata like the super-block plan of
// sb_gs_pipe.cu, built once per operator on the GPU (k_bs6_staged_plan) from
// the mesh geometry and row_starts: for each tile, the complete table the
// consumers read (segment / run / chunk offsets, shared-memory layout of the
// stage), so the producer only validates and issues copies.  Table words
// (offsets in StLayout; S = max segments, R = max runs, C = max chunks):
//   hdr[8]  nseg, nrun, nchunk, -, flags (1: direct, 2: skip), -, -, -
//   koff[S+1]  entry offset of segment s in the tile (value tile index)
//   rso[S] cio[S]  shared-memory word of segment s's first row start / col id
//   e0[S] row0[S] nrow[S]  first entry, first row, row count of segment s
//   rl[S]  the <= 4 runs segment s can touch (bytes, ascending, 0xff = none)
//   cb[R] ce[R] dd[R]  run r: columns [cb, ce) at shared slot column + dd
//   ch[C]  chunk word: segment | first row << 5 | rows << 16
#include <limits.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>

#include "sb_common.cuh"

namespace sb {

namespace {

constexpr int kStMaxNst = 4;  // data stages
constexpr int kStNDesc = 8;   // tile tables in flight (>= stages + prefetch distance)

struct StLayout {
    int D, maxseg, maxrun, chcap;                                                  // table geometry
    int o_koff, o_rso, o_cio, o_e0, o_row0, o_nrow, o_rl, o_cb, o_ce, o_dd, o_ch;  // table offsets
    int rscap, cicap, qcap, vtcap, nst;                                            // stage capacities
    int off_desc, off_vt, off_stage, stage_bytes, st_ci, st_q;                     // shared-memory bytes
};

StLayout table_layout(int S, int R, int C) {
    StLayout L{};
    L.maxseg = S;
    L.maxrun = R;
    L.chcap = C;
    L.o_koff = 8;
    L.o_rso = L.o_koff + S + 1;
    L.o_cio = L.o_rso + S;
    L.o_e0 = L.o_cio + S;
    L.o_row0 = L.o_e0 + S;
    L.o_nrow = L.o_row0 + S;
    L.o_rl = L.o_nrow + S;
    L.o_cb = L.o_rl + S;
    L.o_ce = L.o_cb + R;
    L.o_dd = L.o_ce + R;
    L.o_ch = L.o_dd + R;
    L.D = (L.o_ch + C + 3) / 4 * 4;  // 16-byte multiple (one bulk copy per table)
    return L;
}

__device__ __forceinline__ int imin(int a, int b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ int64_t up4(int64_t v) { return (v + 3) & ~int64_t(3); }
__host__ __device__ __forceinline__ int64_t up2(int64_t v) { return (v + 1) & ~int64_t(1); }

template <bool SWZ>
__device__ __forceinline__ int vslot(int k) {
    return SWZ ? (k ^ ((k >> 4) & 15)) : k;
}

__device__ __forceinline__ void bulk_g2s_nohint(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

template <bool SWZ, int NWC, int NP>
__global__ void __launch_bounds__((NWC + NP) * 32)
    k_bs6_staged(const int32_t *__restrict__ plan, int64_t ntiles, StLayout L, const int32_t *__restrict__ rs,
                 int64_t ng, const int32_t *__restrict__ ci, int64_t nl, const double *__restrict__ q, int64_t nq,
                 double *__restrict__ out, const double *__restrict__ carry, int64_t ncarry, int mode) {
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem);
    uint64_t *empty = full + kStMaxNst;
    uint64_t *dfull = empty + kStMaxNst;
    int32_t *desc = reinterpret_cast<int32_t *>(smem + L.off_desc);
    double *vt = reinterpret_cast<double *>(smem + L.off_vt);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nst = L.nst, D = L.D;
    if (threadIdx.x == 0) {
        for (int s = 0; s < nst; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NWC);
        }
        for (int s = 0; s < kStNDesc; s++) mbar_init(&dfull[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
    const int64_t G = gridDim.x;

    if (warp >= NWC) {
        // ------------------------------------------------------------------
        // producer warps (NP, alternating tiles): lane s issues segment s's
        // row-start and col-id slices, lane r run r's q values; tile tables
        // arrive kStNDesc - nst tiles ahead of their data
        const int pw = warp - NWC;
        const uint64_t pol_first = policy_evict_first();
        if (pw == 0 && lane == 0) {
            for (int j = 0; j < kStNDesc; j++) {
                const int64_t t = blockIdx.x + j * G;
                if (t < ntiles) {
                    mbar_arrive_expect_tx(&dfull[j], (uint32_t)(D * 4));
                    bulk_g2s(desc + j * D, plan + t * D, (uint32_t)(D * 4), &dfull[j], pol_first);
                }
            }
        }
        const int64_t rs_lim = (ng + 1) & ~int64_t(3), ci_lim = nl & ~int64_t(3), q_lim = nq & ~int64_t(1);
        int i = pw;
        for (int64_t t = blockIdx.x + (int64_t)pw * G; t < ntiles; t += NP * G, i += NP) {
            const int ds = i % kStNDesc, st = i % nst;
            mbar_wait(&dfull[ds], (uint32_t)((i / kStNDesc) & 1));
            if (i >= nst) {
                mbar_wait(&empty[st], (uint32_t)(((i / nst) & 1) ^ 1));
                // tile i - nst is consumed: its table slot takes tile i - nst + kStNDesc
                if (lane == 0) {
                    const int64_t tn = t + (int64_t)(kStNDesc - nst) * G;
                    if (tn < ntiles) {
                        const int sl = (i - nst) % kStNDesc;
                        fence_proxy_async();
                        mbar_arrive_expect_tx(&dfull[sl], (uint32_t)(D * 4));
                        bulk_g2s(desc + sl * D, plan + tn * D, (uint32_t)(D * 4), &dfull[sl], pol_first);
                    }
                }
            }
            int32_t *tbl = desc + ds * D;
            unsigned char *sb = smem + L.off_stage + (size_t)st * L.stage_bytes;
            int32_t *rss = reinterpret_cast<int32_t *>(sb);
            int32_t *cis = reinterpret_cast<int32_t *>(sb + L.st_ci);
            double *qs = reinterpret_cast<double *>(sb + L.st_q);
            const int nseg = tbl[0], nrun = tbl[1], nch = tbl[2], flags = tbl[4];
            // a malformed table (never emitted by the builder) skips the tile;
            // slices that would leave the stage demote it to direct loads
            bool ok = (unsigned)nseg <= (unsigned)L.maxseg && (unsigned)nrun <= (unsigned)L.maxrun &&
                      (unsigned)nch <= (unsigned)L.chcap && (flags & ~1) == 0;
            bool fit = true;
            // slice of this lane (int32: rows < 2^31, entries < 2^31, staging offsets < 2^16)
            int ra = 0, rb = 0, r1 = 0, ca = 0, cbe = 0, e1 = 0, qa = 0, qb = 0, c1 = 0;
            int rdo = 0, cdo = 0, qdo = 0;  // shared-memory element offsets of the copies
            if (ok && lane < nseg) {
                const int row0 = tbl[L.o_row0 + lane], nrow = tbl[L.o_nrow + lane], e0 = tbl[L.o_e0 + lane];
                const int k0 = tbl[L.o_koff + lane], k1 = tbl[L.o_koff + lane + 1];
                ok = row0 >= 0 && nrow >= 0 && (int64_t)row0 + nrow <= ng;
                r1 = row0 + nrow;
                e1 = e0 + (k1 - k0);
                ra = row0 & ~3;
                rb = (r1 + 4) & ~3;
                ca = e0 & ~3;
                cbe = (e1 + 3) & ~3;
                rdo = tbl[L.o_rso + lane] - (row0 - ra);
                cdo = tbl[L.o_cio + lane] - (e0 - ca);
                fit = e0 >= 0 && k0 >= 0 && k1 >= k0 && k1 <= L.vtcap && (int64_t)e1 <= nl && rdo >= 0 &&
                      rdo + (rb - ra) <= L.rscap && cdo >= 0 && cdo + (cbe - ca) <= L.cicap;
            }
            if (ok && lane < nrun) {
                const int c0 = tbl[L.o_cb + lane], dd = tbl[L.o_dd + lane];
                c1 = tbl[L.o_ce + lane];
                qa = c0 & ~1;
                qb = (c1 + 1) & ~1;
                qdo = dd + qa;
                fit = fit && c0 >= 0 && c1 >= c0 && (int64_t)c1 <= nq && qdo >= 0 && (qdo & 1) == 0 &&
                      dd + qb <= L.qcap;
            }
            if (ok && lane < nch) {
                const int32_t cw = tbl[L.o_ch + lane];
                const int s = cw & 31, li0 = (cw >> 5) & 2047, cnt = cw >> 16;
                ok = s < nseg && cnt >= 1 && cnt <= 32 && li0 + cnt <= tbl[L.o_nrow + s];
            }
            ok = __all_sync(0xffffffffu, ok);
            fit = __all_sync(0xffffffffu, fit);
            const bool stage = ok && fit && flags == 0;
            int bytes = 0;
            if (stage) {
                if (lane < nseg) {
                    if (rb > rs_lim) {  // tail past the last 16-byte boundary: direct loads
                        for (int x = (int)(ra > rs_lim ? ra : rs_lim); x <= r1; x++) rss[rdo + x - ra] = __ldg(rs + x);
                        rb = (int)(rs_lim > ra ? rs_lim : ra);
                    }
                    if (cbe > ci_lim) {
                        for (int x = (int)(ca > ci_lim ? ca : ci_lim); x < e1; x++) cis[cdo + x - ca] = __ldg(ci + x);
                        cbe = (int)(ci_lim > ca ? ci_lim : ca);
                    }
                    bytes += (rb - ra) * 4 + (cbe - ca) * 4;
                }
                if (lane < nrun) {
                    if (qb > q_lim) {
                        for (int64_t x = qa > q_lim ? qa : q_lim; x < c1; x++) qs[qdo + x - qa] = __ldg(q + x);
                        qb = (int)(q_lim > qa ? q_lim : qa);
                    }
                    bytes += (qb - qa) * 8;
                }
            }
            bytes = __reduce_add_sync(0xffffffffu, bytes);
            if (lane == 0) {
                if (!ok)
                    tbl[4] = 2;
                else if (!stage)
                    tbl[4] = 1;
                if (stage)
                    mbar_arrive_expect_tx(&full[st], (uint32_t)bytes);
                else
                    mbar_arrive(&full[st]);
            }
            __syncwarp();
            if (stage) {
                if (lane < nseg) {
                    if (rb > ra) bulk_g2s(rss + rdo, rs + ra, (uint32_t)(rb - ra) * 4u, &full[st], pol_first);
                    if (cbe > ca) bulk_g2s(cis + cdo, ci + ca, (uint32_t)(cbe - ca) * 4u, &full[st], pol_first);
                }
                if (lane < nrun && qb > qa) bulk_g2s_nohint(qs + qdo, q + qa, (uint32_t)(qb - qa) * 8u, &full[st]);
            }
        }
        return;
    }

    // ------------------------------------------------------------ consumers
    // Chunks are dealt round-robin over the warps across tiles (running offset).
    int deal = 0, ds = 0, dph = 0, st = 0, sph = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += G) {
        mbar_wait(&dfull[ds], (uint32_t)dph);  // (complete long ago: makes the table visible here)
        mbar_wait(&full[st], (uint32_t)sph);
        const int32_t *tbl = desc + ds * D;
        const unsigned char *sb = smem + L.off_stage + (size_t)st * L.stage_bytes;
        const int32_t *rss = reinterpret_cast<const int32_t *>(sb);
        const int32_t *cis = reinterpret_cast<const int32_t *>(sb + L.st_ci);
        const double *qs = reinterpret_cast<const double *>(sb + L.st_q);
        double *vtb = vt + (size_t)st * L.vtcap;
        const int flags = tbl[4], nch = (flags == 2 || mode == 1) ? 0 : tbl[2], nrun = tbl[1];
        int c = (warp - deal) & (NWC - 1);
        deal = (deal + nch) & (NWC - 1);
        for (; c < nch; c += NWC) {
            const int32_t cw = tbl[L.o_ch + c];
            const int s = cw & 31, li0 = (cw >> 5) & 2047, cnt = cw >> 16;  // warp-uniform
            const int64_t row = (int64_t)tbl[L.o_row0 + s] + li0 + lane;
            const bool valid = lane < cnt;
            double acc = 0.0;
            if (valid && row < ncarry) acc = carry[row];
            if (flags == 0) {
                const int koff = tbl[L.o_koff + s], rso = tbl[L.o_rso + s] + li0, cio = tbl[L.o_cio + s];
                const int e0s = tbl[L.o_e0 + s];
                const uint32_t rl = (uint32_t)tbl[L.o_rl + s];
                int cb[4], ce[4], dd[4];
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    const int r = (rl >> (8 * j)) & 0xff;
                    const bool has = r < nrun;
                    cb[j] = has ? tbl[L.o_cb + r] : INT_MAX;
                    ce[j] = has ? tbl[L.o_ce + r] : INT_MIN;
                    dd[j] = has ? tbl[L.o_dd + r] : 0;
                }
                int kk = 0, n = 0;  // entries of this lane's row, relative to the segment
                if (valid) {
                    const int lo = rss[rso + lane];
                    n = rss[rso + lane + 1] - lo;
                    kk = lo - e0s;
                }
                const int kb = __shfl_sync(0xffffffffu, kk, 0);
                const int ke = __shfl_sync(0xffffffffu, kk + n, cnt - 1);
                for (int k = kb + lane; k < ke; k += 32) {
                    const int col = cis[cio + k];
                    int dsel = dd[0], lim = ce[0];
                    const bool in0 = col >= cb[0];
#pragma unroll
                    for (int j = 1; j < 4; j++)
                        if (col >= cb[j]) {
                            dsel = dd[j];
                            lim = ce[j];
                        }
                    double v;
                    if (in0 && col < lim)
                        v = qs[col + dsel];
                    else
                        v = __ldg(q + col);  // column outside the staged runs
                    vtb[vslot<SWZ>(koff + k)] = v;
                }
                __syncwarp();
                if (valid) {
#pragma unroll 1
                    for (int j = 0; j < n; j++) acc = add(acc, vtb[vslot<SWZ>(koff + kk + j)]);
                }
            } else if (valid) {
                const int lo = __ldg(rs + row), hi = __ldg(rs + row + 1);
#pragma unroll 1
                for (int j = lo; j < hi; j++) acc = add(acc, __ldg(q + __ldg(ci + j)));
            }
            if (valid) st_stream(out + row, acc);
            __syncwarp();  // the next chunk's value writes come after these reads
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
        if (++ds == kStNDesc) {
            ds = 0;
            dph ^= 1;
        }
        if (++st == nst) {
            st = 0;
            sph ^= 1;
        }
    }
}

// ---- structured tile plan ----------------------------------------------
struct StGeom {
    int K, p, z0, z1, c_lo, c_hi, ey, ez, w, g;
    int64_t na, nb;  // tiles along x (rows), along y (row-line patches)
};

// element range of lattice coordinate x (0 .. K*p) along one axis
__device__ __forceinline__ int el_lo(int x, int p, int K) {
    return (x % p == 0 && x > 0) ? imin(x / p - 1, K - 1) : imin(x / p, K - 1);
}
__device__ __forceinline__ int el_hi(int x, int p, int K) { return imin(x / p, K - 1); }

__global__ void k_bs6_staged_plan(StGeom G, StLayout L, const int32_t *__restrict__ rs, int32_t *__restrict__ plan,
                                  int64_t ntiles) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < ntiles;
         t += (int64_t)gridDim.x * blockDim.x) {
        int32_t *d = plan + t * L.D;
        for (int x = 0; x < L.D; x++) d[x] = 0;
        const int64_t ab = t % G.na, bb = (t / G.na) % G.nb, cb = t / (G.na * G.nb);
        const int Pb = G.ey * G.p, Pc = G.ez * G.p;
        const int a0 = (int)(ab * G.w), a1 = min(G.g, a0 + G.w);
        const int b0 = (int)(bb * Pb), b1 = min(G.g, b0 + Pb);
        const int c0 = G.c_lo + (int)(cb * Pc), c1 = min(G.c_hi, c0 + Pc);
        const int xlo = el_lo(a0, G.p, G.K), xhi = el_hi(a1 - 1, G.p, G.K);
        const int ylo = el_lo(b0, G.p, G.K), yhi = el_hi(b1 - 1, G.p, G.K);
        const int zlo = max(el_lo(c0, G.p, G.K), G.z0), zhi = min(el_hi(c1 - 1, G.p, G.K), G.z1 - 1);
        const int ny = yhi - ylo + 1;
        const int64_t n3 = (int64_t)(G.p + 1) * (G.p + 1) * (G.p + 1);
        // runs (element rows), ascending columns; shared slots keep each run's
        // 128-byte phase of an (assumed 128-B aligned) q_local: the bank pattern of HBM order
        int nrun = 0;
        int64_t qp = 0;
        for (int ez = zlo; ez <= zhi; ez++)
            for (int ey = ylo; ey <= yhi; ey++) {
                const int64_t e = ((int64_t)(ez - G.z0) * G.K + ey) * G.K + xlo;
                const int64_t cc0 = e * n3, cc1 = (e + (xhi - xlo + 1)) * n3, qa = cc0 & ~int64_t(1);
                const int64_t qo = qp + ((qa - qp) & 15);
                d[L.o_cb + nrun] = (int32_t)cc0;
                d[L.o_ce + nrun] = (int32_t)cc1;
                d[L.o_dd + nrun] = (int32_t)(qo - qa);
                qp = qo + (up2(cc1) - qa);
                nrun++;
            }
        // segments (row lines in ascending row order), their staging offsets and chunks
        int nseg = 0, nch = 0;
        int64_t ne = 0, rso = 0, cio = 0;
        for (int c = c0; c < c1; c++)
            for (int b = b0; b < b1; b++) {
                const int64_t r0 = ((int64_t)(c - G.c_lo) * G.g + b) * G.g + a0, nrow = a1 - a0;
                const int64_t e0 = rs[r0], e1 = rs[r0 + nrow];
                const int64_t ra = r0 & ~int64_t(3), ca = e0 & ~int64_t(3);
                d[L.o_koff + nseg] = (int32_t)ne;
                d[L.o_rso + nseg] = (int32_t)(rso + (r0 - ra));
                d[L.o_cio + nseg] = (int32_t)(cio + (e0 - ca));
                d[L.o_e0 + nseg] = (int32_t)e0;
                d[L.o_row0 + nseg] = (int32_t)r0;
                d[L.o_nrow + nseg] = (int32_t)nrow;
                uint32_t rl = 0xffffffffu;
                int nl4 = 0;
                const int zl = max(el_lo(c, G.p, G.K), G.z0), zh = min(el_hi(c, G.p, G.K), G.z1 - 1);
                for (int ez = zl; ez <= zh; ez++)
                    for (int ey = el_lo(b, G.p, G.K); ey <= el_hi(b, G.p, G.K); ey++)
                        if (nl4 < 4) {
                            const uint32_t r = (uint32_t)((ez - zlo) * ny + (ey - ylo));
                            rl = (rl & ~(0xffu << (8 * nl4))) | (r << (8 * nl4));
                            nl4++;
                        }
                d[L.o_rl + nseg] = (int32_t)rl;
                for (int64_t j = 0; j < nrow; j += 32)
                    if (nch < L.chcap)
                        d[L.o_ch + nch++] = nseg | ((int32_t)j << 5) | ((int32_t)(nrow - j < 32 ? nrow - j : 32) << 16);
                rso += up4(r0 + nrow + 1) - ra;
                cio += up4(e1) - ca;
                ne += e1 - e0;
                nseg++;
            }
        for (int s = nseg; s <= L.maxseg; s++) d[L.o_koff + s] = (int32_t)ne;
        d[0] = nseg;
        d[1] = nrun;
        d[2] = nch;
        d[4] = (rso <= L.rscap && cio <= L.cicap && qp <= L.qcap && ne <= L.vtcap) ? 0 : 1;
    }
}

constexpr int kMaxSeg = 31;  // one producer lane per segment / run
constexpr int kMaxRun = 32;

StLayout full_layout(const sb_bs6_staged_t &I, int nst) {
    StLayout L = table_layout(I.max_segments, I.max_runs, I.max_segments * ((I.w + 31) / 32));
    L.rscap = I.rs_cap;
    L.cicap = I.ci_cap;
    L.qcap = I.q_cap;
    L.vtcap = I.vt_cap;
    L.nst = nst;
    auto up = [](int v, int a) { return (v + a - 1) / a * a; };
    L.off_desc = 128;  // mbarriers: full[4], empty[4], dfull[8]
    L.off_vt = up(L.off_desc + kStNDesc * L.D * 4, 128);
    L.off_stage = up(L.off_vt + nst * L.vtcap * 8, 128);  // one value tile per stage
    L.st_ci = up(L.rscap * 4, 16);
    L.st_q = up(L.st_ci + L.cicap * 4, 128);
    L.stage_bytes = up(L.st_q + L.qcap * 8, 128);
    return L;
}

size_t layout_bytes(const StLayout &L) { return (size_t)L.off_stage + (size_t)L.nst * L.stage_bytes; }

}  // namespace
}  // namespace sb

using namespace sb;

extern "C" {

int sb_bs6_staged_init(int32_t K, int32_t p, int32_t z0, int32_t z1, int32_t c_lo, int32_t c_hi, int32_t ey,
                       int32_t ez, int32_t w, sb_bs6_staged_t *info) {
    clear_error();
    if (!info || K < 1 || p < 1 || z0 < 0 || z1 > K || z0 >= z1 || c_lo < 0 || c_hi > K * p + 1 || c_lo >= c_hi) {
        set_error("sb_bs6_staged_init: invalid geometry");
        return SB_E_INVALID;
    }
    if (ey <= 0 || ez <= 0 || w <= 0) {  // defaults by order (measured, profiles/r02_bs6_staged.md)
        if (p == 1) {
            ey = 2; ez = 2; w = 32;
        } else if (p == 2) {
            ey = 2; ez = 2; w = 16;
        } else {
            set_error("sb_bs6_staged_init: no default tile for p = %d (the staged kernel is for p <= 2)", p);
            return SB_E_INVALID;
        }
    }
    const int64_t g = (int64_t)K * p + 1;
    const int Pb = ey * p, Pc = ez * p;
    if ((int64_t)Pb * Pc > kMaxSeg || (int64_t)(ey + 1) * (ez + 1) > kMaxRun || w > 1024 ||
        (int64_t)Pb * Pc * ((w + 31) / 32) > 32) {
        set_error("sb_bs6_staged_init: tile %d x %d elements x %d rows too large", ey, ez, w);
        return SB_E_INVALID;
    }
    sb_bs6_staged_t I{};
    I.K = K; I.p = p; I.z0 = z0; I.z1 = z1; I.c_lo = c_lo; I.c_hi = c_hi;
    I.ey = ey; I.ez = ez; I.w = w;
    I.max_segments = Pb * Pc;
    I.max_runs = (ey + 1) * (ez + 1);
    I.words_per_tile = table_layout(I.max_segments, I.max_runs, I.max_segments * ((w + 31) / 32)).D;
    // per-axis bounds: a window of n lattice points holds <= n + ceil(n/p)
    // entries per row-line direction and touches <= floor((n-1)/p) + 2 elements
    const int n3 = (p + 1) * (p + 1) * (p + 1);
    const int ex = (w - 1) / p + 2;
    const int vt = (w + (w + p - 1) / p) * (Pb + ey) * (Pc + ez);
    I.vt_cap = (vt + 255) / 256 * 256;  // the value-tile swizzle permutes within 256-entry groups
    I.ci_cap = vt + 8 * I.max_segments;
    I.rs_cap = I.max_segments * (w + 8);
    I.q_cap = I.max_runs * (ex * n3 + 2 + 16);
    const int64_t na = (g + w - 1) / w, nb = (g + Pb - 1) / Pb, nc = (c_hi - c_lo + Pc - 1) / Pc;
    I.n_tiles = na * nb * nc;
    I.n_local = (int64_t)K * K * (z1 - z0) * n3;
    *info = I;
    return SB_OK;
}

int sb_bs6_staged_make_plan(const sb_bs6_staged_t *info, const int32_t *row_starts, int32_t *plan, sb_stream_t s) {
    clear_error();
    if (!info || !row_starts || !plan || info->n_tiles < 0) {
        set_error("sb_bs6_staged_make_plan: invalid arguments");
        return SB_E_INVALID;
    }
    if (info->n_tiles == 0) return SB_OK;
    const int64_t g = (int64_t)info->K * info->p + 1;
    const StGeom G{info->K, info->p, info->z0, info->z1, info->c_lo, info->c_hi, info->ey, info->ez, info->w,
                   (int)g, (g + info->w - 1) / info->w, (g + info->ey * info->p - 1) / (info->ey * info->p)};
    const StLayout L = full_layout(*info, 2);
    if (L.D != info->words_per_tile) {
        set_error("sb_bs6_staged_make_plan: info does not come from sb_bs6_staged_init");
        return SB_E_INVALID;
    }
    const int64_t grid = std::min<int64_t>((info->n_tiles + 127) / 128, (int64_t)sm_count() * 32);
    k_bs6_staged_plan<<<(unsigned)std::max<int64_t>(1, grid), 128, 0, as_stream(s)>>>(G, L, row_starts, plan,
                                                                                     info->n_tiles);
    return launch_check("sb_bs6_staged_make_plan");
}

int sb_bs6_gather_staged(const sb_bs6_staged_t *info, const int32_t *plan, const int32_t *rs, const int32_t *ci,
                         int64_t ng, int64_t nl, const double *q, double *out, const double *carry, int64_t ncarry,
                         sb_stream_t s) {
    clear_error();
    if (!info || ng < 0 || nl < 0 || ncarry < 0 || (ncarry > 0 && !carry) || (info->n_tiles > 0 && !plan) ||
        (ng > 0 && (!rs || !out)) || (nl > 0 && (!ci || !q)) || info->max_segments < 1 ||
        info->max_segments > kMaxSeg || info->max_runs < 1 || info->max_runs > kMaxRun || info->w < 1 ||
        info->w > 1024) {
        set_error("sb_bs6_gather_staged: invalid arguments");
        return SB_E_INVALID;
    }
    if (!aligned16(plan) || !aligned16(rs) || !aligned16(ci) || !aligned16(q)) {
        set_error("sb_bs6_gather_staged: plan, row_starts, col_ids and q_local must be 16-byte aligned");
        return SB_E_INVALID;
    }
    if (ng == 0 || info->n_tiles == 0) return SB_OK;
    if (ncarry > ng) ncarry = ng;
    static const char *nst_env = getenv("SB200_BS6_STAGES");
    static const char *nwc_env = getenv("SB200_BS6_NWC");
    int nst = std::min(kStMaxNst, std::max(2, nst_env ? atoi(nst_env) : 3));
    const int nwc = nwc_env && atoi(nwc_env) == 4 ? 4 : 8;
    StLayout L = full_layout(*info, nst);
    while (nst > 2 && layout_bytes(L) > 227 * 1024) L = full_layout(*info, --nst);  // large tiles: fewer stages
    if (L.D != info->words_per_tile) {
        set_error("sb_bs6_gather_staged: info does not come from sb_bs6_staged_init");
        return SB_E_INVALID;
    }
    const size_t bytes = layout_bytes(L);
    if (bytes > 227 * 1024) {
        set_error("sb_bs6_gather_staged: tile needs %zu B of shared memory", bytes);
        return SB_E_INVALID;
    }
    const bool swz = info->p == 1;
    using KernT = void (*)(const int32_t *, int64_t, StLayout, const int32_t *, int64_t, const int32_t *, int64_t,
                           const double *, int64_t, double *, const double *, int64_t, int);
    static const char *np_env = getenv("SB200_BS6_NP");
    const int np = np_env && atoi(np_env) == 1 ? 1 : (np_env && atoi(np_env) == 4 ? 4 : 2);
#define SB_KS(SW_) (nwc == 4 ? (np == 1 ? k_bs6_staged<SW_, 4, 1> : np == 2 ? k_bs6_staged<SW_, 4, 2> : k_bs6_staged<SW_, 4, 4>) \
                            : (np == 1 ? k_bs6_staged<SW_, 8, 1> : np == 2 ? k_bs6_staged<SW_, 8, 2> : k_bs6_staged<SW_, 8, 4>))
    const KernT k = swz ? SB_KS(true) : SB_KS(false);
#undef SB_KS
    int rc = cuda_check(cudaFuncSetAttribute((const void *)k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes),
                        "sb_bs6_gather_staged: shared memory");
    if (rc) return rc;
    const int threads = (nwc + np) * 32;
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void *)k, threads, bytes);
    const int64_t grid = std::min<int64_t>(info->n_tiles, (int64_t)sm_count() * std::max(1, per_sm));
    static int dbg = getenv("SB200_BS6_DEBUG") ? 1 : 0;
    if (dbg == 1) {
        dbg = 2;
        fprintf(stderr,
                "sb_bs6_gather_staged: %d x %d x %d tile, %d warps + producer, %d stages, %zu B smem, "
                "%d CTAs/SM, grid %lld, %lld tiles of %d words, %d producer warps\n",
                info->ey, info->ez, info->w, nwc, nst, bytes, per_sm, (long long)grid, (long long)info->n_tiles,
                L.D, np);
    }
    static const char *mode_env = getenv("SB200_BS6_MODE");  // 1: consumers skip the work (pipeline probe)
    k<<<(unsigned)grid, threads, bytes, as_stream(s)>>>(plan, info->n_tiles, L, rs, ng, ci, nl, q, info->n_local, out,
                                                       carry, ncarry, mode_env ? atoi(mode_env) : 0);
    return launch_check("sb_bs6_gather_staged");
}

}  // extern "C"
