// sb_gs_pipe.cu -- BS6 gather (persistent, software-pipelined) and BS7 scatter.
//
// The gather/scatter chains are index -> value -> store: dependent DRAM round
// trips.  The one-tile-per-CTA kernels in sb_gs.cu pay them serially inside
// each CTA (block_starts -> row_starts -> col_ids -> q -> sum -> store), which
// leaves HBM half idle (ncu: ~50% DRAM throughput, long-scoreboard bound).
// Here each CTA is persistent and prefetches the *indices of the next tile*
// (and, for BS6, the plan entry of the tile after that) into registers while
// the current tile's value gathers are in flight, so every iteration exposes a
// single round trip and ~30 KB per CTA stay in flight.  (A cp.async/LDGSTS
// 3-stage variant of this pipeline was measured slower: MIO-throttle bound on
// the 8-byte gathers; so was a two-deep variant that overlapped one
// super-block's row sums with the next one's gathers.)
//
// BS6 is bounded by the L1 data pipe as much as by DRAM (ncu at N=7, product
// kernel: l1tex wavefronts 79% of peak, DRAM 76%; the r01 kernel was at 78% /
// 66%): every gather instruction costs one L1 tag lookup per distinct 128 B
// line its lanes touch, and the one-thread-per-row sums cost shared-memory
// wavefronts.  The kernels below are shaped to cut both; ~20 variants that
// did not (TMA-fed, two-deep, row-mapped, partner plans, TMA gather4, ...)
// are recorded in profiles/r01_bs6_variants.md.
//
// Results are bitwise those of the one-tile kernels: BS6 still sums each row
// in ascending column order from +0.0 (or the carry-in) in one thread.
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <mutex>
#include <unordered_map>

#include "sb_common.cuh"

namespace sb {

// BS6: many small CTAs beat few large ones (measured on B200, K=66 N=7: CAP
// 2048 x 256 thr x 3 CTA/SM 4.47 TB/s; CAP 512 x 128 thr x 12 CTA/SM 5.72 TB/s)
constexpr int kBs6T = 128;
constexpr int kBs6Cap = 512;   // entries per BS6 super-block (4 per thread)
constexpr int kBs6MinCtas = 12;

// ---- BS7 ----------------------------------------------------------------
// One entry per lane per load: a warp instruction covers 32 consecutive
// local entries (ids: one 128 B row; gathers: ~32/(p+1)+1 element-edge runs;
// stores: two 128 B rows), where the int4 kernel above spreads a warp over
// 128 entries and pays more L1 tag lookups per instruction.
// SPLIT: q_global lives in two pieces -- ids < split index `qg`, ids >= split
// index `qh` (the multi-GPU slab's own rows and the halo plane written over
// NVLink by the rank above, dist.py DistScatter.enable_lsa).  With `cnt` the
// halo is one of two alternating buffers, qh or qh1 by the call count the
// LSA barrier advanced just before (buffer (cnt - 1) & 1): the parity lives in
// device memory, so CUDA-graph replays alternate correctly.
template <int T, int U, bool MASK, bool SPLIT = false>
__global__ void __launch_bounds__(T) k_bs7_lanes(const int32_t *__restrict__ ids, int64_t nl,
                                                const double *__restrict__ qg, double *__restrict__ ql,
                                                int32_t split = 0, const double *__restrict__ qh = nullptr,
                                                const double *__restrict__ qh1 = nullptr,
                                                const unsigned long long *__restrict__ cnt = nullptr) {
    if (SPLIT && cnt && ((*cnt - 1) & 1)) qh = qh1;
    const uint64_t pol = policy_evict_last();
    const int64_t base = (int64_t)blockIdx.x * T * U + threadIdx.x;
    int32_t d[U];
#pragma unroll
    for (int j = 0; j < U; j++)
        if (base + j * T < nl) d[j] = ld_stream(ids + base + j * T);
    double v[U];
#pragma unroll
    for (int j = 0; j < U; j++)
        if (base + j * T < nl && (!MASK || d[j] >= 0))
            v[j] = (!SPLIT || d[j] < split) ? ld_keep(qg + d[j], pol) : ld_keep(qh + (d[j] - split), pol);
#pragma unroll
    for (int j = 0; j < U; j++)
        if (base + j * T < nl && (!MASK || d[j] >= 0)) st_stream(ql + base + j * T, v[j]);
}

int bs7_split_launch(const int32_t *ids, int64_t nl, const double *qg, int32_t split, const double *qh,
                     const double *qh1, const unsigned long long *cnt, double *ql, int has_mask, cudaStream_t st) {
    constexpr int T = 128, U = 4;
    const unsigned grid = (unsigned)std::max<int64_t>(1, (nl + T * U - 1) / (T * U));
    if (has_mask)
        k_bs7_lanes<T, U, true, true><<<grid, T, 0, st>>>(ids, nl, qg, ql, split, qh, qh1, cnt);
    else
        k_bs7_lanes<T, U, false, true><<<grid, T, 0, st>>>(ids, nl, qg, ql, split, qh, qh1, cnt);
    return launch_check("sb_bs7_scatter_split");
}

// BS7 halo put: n doubles of src into dst0 or dst1 by the parity of the call
// count *cnt (read before the LSA barrier advances it; dist.py DistScatter)
__global__ void k_halo_put(const double *__restrict__ src, double *dst0, double *dst1, int64_t n,
                           const unsigned long long *__restrict__ cnt) {
    double *dst = (*cnt & 1) ? dst1 : dst0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = ld_stream(src + i);
}

int halo_put_launch(const double *src, double *dst0, double *dst1, int64_t n, const unsigned long long *cnt,
                    cudaStream_t st) {
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)sm_count() * 8));
    k_halo_put<<<(unsigned)grid, 256, 0, st>>>(src, dst0, dst1, n, cnt);
    return launch_check("sb_bs7_halo_put");
}

int bs7_lanes_launch(const int32_t *ids, int64_t nl, const double *qg, double *ql, int has_mask,
                     cudaStream_t st) {
    // 128 threads x 4 entries per CTA, one tile per CTA (an oversubscribed
    // grid: CTA scheduling balances the tail).  Measured on B200 over N = 1..15
    // against int4 ids / double2 stores (the r01 kernel), entry pairs and other
    // tile shapes (profiles/r01_bs7_variants.md): +8% at N=7, +37% at N=4.
    constexpr int T = 128, U = 4;
    const unsigned grid = (unsigned)std::max<int64_t>(1, (nl + T * U - 1) / (T * U));
    if (has_mask)
        k_bs7_lanes<T, U, true><<<grid, T, 0, st>>>(ids, nl, qg, ql);
    else
        k_bs7_lanes<T, U, false><<<grid, T, 0, st>>>(ids, nl, qg, ql);
    return launch_check("sb_bs7_scatter");
}

// ---- BS6 ----------------------------------------------------------------
// plan[2i] = first row of super-block i, plan[2i+1] = its first entry;
// super-block i = operator blocks [i*G, (i+1)*G), G = max(1, CAP/npb), so a
// super-block has <= CAP entries and <= CAP rows (rows are non-empty).
// plan[2 (nsb+1)] (the trailer word, zeroed by the host first) is set when a
// super-block holds more than CAP rows or entries (empty rows, or a
// hand-built block_starts -- never from build_gather).  sb_bs6_make_plan reads
// it back once and records the plan as oversize; sb_bs6_gather_planned then
// sums its rows straight from global memory (bs6_rows_launch).  (A check
// inside the kernels cost 2-10% even at entry: profiles/r02_bs6_sweep.md.)
__global__ void k_bs6_plan(const int32_t *bst, int64_t nblk, const int32_t *rs, int G, int64_t nsb,
                           int32_t *plan) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= nsb;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = i * G < nblk ? i * G : nblk;
        const int32_t r = bst[b];
        const int32_t e = rs[r];
        plan[2 * i] = r;
        plan[2 * i + 1] = e;
        if (i < nsb) {
            const int64_t bn = (i + 1) * G < nblk ? (i + 1) * G : nblk;
            const int32_t rn = bst[bn];
            if ((int64_t)rn - r > kBs6Cap || (int64_t)rs[rn] - e > kBs6Cap) atomicOr(plan + 2 * (nsb + 1), 1);
        }
    }
}

struct SbMeta {
    int32_t r0, e0, r1, e1;
};

// Kernel super-block i = PS consecutive plan super-blocks (rows never split:
// plan boundaries are operator-block boundaries); nsbk = ceil(nsb / PS).
template <int PS>
__device__ __forceinline__ SbMeta load_meta_ps(const int32_t *plan, int64_t i, int64_t nsbk, int64_t nsb) {
    SbMeta m{0, 0, 0, 0};
    if (i < nsbk) {
        const int64_t j = PS * i + PS < nsb ? PS * i + PS : nsb;
        const int2 lo = __ldg(reinterpret_cast<const int2 *>(plan + 2 * PS * i));
        const int2 hi = __ldg(reinterpret_cast<const int2 *>(plan + 2 * j));
        m = SbMeta{lo.x, lo.y, hi.x, hi.y};
    }
    return m;
}

__device__ __forceinline__ SbMeta load_meta(const int32_t *plan, int64_t i, int64_t nsb) {
    SbMeta m{0, 0, 0, 0};
    if (i < nsb) {
        const int2 lo = __ldg(reinterpret_cast<const int2 *>(plan + 2 * i));
        const int2 hi = __ldg(reinterpret_cast<const int2 *>(plan + 2 * i + 2));
        m = SbMeta{lo.x, lo.y, hi.x, hi.y};
    }
    return m;
}

// Shared-memory slot of super-block entry k.  With long rows (p = 1: 8
// entries) the one-thread-per-row sums read qs[8l + j] across lanes l -- a
// 16-way bank conflict; XOR-ing the low 4 bits of the double index with bits
// 4..7 makes those reads 2 wavefronts (the minimum for 32 x 8 B).  For the
// 1-2 entry rows of p >= 7 the lanes' first entries spread over ~48-90
// doubles and collide 3-4 ways; the same swizzle measured +7% there, and
// -5% at p = 3..5, so SWZ is chosen per operator from the mean row length.
template <bool SWZ>
__device__ __forceinline__ int qslot(int k) {
    return SWZ ? (k ^ ((k >> 4) & 15)) : k;
}

template <int T, int CAP, bool SWZ>
__device__ __forceinline__ void bs6_issue_vals(const SbMeta &m, const int2 (&cols)[CAP / (2 * T)],
                                               const double *__restrict__ q, double2 (&v)[CAP / (2 * T)]) {
    constexpr int M = CAP / (2 * T);
    const int ne = m.e1 - m.e0;
#pragma unroll
    for (int j = 0; j < M; j++) {
        const int k = 2 * (threadIdx.x + j * T);
        if (k + 1 < ne) {
            if (cols[j].y == cols[j].x + 1 && aligned16(q + cols[j].x)) {
                v[j] = __ldg(reinterpret_cast<const double2 *>(q + cols[j].x));
            } else {
                v[j].x = __ldg(q + cols[j].x);
                v[j].y = __ldg(q + cols[j].y);
            }
        } else if (k < ne) {
            v[j].x = __ldg(q + cols[j].x);
        }
    }
}

template <int T, int CAP>
__device__ __forceinline__ void bs6_issue_cols(const SbMeta &m, const int32_t *__restrict__ ci,
                                               int2 (&cols)[CAP / (2 * T)]) {
    constexpr int M = CAP / (2 * T);
    const int ne = m.e1 - m.e0;
#pragma unroll
    for (int j = 0; j < M; j++) {
        const int k = 2 * (threadIdx.x + j * T);
        if (k < ne) cols[j].x = ld_stream(ci + m.e0 + k);
        if (k + 1 < ne) cols[j].y = ld_stream(ci + m.e0 + k + 1);
    }
}

// Row starts stay in registers: thread t owns rows t + j*T of its
// super-block; the end of row k is the start of row k+1 (a shuffle; lane 31
// loads it).  The row loop is not unrolled (rows are 1-8 entries long) and
// output / carry addressing is 32-bit per super-block.
template <int T, int CAP>
struct Bs6Rows {
    static constexpr int R = (CAP + T - 1) / T;  // rows per thread (rows <= CAP)
    int32_t lo[R], hi31[R];                      // row start; lane 31: start of the next row
};

template <int T, int CAP>
__device__ __forceinline__ void bs6_load_rows(const SbMeta &m, const int32_t *__restrict__ rs,
                                              Bs6Rows<T, CAP> &rw) {
    const int nrows = m.r1 - m.r0;
    const int32_t *base = rs + m.r0;
    const bool last = (threadIdx.x & 31) == 31;
#pragma unroll
    for (int j = 0; j < Bs6Rows<T, CAP>::R; j++) {
        const int k = threadIdx.x + j * T;
        if (k <= nrows) rw.lo[j] = ld_stream(base + k);  // row k+1's start ends row k
        if (last && k < nrows) rw.hi31[j] = __ldg(base + k + 1);
    }
}

template <int T, int CAP, bool SWZ>
__device__ __forceinline__ void bs6_row_sums(const SbMeta &m, const Bs6Rows<T, CAP> &rw, const double *qs,
                                             double *__restrict__ out, const double *__restrict__ carry,
                                             int64_t ncarry) {
    const int nrows = m.r1 - m.r0;
    const bool last = (threadIdx.x & 31) == 31;
    double *ob = out + m.r0;
    const int ncar = ncarry > m.r0 ? (int)std::min<int64_t>(ncarry - m.r0, (int64_t)nrows) : 0;
    const double *cb = carry + m.r0;
#pragma unroll
    for (int j = 0; j < Bs6Rows<T, CAP>::R; j++) {
        const int k = threadIdx.x + j * T;
        int b = __shfl_down_sync(0xffffffffu, rw.lo[j], 1);
        if (last) b = rw.hi31[j];
        if (k < nrows) {
            int c = rw.lo[j] - m.e0;
            b -= m.e0;
            double acc = k < ncar ? cb[k] : 0.0;
#pragma unroll 1
            for (; c < b; c++) acc = add(acc, qs[qslot<SWZ>(c)]);
            st_stream(ob + k, acc);
        }
    }
}

template <int T, int CAP, bool SWZ>
__device__ __forceinline__ void bs6_publish_vals(const SbMeta &m, const double2 (&v)[CAP / (2 * T)], double *qs) {
    constexpr int M = CAP / (2 * T);
    const int ne = m.e1 - m.e0;
#pragma unroll
    for (int j = 0; j < M; j++) {
        const int k = 2 * (threadIdx.x + j * T);
        if (SWZ) {
            if (k < ne) qs[qslot<SWZ>(k)] = v[j].x;
            if (k + 1 < ne) qs[qslot<SWZ>(k + 1)] = v[j].y;
        } else if (k + 1 < ne) {
            *reinterpret_cast<double2 *>(&qs[k]) = v[j];
        } else if (k < ne) {
            qs[k] = v[j].x;
        }
    }
}

// Pairs kernel (long rows, p <= 1): thread t owns the entry pairs (2t, 2t+1)
// and (2t+2T, 2t+2T+1) of its super-block, gathered with one 16 B load when
// the two columns are adjacent (the 8-entry rows of p = 1 meshes pair up
// often enough for that to beat one entry per lane).
template <int T, int CAP, bool SWZ, int MINB = kBs6MinCtas, int PS = 1>
__global__ void __launch_bounds__(T, MINB) k_bs6_pairs(const int32_t *__restrict__ plan, int64_t nsb,
                                                             const int32_t *__restrict__ rs,
                                                             const int32_t *__restrict__ ci,
                                                             const double *__restrict__ q,
                                                             double *__restrict__ out,
                                                             const double *__restrict__ carry, int64_t ncarry) {
    constexpr int M = CAP / (2 * T);
    extern __shared__ __align__(16) unsigned char bs6_smem[];
    double(*qs)[CAP] = reinterpret_cast<double(*)[CAP]>(bs6_smem);
    const int64_t g = gridDim.x;
    const int64_t nsbk = (nsb + PS - 1) / PS;
    int64_t sbi = blockIdx.x;
    if (sbi >= nsbk) return;
    int2 cols[M];
    double2 v[M];
    Bs6Rows<T, CAP> rw;
    int buf = 0;
    SbMeta mc = load_meta_ps<PS>(plan, sbi, nsbk, nsb), mn = load_meta_ps<PS>(plan, sbi + g, nsbk, nsb);
    bs6_issue_cols<T, CAP>(mc, ci, cols);
    for (; sbi < nsbk; sbi += g) {
        bs6_issue_vals<T, CAP, SWZ>(mc, cols, q, v);  // A: values of this super-block
        bs6_load_rows<T, CAP>(mc, rs, rw);             // B: its row starts
        bs6_issue_cols<T, CAP>(mn, ci, cols);          // C: indices of the next one
        const SbMeta mnn = load_meta_ps<PS>(plan, sbi + 2 * g, nsbk, nsb);
        bs6_publish_vals<T, CAP, SWZ>(mc, v, qs[buf]);
        __syncthreads();
        bs6_row_sums<T, CAP, SWZ>(mc, rw, qs[buf], out, carry, ncarry);
        buf ^= 1;  // the next iteration's barrier orders reuse of this buffer
        mc = mn;
        mn = mnn;
    }
}

// Lanes kernel (short rows, p >= 2): one entry per lane per load.
// The q gathers are L1-tag bound (ncu: l1tex 78-91% busy at N=7): an
// instruction costs one tag lookup per distinct 128 B line its lanes touch.
// With one entry per lane, a warp instruction covers 32 consecutive entries
// (4 element-edge runs of 8 at N=7 -> ~4 lines) whatever the parity of the
// run starts, and the column loads are fully coalesced 128 B rows; paired
// 16 B gathers only pay off when a run starts on an even entry.
template <int T, int CAP, bool SWZ, int MINB = kBs6MinCtas>
__global__ void __launch_bounds__(T, MINB) k_bs6_lanes(const int32_t *__restrict__ plan, int64_t nsb,
                                                             const int32_t *__restrict__ rs,
                                                             const int32_t *__restrict__ ci,
                                                             const double *__restrict__ q,
                                                             double *__restrict__ out,
                                                             const double *__restrict__ carry, int64_t ncarry) {
    constexpr int E = CAP / T;  // entries per thread
    extern __shared__ __align__(16) unsigned char bs6_smem[];
    double(*qs)[CAP] = reinterpret_cast<double(*)[CAP]>(bs6_smem);
    const int64_t g = gridDim.x;
    int64_t sbi = blockIdx.x;
    if (sbi >= nsb) return;
    int32_t col[E];
    Bs6Rows<T, CAP> rw;
    int buf = 0;
    SbMeta mc = load_meta(plan, sbi, nsb), mn = load_meta(plan, sbi + g, nsb);
    {
        const int ne = mc.e1 - mc.e0;
#pragma unroll
        for (int j = 0; j < E; j++)
            if ((int)threadIdx.x + j * T < ne) col[j] = ld_stream(ci + mc.e0 + threadIdx.x + j * T);
    }
    for (; sbi < nsb; sbi += g) {
        const int ne = mc.e1 - mc.e0;
        double v[E];
#pragma unroll
        for (int j = 0; j < E; j++)
            if ((int)threadIdx.x + j * T < ne) v[j] = __ldg(q + col[j]);
        bs6_load_rows<T, CAP>(mc, rs, rw);
        const int nne = mn.e1 - mn.e0;
#pragma unroll
        for (int j = 0; j < E; j++)
            if ((int)threadIdx.x + j * T < nne) col[j] = ld_stream(ci + mn.e0 + threadIdx.x + j * T);
        const SbMeta mnn = load_meta(plan, sbi + 2 * g, nsb);
#pragma unroll
        for (int j = 0; j < E; j++)
            if ((int)threadIdx.x + j * T < ne) qs[buf][qslot<SWZ>(threadIdx.x + j * T)] = v[j];
        __syncthreads();
        bs6_row_sums<T, CAP, SWZ>(mc, rw, qs[buf], out, carry, ncarry);
        buf ^= 1;
        mc = mn;
        mn = mnn;
    }
}

int bs6_rows_launch(const int32_t *rs, const int32_t *ci, int64_t ng, const double *q, double *out,
                    const double *carry, int64_t ncarry, cudaStream_t st);  // sb_gs.cu

static int64_t bs6_G(int64_t npb) { return std::max<int64_t>(1, kBs6Cap / npb); }

// Kernel, value-tile swizzle and CTAs per SM of the planned gather, by the
// mean row length rho = nl/ng (measured on B200 over N = 1..15,
// profiles/r01_bs6_variants.md):
//   rho >= 4    (p = 1)   pairs, swizzled, 1024-entry super-blocks (two plan
//                         super-blocks each), 6 CTAs/SM (+3-6% over 512
//                         entries at 12/SM) once the operator fills two waves
//                         of them; else 512 entries, 12/SM
//   rho >= 3    (p = 2)   lanes, plain,    12 CTAs/SM
//   rho >= 2.2  (p = 3)   lanes, swizzled,  8 CTAs/SM (64 registers)
//   rho <  2.2  (p >= 4)  lanes, plain,    10 CTAs/SM (48 registers)
// SB200_BS6_CFG="<lanes|pairs|wide|rows>,<swizzle 0|1>,<CTAs/SM 6|8|10|12>"
// overrides the choice (A/B runs, scripts/expt/time_bs6.py; read per call).
struct Bs6Choice {
    bool rows, pairs, sw, wide;
    int mb;
};
static Bs6Choice bs6_choose(int64_t nsb, int64_t ng, int64_t nl) {
    Bs6Choice c{false, false, false, false, 10};
    if (nl >= 4 * ng) {
        // wide only when every SM gets at least two of its super-blocks: on
        // small operators half as many CTAs is a longer critical path
        c.pairs = true; c.sw = true; c.mb = 12;
        c.wide = nsb >= 2 * 2 * 6 * (int64_t)sm_count();
    } else if (nl >= 3 * ng) {
        c.mb = 12;
    } else if (5 * nl >= 11 * ng) {
        c.sw = true; c.mb = 8;
    }
    const char *cfg = getenv("SB200_BS6_CFG");
    if (cfg && strncmp(cfg, "rows", 4) == 0) {
        c.rows = true;
    } else if (cfg) {
        c.wide = cfg[0] == 'w';  // "wide": the 1024-entry pairs kernel
        c.pairs = cfg[0] == 'p' || c.wide;
        const char *c1 = strchr(cfg, ',');
        c.sw = c1 && c1[1] == '1';
        const char *c2 = c1 ? strchr(c1 + 1, ',') : nullptr;
        c.mb = c2 ? atoi(c2 + 1) : 12;
    }
    return c;
}

// plans sb_bs6_make_plan found oversize (keyed by the plan's address; a new
// plan built at the same address overwrites its entry)
static std::mutex g_plan_mu;
static std::unordered_map<const int32_t *, bool> g_plan_oversize;

// ---- BS6 + the multi-GPU carry halo in ONE launch ------
// Rank r of a z-slab partition (dist.py DistGather) computes the partial sums
// of its top interface plane (the "send" operator) and hands them to rank
// r+1, which seeds those rows with them (carry) -- bitwise the 1-GPU gather
// (SURVEY Appendix A.4).  Here both operators run in one persistent kernel:
// virtual super-block v < nsb_send is a send super-block (its row sums are
// stored straight into rank r+1's carry buffer, an NVLink-mapped address),
// v >= nsb_send an own one; CTAs take v in increasing order, so every send
// super-block is issued before any own one.  Protocol, all state in device
// memory (so CUDA-graph replays stay correct; the host never tracks parity):
//   sync[0] ready  -- written by rank r-1: its call e's carry is complete (e+1)
//   sync[1] ack    -- written by rank r+1: it consumed call e's carry (e+1)
//   sync[2] epoch  -- this rank's call count e (carry buffer e & 1)
//   sync[3], [4]   -- CTA counters (send phase done, kernel done)
// * before storing call e's partials into buffer e&1 of rank r+1: wait until
//   ack >= e-1 (rank r+1 has consumed call e-2, the buffer's last user);
// * the last CTA through the send phase publishes peer_ready = e+1 after a
//   system-scope fence (every CTA fences its stores before counting);
// * before reading carry rows: wait until ready >= e+1;
// * the last CTA out stores peer_ack = e+1 into rank r-1 and advances epoch.
// No wait depends on this rank's own later work, and every CTA is resident
// (grid = occupancy x SMs), so the kernel cannot deadlock against itself.
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t *p) {
    uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(uint64_t *p, uint64_t v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void wait_at_least(const uint64_t *flag, uint64_t v) {
    while (ld_acquire_sys(flag) < v) __nanosleep(64);
}

struct Bs6HaloArgs {
    const int32_t *plan[2];   // send, own
    int64_t nsb[2];
    const int32_t *rs[2], *ci[2];
    double *send_out[2];      // rank r+1's carry buffers (NVLink-mapped), by epoch parity
    double *own_out;
    const double *carry[2];   // this rank's carry buffers (written by rank r-1)
    int64_t ncarry;
    const double *q;
    uint64_t *sync;           // this rank's ready / ack / epoch / counters
    uint64_t *peer_ready;     // rank r+1's sync[0] (NULL on the last rank)
    uint64_t *peer_ack;       // rank r-1's sync[1] (NULL on the first rank)
};

template <int T, int CAP, bool SWZ, int MINB>
__global__ void __launch_bounds__(T, MINB) k_bs6_halo(Bs6HaloArgs A) {
    constexpr int E = CAP / T;
    extern __shared__ __align__(16) unsigned char bs6_smem[];
    double(*qs)[CAP] = reinterpret_cast<double(*)[CAP]>(bs6_smem);
    __shared__ uint64_t s_epoch;
    if (threadIdx.x == 0) s_epoch = *reinterpret_cast<volatile uint64_t *>(A.sync + 2);
    __syncthreads();
    const uint64_t epoch = s_epoch;
    const int par = (int)(epoch & 1);
    const int64_t g = gridDim.x, nsend = A.nsb[0], ntot = A.nsb[0] + A.nsb[1];
    auto meta = [&](int64_t v) { return v < nsend ? load_meta(A.plan[0], v, nsend) : load_meta(A.plan[1], v - nsend, A.nsb[1]); };
    bool send_counted = false, acked = false, readied = false;
    auto count_send = [&]() {  // this CTA is past its last send super-block
        __threadfence_system();  // every thread's stores into rank r+1's buffer
        __syncthreads();
        if (threadIdx.x == 0) {
            const unsigned long long old = atomicAdd(reinterpret_cast<unsigned long long *>(A.sync + 3), 1ull);
            if (old == (unsigned long long)(g - 1)) {
                A.sync[3] = 0;
                __threadfence_system();
                if (A.peer_ready) st_release_sys(A.peer_ready, epoch + 1);
            }
        }
        send_counted = true;
    };
    int64_t v = blockIdx.x;
    int32_t col[E];
    Bs6Rows<T, CAP> rw;
    int buf = 0;
    if (v < ntot) {
        SbMeta mc = meta(v), mn = meta(v + g);
        int side = v < nsend ? 0 : 1;
        {
            const int ne = mc.e1 - mc.e0;
#pragma unroll
            for (int j = 0; j < E; j++)
                if ((int)threadIdx.x + j * T < ne) col[j] = ld_stream(A.ci[side] + mc.e0 + threadIdx.x + j * T);
        }
        for (; v < ntot; v += g) {
            const int nside = v + g < nsend ? 0 : 1;
            if (side == 1 && !send_counted) count_send();
            const int ne = mc.e1 - mc.e0;
            double vv[E];
#pragma unroll
            for (int j = 0; j < E; j++)
                if ((int)threadIdx.x + j * T < ne) vv[j] = __ldg(A.q + col[j]);
            bs6_load_rows<T, CAP>(mc, A.rs[side], rw);
            const int nne = mn.e1 - mn.e0;
#pragma unroll
            for (int j = 0; j < E; j++)
                if ((int)threadIdx.x + j * T < nne) col[j] = ld_stream(A.ci[nside] + mn.e0 + threadIdx.x + j * T);
            const SbMeta mnn = meta(v + 2 * g);
#pragma unroll
            for (int j = 0; j < E; j++)
                if ((int)threadIdx.x + j * T < ne) qs[buf][qslot<SWZ>(threadIdx.x + j * T)] = vv[j];
            if (side == 0 && !acked) {  // rank r+1 is done with this buffer's previous contents
                if (threadIdx.x == 0 && epoch >= 2) wait_at_least(A.sync + 1, epoch - 1);
                acked = true;
            }
            const bool carry_rows = side == 1 && mc.r0 < A.ncarry;
            if (carry_rows && !readied) {  // rank r-1's partials of this call have landed
                if (threadIdx.x == 0) wait_at_least(A.sync + 0, epoch + 1);
                readied = true;
            }
            __syncthreads();
            if (side == 0)
                bs6_row_sums<T, CAP, SWZ>(mc, rw, qs[buf], A.send_out[par], nullptr, 0);
            else
                bs6_row_sums<T, CAP, SWZ>(mc, rw, qs[buf], A.own_out, A.carry[par], carry_rows ? A.ncarry : 0);
            buf ^= 1;
            mc = mn;
            mn = mnn;
            side = nside;
        }
    }
    if (!send_counted) count_send();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned long long old = atomicAdd(reinterpret_cast<unsigned long long *>(A.sync + 4), 1ull);
        if (old == (unsigned long long)(g - 1)) {
            A.sync[4] = 0;
            A.sync[2] = epoch + 1;
            __threadfence_system();
            if (A.peer_ack) st_release_sys(A.peer_ack, epoch + 1);
        }
    }
}

}  // namespace sb

using namespace sb;

extern "C" {

int64_t sb_bs6_plan_size(int64_t n_blocks, int64_t npb) {
    if (n_blocks < 1 || npb < 1 || npb > kBs6Cap) return 0;
    const int64_t G = bs6_G(npb);
    return 2 * ((n_blocks + G - 1) / G + 1) + 2;  // + the oversize trailer (and its pad)
}

int sb_bs6_make_plan(const int32_t *bst, int64_t nblk, const int32_t *rs, int64_t npb, int32_t *plan,
                     sb_stream_t s) {
    clear_error();
    if (!bst || !rs || !plan || sb_bs6_plan_size(nblk, npb) == 0) {
        set_error("sb_bs6_make_plan: invalid arguments (nodes_per_block must be <= %d)", kBs6Cap);
        return SB_E_INVALID;
    }
    const int G = (int)bs6_G(npb);
    const int64_t nsb = (nblk + G - 1) / G;
    const int64_t grid = std::min<int64_t>((nsb + 256) / 256, (int64_t)sm_count() * 16);
    int rc = cuda_check(cudaMemsetAsync(plan + 2 * (nsb + 1), 0, 2 * sizeof(int32_t), as_stream(s)),
                        "sb_bs6_make_plan");
    if (rc) return rc;
    k_bs6_plan<<<(unsigned)std::max<int64_t>(1, grid), 256, 0, as_stream(s)>>>(bst, nblk, rs, G, nsb, plan);
    rc = launch_check("sb_bs6_make_plan");
    if (rc) return rc;
    // one-time readback of the trailer (a plan is built once per operator)
    int32_t flag = 0;
    rc = cuda_check(cudaMemcpyAsync(&flag, plan + 2 * (nsb + 1), sizeof(flag), cudaMemcpyDeviceToHost, as_stream(s)),
                    "sb_bs6_make_plan");
    if (!rc) rc = cuda_check(cudaStreamSynchronize(as_stream(s)), "sb_bs6_make_plan");
    if (rc) return rc;
    std::lock_guard<std::mutex> lk(g_plan_mu);
    g_plan_oversize[plan] = flag != 0;
    return SB_OK;
}

int sb_bs6_planned_kernel(int64_t n_blocks, int64_t nodes_per_block, int64_t ng, int64_t nl, char *name,
                          size_t cap) {
    clear_error();
    const int64_t psize = sb_bs6_plan_size(n_blocks, nodes_per_block);
    if (psize == 0 || !name || cap == 0) {
        set_error("sb_bs6_planned_kernel: invalid arguments");
        return SB_E_INVALID;
    }
    const Bs6Choice c = bs6_choose(psize / 2 - 2, ng, nl);
    if (c.rows)
        snprintf(name, cap, "k_bs6_rows");
    else if (c.wide)
        snprintf(name, cap, "k_bs6_pairs<128,1024,%s,6,2>", c.sw ? "swz" : "plain");
    else
        snprintf(name, cap, "%s<128,512,%s,%d>", c.pairs ? "k_bs6_pairs" : "k_bs6_lanes", c.sw ? "swz" : "plain",
                 c.mb);
    return SB_OK;
}

int sb_bs6_gather_halo(const int32_t *send_plan, int64_t send_nblk, const int32_t *send_rs,
                       const int32_t *send_ci, double *const send_out[2], const int32_t *own_plan,
                       int64_t own_nblk, const int32_t *own_rs, const int32_t *own_ci, int64_t own_ng,
                       double *own_out, const double *const carry[2], int64_t n_carry, int64_t npb,
                       const double *q, uint64_t *sync, uint64_t *peer_ready, uint64_t *peer_ack,
                       sb_stream_t s) {
    clear_error();
    const int64_t own_size = sb_bs6_plan_size(own_nblk, npb);
    const bool has_send = send_plan != nullptr;
    const int64_t send_size = has_send ? sb_bs6_plan_size(send_nblk, npb) : 0;
    if (own_size == 0 || !own_plan || !own_rs || !own_ci || !own_out || !q || !sync || n_carry < 0 ||
        (n_carry > 0 && (!carry || !carry[0] || !carry[1])) ||
        (has_send && (send_size == 0 || !send_rs || !send_ci || !send_out || !send_out[0] || !send_out[1])) ||
        (!has_send && peer_ready) || (n_carry == 0 && peer_ack)) {
        set_error("sb_bs6_gather_halo: invalid arguments");
        return SB_E_INVALID;
    }
    if ((reinterpret_cast<uintptr_t>(own_plan) | reinterpret_cast<uintptr_t>(send_plan) |
         reinterpret_cast<uintptr_t>(sync)) & 7u) {
        set_error("sb_bs6_gather_halo: plans and sync must be 8-byte aligned");
        return SB_E_INVALID;
    }
    {
        std::lock_guard<std::mutex> lk(g_plan_mu);
        for (const int32_t *pl : {own_plan, send_plan}) {
            const auto f = pl ? g_plan_oversize.find(pl) : g_plan_oversize.end();
            if (f != g_plan_oversize.end() && f->second) {
                set_error("sb_bs6_gather_halo: an operator's plan is oversize (use the unfused path)");
                return SB_E_INVALID;
            }
        }
    }
    if (n_carry > own_ng) n_carry = own_ng;
    Bs6HaloArgs A{};
    A.plan[0] = send_plan;
    A.plan[1] = own_plan;
    A.nsb[0] = has_send ? send_size / 2 - 2 : 0;
    A.nsb[1] = own_size / 2 - 2;
    A.rs[0] = has_send ? send_rs : own_rs;
    A.ci[0] = has_send ? send_ci : own_ci;
    A.rs[1] = own_rs;
    A.ci[1] = own_ci;
    A.send_out[0] = has_send ? send_out[0] : nullptr;
    A.send_out[1] = has_send ? send_out[1] : nullptr;
    A.own_out = own_out;
    A.carry[0] = n_carry ? carry[0] : nullptr;
    A.carry[1] = n_carry ? carry[1] : nullptr;
    A.ncarry = n_carry;
    A.q = q;
    A.sync = sync;
    A.peer_ready = peer_ready;
    A.peer_ack = peer_ack;
    constexpr int T = kBs6T;
    const size_t smem = 2 * kBs6Cap * sizeof(double);
    // one kernel shape for both operators: lanes, 10 CTAs/SM (48 registers)
    const auto k = k_bs6_halo<T, kBs6Cap, false, 10>;
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void *)k, T, smem);
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(A.nsb[0] + A.nsb[1], (int64_t)sm_count() * std::max(1, per_sm)));
    k<<<(unsigned)grid, T, smem, as_stream(s)>>>(A);
    return launch_check("sb_bs6_gather_halo");
}

int sb_bs6_gather_planned(const int32_t *plan, int64_t nblk, int64_t npb, const int32_t *rs,
                          const int32_t *ci, int64_t ng, int64_t nl, const double *q, double *out,
                          const double *carry, int64_t ncarry, sb_stream_t s) {
    clear_error();
    const int64_t psize = sb_bs6_plan_size(nblk, npb);
    if (ng < 0 || nl < 0 || ncarry < 0 || (ncarry > 0 && !carry) || !plan || psize == 0 ||
        (ng > 0 && (!rs || !out)) || (nl > 0 && (!ci || !q))) {
        set_error("sb_bs6_gather_planned: invalid arguments");
        return SB_E_INVALID;
    }
    if (reinterpret_cast<uintptr_t>(plan) & 7u) {
        set_error("sb_bs6_gather_planned: plan must be 8-byte aligned");
        return SB_E_INVALID;
    }
    if (ng == 0) return SB_OK;
    if (ncarry > ng) ncarry = ng;
    const int64_t nsb = psize / 2 - 2;
    {
        std::lock_guard<std::mutex> lk(g_plan_mu);
        const auto f = g_plan_oversize.find(plan);
        if (f != g_plan_oversize.end() && f->second) return bs6_rows_launch(rs, ci, ng, q, out, carry, ncarry, as_stream(s));
    }
    constexpr int T = kBs6T;
    const size_t smem = 2 * kBs6Cap * sizeof(double);
    using KernT = void (*)(const int32_t *, int64_t, const int32_t *, const int32_t *, const double *, double *,
                           const double *, int64_t);
    Bs6Choice ch = bs6_choose(nsb, ng, nl);
    if (ch.rows) return bs6_rows_launch(rs, ci, ng, q, out, carry, ncarry, as_stream(s));
    const bool pairs = ch.pairs, sw = ch.sw, wide = ch.wide;
    const int mb = ch.mb;
#define SB_PICK(K_, MB_) (sw ? K_<T, kBs6Cap, true, MB_> : K_<T, kBs6Cap, false, MB_>)
#define SB_PICK_MB(K_) (mb == 6 ? SB_PICK(K_, 6) : mb == 8 ? SB_PICK(K_, 8) : mb == 10 ? SB_PICK(K_, 10) : SB_PICK(K_, 12))
    auto grid_for = [&](const void *k) {
        int per_sm = 1;  // (8 KB of dynamic shared memory: below the default limit)
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, T, smem);
        return (unsigned)std::max<int64_t>(1, std::min<int64_t>(nsb, (int64_t)sm_count() * std::max(1, per_sm)));
    };
    if (wide) {
        constexpr int CAPW = 2 * kBs6Cap;
        const size_t smemw = 2 * CAPW * sizeof(double);
        const KernT kw = sw ? k_bs6_pairs<T, CAPW, true, 6, 2> : k_bs6_pairs<T, CAPW, false, 6, 2>;
        int per_sm = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void *)kw, T, smemw);
        const int64_t nsbk = (nsb + 1) / 2;
        const unsigned grid =
            (unsigned)std::max<int64_t>(1, std::min<int64_t>(nsbk, (int64_t)sm_count() * std::max(1, per_sm)));
        kw<<<grid, T, smemw, as_stream(s)>>>(plan, nsb, rs, ci, q, out, carry, ncarry);
        return launch_check("sb_bs6_gather_planned");
    }
    const KernT kern = pairs ? SB_PICK_MB(k_bs6_pairs) : SB_PICK_MB(k_bs6_lanes);
    kern<<<grid_for((const void *)kern), T, smem, as_stream(s)>>>(plan, nsb, rs, ci, q, out, carry, ncarry);
#undef SB_PICK_MB
#undef SB_PICK
    return launch_check("sb_bs6_gather_planned");
}

}  // extern "C"
