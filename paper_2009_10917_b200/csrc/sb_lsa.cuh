// sb_lsa.cuh -- multi-GPU scalar combine fused into the reduction kernels,
// over NVLink load/store-accessible (LSA) peer memory with the NCCL 2.28
// device API (BS3/BS4/BS5 + allreduce in one launch).
//
// Each rank's lattice kernel ends in one CTA holding the rank's scalar.  That
// CTA stores it into slot [epoch][rank] of every peer's symmetric window
// (plain st.global through the NVLink mapping), meets the peers at an LSA
// barrier (acq_rel), and sums slots [epoch][0..world) from +0.0 in rank order
// -- the same value, bit for bit, as dist.py's all-gather + sb_sum_ordered
// path, with no collective launch, proxy thread or extra stream round trip.
// Two slot sets (epoch = call parity) keep a fast rank's next call from
// overwriting values a slow rank has not read yet: reaching call k+2 needs
// every peer past call k+1's barrier, hence done reading call k.  The parity
// comes from a call counter in this rank's window (kLsaCounterOff), read and
// advanced by the combining thread -- never from the host, so a CUDA graph
// that captured an odd number of calls still alternates across replays.
#pragma once

#include <nccl.h>
#include <nccl_device.h>

#include "sb_common.cuh"

namespace sb {

constexpr int kLsaMaxRanks = 128;  // slots per epoch (NVLink domains up to NVL72)
constexpr size_t kLsaCounterOff = 2 * kLsaMaxRanks * sizeof(double);  // uint64 call counter
constexpr size_t kLsaWindowBytes = kLsaCounterOff + 64;

struct LsaArgs {
    ncclDevComm dc;
    ncclWindow_t win;  // 2 x kLsaMaxRanks doubles, symmetric over the LSA team
    int epoch;         // (unused: the parity is device-side, kLsaCounterOff)
    int enabled;
};

// Thread 0 of the reduction's last CTA.
__device__ __forceinline__ double lsa_combine(const LsaArgs &L, double v) {
    const ncclTeam lsa = ncclTeamLsa(L.dc);
    volatile unsigned long long *calls =
        static_cast<volatile unsigned long long *>(ncclGetLocalPointer(L.win, kLsaCounterOff));
    const unsigned long long call = *calls;
    *calls = call + 1;  // (stream-ordered: the next combine runs in a later launch)
    const size_t base = (size_t)(call & 1) * kLsaMaxRanks;
    for (int p = 0; p < lsa.nRanks; p++) {
        double *dst = static_cast<double *>(ncclGetLsaPointer(L.win, sizeof(double) * (base + lsa.rank), p));
        *reinterpret_cast<volatile double *>(dst) = v;
    }
    ncclLsaBarrierSession<ncclCoopThread> bar(ncclCoopThread(), L.dc, ncclTeamTagLsa(), 0);
    bar.sync(ncclCoopThread(), cuda::memory_order_acq_rel);
    const volatile double *mine =
        static_cast<const volatile double *>(ncclGetLocalPointer(L.win, sizeof(double) * base));
    double acc = 0.0;
    for (int p = 0; p < lsa.nRanks; p++) acc = __dadd_rn(acc, mine[p]);
    return acc;
}

int lsa_reduce(int mode, double alpha, const double *u, const double *v, double *x, double *r, int64_t n,
               int64_t bs, int64_t nb, void *ws, double *result, const LsaArgs &lsa, cudaStream_t st,
               const char *name);

}  // namespace sb
