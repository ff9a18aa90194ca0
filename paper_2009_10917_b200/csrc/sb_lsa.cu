// sb_lsa.cu -- host side of the fused multi-GPU reductions (sb_lsa.cuh).
//
// The NCCL host API (communicator, symmetric window, device communicator) is
// resolved at run time from the libnccl.so.2 already loaded by the process
// (torch's, NCCL 2.28) with dlsym, so libsb200.so itself has no link-time
// NCCL dependency; the device half is NCCL's header-only device API.
#include <dlfcn.h>
#include <string.h>

#include <new>

#include "sb_lsa.cuh"

namespace sb {

struct NcclApi {
    bool ok = false;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *);
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int);
    ncclResult_t (*CommDestroy)(ncclComm_t);
    ncclResult_t (*CommAbort)(ncclComm_t);
    ncclResult_t (*MemAlloc)(void **, size_t);
    ncclResult_t (*MemFree)(void *);
    ncclResult_t (*CommWindowRegister)(ncclComm_t, void *, size_t, ncclWindow_t *, int);
    ncclResult_t (*CommWindowDeregister)(ncclComm_t, ncclWindow_t);
    ncclResult_t (*DevCommCreate)(ncclComm_t, const ncclDevCommRequirements_t *, ncclDevComm_t *);
    ncclResult_t (*DevCommDestroy)(ncclComm_t, const ncclDevComm_t *);
    ncclTeam_t (*TeamLsa)(ncclComm_t);
    const char *(*GetErrorString)(ncclResult_t);
    ncclResult_t (*GetVersion)(int *);
};

static NcclApi &nccl_api() {
    static NcclApi api = [] {
        NcclApi a;
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return a;
#define SB_SYM(F) a.F = reinterpret_cast<decltype(a.F)>(dlsym(h, "nccl" #F))
        SB_SYM(GetUniqueId);
        SB_SYM(CommInitRank);
        SB_SYM(CommDestroy);
        SB_SYM(CommAbort);
        SB_SYM(MemAlloc);
        SB_SYM(MemFree);
        SB_SYM(CommWindowRegister);
        SB_SYM(CommWindowDeregister);
        SB_SYM(DevCommCreate);
        SB_SYM(DevCommDestroy);
        SB_SYM(TeamLsa);
        SB_SYM(GetErrorString);
        SB_SYM(GetVersion);
#undef SB_SYM
        a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.CommAbort && a.MemAlloc && a.MemFree &&
               a.CommWindowRegister && a.CommWindowDeregister && a.DevCommCreate && a.DevCommDestroy &&
               a.TeamLsa && a.GetErrorString && a.GetVersion;
        return a;
    }();
    return api;
}

}  // namespace sb

struct sb_lsa {
    ncclComm_t comm = nullptr;
    void *buf = nullptr;
    ncclWindow_t win{};
    ncclDevComm dc{};
    bool has_win = false, has_dc = false;
    int nranks = 0, rank = 0;
    long long calls = 0;
    // BS6 carry halo window (sb_lsa_halo_window): 2 x plane doubles
    void *hbuf = nullptr;
    ncclWindow_t hwin{};
    bool has_hwin = false;
    size_t hbytes = 0;
};

namespace sb {
__global__ void k_lsa_peer_ptr(ncclWindow_t w, size_t off, int peer, void **out) {
    *out = ncclGetLsaPointer(w, off, peer);
}
// (cnt: a call counter in this rank's memory, advanced after the barrier --
// the BS7 halo buffers' parity, read by the put before and the split scatter
// after it, dist.py DistScatter)
__global__ void k_lsa_barrier(ncclDevComm dc, unsigned long long *cnt) {
    ncclLsaBarrierSession<ncclCoopThread> bar(ncclCoopThread(), dc, ncclTeamTagLsa(), 0);
    bar.sync(ncclCoopThread(), cuda::memory_order_acq_rel);
    if (cnt) *cnt += 1;
}
}  // namespace sb

using namespace sb;

static int nccl_check(ncclResult_t r, const char *what) {
    if (r == ncclSuccess) return SB_OK;
    set_error("%s: %s", what, nccl_api().GetErrorString ? nccl_api().GetErrorString(r) : "nccl error");
    return SB_E_CUDA;
}

static int need_api(const char *what) {
    if (nccl_api().ok) {
        int v = 0;
        nccl_api().GetVersion(&v);
        if (v >= 22800) return SB_OK;
        set_error("%s: libnccl.so.2 is version %d, the device API needs >= 2.28", what, v);
        return SB_E_INVALID;
    }
    set_error("%s: libnccl.so.2 (>= 2.28, with the device API) is not loadable", what);
    return SB_E_INVALID;
}

static void lsa_free(sb_lsa_t *c) {
    NcclApi &a = nccl_api();
    if (c->has_hwin) a.CommWindowDeregister(c->comm, c->hwin);
    if (c->hbuf) a.MemFree(c->hbuf);
    if (c->has_dc) a.DevCommDestroy(c->comm, &c->dc);
    if (c->has_win) a.CommWindowDeregister(c->comm, c->win);
    if (c->buf) a.MemFree(c->buf);
    if (c->comm) a.CommDestroy(c->comm);
    delete c;
}

extern "C" {

int sb_lsa_available(void) {
    clear_error();
    return need_api("sb_lsa_available");
}

int sb_lsa_unique_id(void *out, size_t bytes) {
    clear_error();
    if (int rc = need_api("sb_lsa_unique_id")) return rc;
    if (!out || bytes < sizeof(ncclUniqueId)) {
        set_error("sb_lsa_unique_id: need a %zu-byte buffer", sizeof(ncclUniqueId));
        return SB_E_INVALID;
    }
    ncclUniqueId id;
    if (int rc = nccl_check(nccl_api().GetUniqueId(&id), "ncclGetUniqueId")) return rc;
    memcpy(out, &id, sizeof(id));
    return SB_OK;
}

int sb_lsa_create(const void *uid, size_t bytes, int nranks, int rank, sb_lsa_t **out) {
    clear_error();
    if (int rc = need_api("sb_lsa_create")) return rc;
    if (!uid || bytes < sizeof(ncclUniqueId) || nranks < 1 || nranks > kLsaMaxRanks || rank < 0 ||
        rank >= nranks || !out) {
        set_error("sb_lsa_create: invalid arguments (1 <= nranks <= %d)", kLsaMaxRanks);
        return SB_E_INVALID;
    }
    NcclApi &a = nccl_api();
    sb_lsa_t *c = new (std::nothrow) sb_lsa_t;
    if (!c) return SB_E_INVALID;
    c->nranks = nranks;
    c->rank = rank;
    ncclUniqueId id;
    memcpy(&id, uid, sizeof(id));
    int rc = nccl_check(a.CommInitRank(&c->comm, nranks, id, rank), "ncclCommInitRank");
    if (!rc) {
        const ncclTeam_t t = a.TeamLsa(c->comm);
        if (t.nRanks != nranks) {
            set_error("sb_lsa_create: %d of %d ranks are NVLink (LSA) peers; the fused path needs all", t.nRanks,
                      nranks);
            rc = SB_E_INVALID;
        }
    }
    const size_t wbytes = kLsaWindowBytes;  // slots [2][kLsaMaxRanks] + the call counter
    if (!rc) rc = nccl_check(a.MemAlloc(&c->buf, wbytes), "ncclMemAlloc");
    if (!rc) rc = cuda_check(cudaMemset(c->buf, 0, wbytes), "sb_lsa_create memset");
    if (!rc) {
        rc = nccl_check(a.CommWindowRegister(c->comm, c->buf, wbytes, &c->win, NCCL_WIN_COLL_SYMMETRIC),
                        "ncclCommWindowRegister");
        c->has_win = rc == SB_OK;
    }
    if (!rc) {
        ncclDevCommRequirements_t req;
        memset(&req, 0, sizeof(req));
        req.lsaBarrierCount = 1;
        rc = nccl_check(a.DevCommCreate(c->comm, &req, &c->dc), "ncclDevCommCreate");
        c->has_dc = rc == SB_OK;
    }
    if (!rc) rc = cuda_check(cudaDeviceSynchronize(), "sb_lsa_create");
    if (rc) {
        // local teardown: the peers may be anywhere in the setup, so no
        // collective deregistration (it could wait for a rank that failed
        // before registering); the small symmetric buffers are left to exit
        if (c->comm) a.CommAbort(c->comm);
        delete c;
        return rc;
    }
    *out = c;
    return SB_OK;
}

// Local teardown for when the ranks disagree (some failed sb_lsa_create):
// no collective call (window deregistration / device-communicator destroy
// may wait for peers that never registered), just ncclCommAbort; the small
// symmetric buffers are left to process exit.
int sb_lsa_abort(sb_lsa_t *ctx) {
    clear_error();
    if (!ctx) return SB_OK;
    cudaDeviceSynchronize();
    if (ctx->comm) nccl_api().CommAbort(ctx->comm);
    delete ctx;
    return SB_OK;
}

int sb_lsa_destroy(sb_lsa_t *ctx) {
    clear_error();
    if (!ctx) return SB_OK;
    cudaDeviceSynchronize();
    lsa_free(ctx);
    return SB_OK;
}

static LsaArgs lsa_args(sb_lsa_t *c) {
    LsaArgs L{};
    L.dc = c->dc;
    L.win = c->win;
    L.epoch = (int)(c->calls++ & 1);  // (informational; the kernels use the window's counter)
    L.enabled = 1;
    return L;
}

int sb_lsa_halo_window(sb_lsa_t *ctx, size_t bytes) {
    clear_error();
    if (!ctx || bytes == 0 || ctx->has_hwin) {
        set_error("sb_lsa_halo_window: invalid arguments (one halo window per context)");
        return SB_E_INVALID;
    }
    NcclApi &a = nccl_api();
    int rc = nccl_check(a.MemAlloc(&ctx->hbuf, bytes), "ncclMemAlloc");
    if (!rc) rc = cuda_check(cudaMemset(ctx->hbuf, 0, bytes), "sb_lsa_halo_window memset");
    if (!rc) {
        rc = nccl_check(a.CommWindowRegister(ctx->comm, ctx->hbuf, bytes, &ctx->hwin, NCCL_WIN_COLL_SYMMETRIC),
                        "ncclCommWindowRegister");
        ctx->has_hwin = rc == SB_OK;
    }
    if (!rc) rc = cuda_check(cudaDeviceSynchronize(), "sb_lsa_halo_window");
    if (!rc) ctx->hbytes = bytes;
    return rc;
}

int sb_lsa_halo_pointers(sb_lsa_t *ctx, size_t offset, int peer, void **local, void **remote) {
    clear_error();
    if (!ctx || !ctx->has_hwin || offset >= ctx->hbytes || peer < 0 || peer >= ctx->nranks) {
        set_error("sb_lsa_halo_pointers: invalid arguments");
        return SB_E_INVALID;
    }
    if (local) *local = static_cast<char *>(ctx->hbuf) + offset;
    if (remote) {
        void **d = nullptr;
        int rc = cuda_check(cudaMalloc(&d, sizeof(void *)), "sb_lsa_halo_pointers");
        if (rc) return rc;
        k_lsa_peer_ptr<<<1, 1>>>(ctx->hwin, offset, peer, d);
        rc = cuda_check(cudaMemcpy(remote, d, sizeof(void *), cudaMemcpyDeviceToHost), "sb_lsa_halo_pointers");
        cudaFree(d);
        if (rc) return rc;
    }
    return SB_OK;
}

int sb_lsa_barrier(sb_lsa_t *ctx, sb_stream_t s) {
    clear_error();
    if (!ctx) {
        set_error("sb_lsa_barrier: null context");
        return SB_E_INVALID;
    }
    k_lsa_barrier<<<1, 1, 0, as_stream(s)>>>(ctx->dc, nullptr);
    return launch_check("sb_lsa_barrier");
}

int sb_lsa_barrier_advance(sb_lsa_t *ctx, unsigned long long *call_count, sb_stream_t s) {
    clear_error();
    if (!ctx || !call_count) {
        set_error("sb_lsa_barrier_advance: null argument");
        return SB_E_INVALID;
    }
    k_lsa_barrier<<<1, 1, 0, as_stream(s)>>>(ctx->dc, call_count);
    return launch_check("sb_lsa_barrier_advance");
}

int sb_lsa_cg_pap(const double *p, const double *ap, int64_t n, int64_t bs, int64_t nb, void *ws, sb_cg_state *st,
                  sb_lsa_t *ctx, sb_stream_t s) {
    clear_error();
    if (!ctx) { set_error("sb_lsa_cg_pap: null context"); return SB_E_INVALID; }
    const LsaArgs L = lsa_args(ctx);
    return cg_pap_impl(p, ap, n, bs, nb, ws, st, &L, as_stream(s));
}

int sb_lsa_cg_update(int fused, const double *p, const double *ap, double *x, double *r, int64_t n, int64_t bs,
                     int64_t nb, void *ws, sb_cg_state *st, sb_lsa_t *ctx, sb_stream_t s) {
    clear_error();
    if (!ctx) { set_error("sb_lsa_cg_update: null context"); return SB_E_INVALID; }
    const LsaArgs L = lsa_args(ctx);
    return cg_update_impl(fused, p, ap, x, r, n, bs, nb, ws, st, &L, as_stream(s));
}

int sb_lsa_bs3_norm2(const double *x, int64_t n, int64_t bs, int64_t nb, void *ws, double *result, sb_lsa_t *ctx,
                     sb_stream_t s) {
    clear_error();
    if (!ctx) { set_error("sb_lsa_bs3_norm2: null context"); return SB_E_INVALID; }
    return lsa_reduce(0, 0.0, x, x, nullptr, nullptr, n, bs, nb, ws, result, lsa_args(ctx), as_stream(s),
                      "sb_lsa_bs3_norm2");
}

int sb_lsa_bs4_dot(const double *x, const double *y, int64_t n, int64_t bs, int64_t nb, void *ws, double *result,
                   sb_lsa_t *ctx, sb_stream_t s) {
    clear_error();
    if (!ctx) { set_error("sb_lsa_bs4_dot: null context"); return SB_E_INVALID; }
    return lsa_reduce(1, 0.0, x, y, nullptr, nullptr, n, bs, nb, ws, result, lsa_args(ctx), as_stream(s),
                      "sb_lsa_bs4_dot");
}

int sb_lsa_bs5_fused_cg_update(double alpha, const double *p, const double *ap, double *x, double *r, int64_t n,
                               int64_t bs, int64_t nb, void *ws, double *result, sb_lsa_t *ctx, sb_stream_t s) {
    clear_error();
    if (!ctx) { set_error("sb_lsa_bs5_fused_cg_update: null context"); return SB_E_INVALID; }
    return lsa_reduce(2, alpha, p, ap, x, r, n, bs, nb, ws, result, lsa_args(ctx), as_stream(s),
                      "sb_lsa_bs5_fused_cg_update");
}

}  // extern "C"
