// stkde_trace_comm.cu -- per-phase timing + NVTX ranges, and the NCCL gather of per-rank
// slabs (include/stkde.h).
//
// Phase timing (SURVEY.md §5 "CUDA events per phase ... NVTX ranges"): a call records one
// event at its start and one at the end of every phase, all on the caller's stream; the
// interval between consecutive marks is charged to the phase that ends there.  Events are
// skipped while the stream is being captured (a graph replays the same kernels; time it
// from outside).  NVTX v3 is header-only: without an attached tool a range costs a branch.
//
// Gather: the hot path has no collective.  The optional whole-grid
// gather is NCCL point-to-point inside one ncclGroup: every rank sends its slab, the root
// receives all of them.  An x-slab is a contiguous block of the T-innermost grid, so the
// root receives it in place; a time slab is strided, so it is received into staging and
// unpacked by launch_gather.  NCCL is dlopen'ed at first use so the library has no link-time
// dependency on it (it loads and computes without NCCL; only these calls need it).
#include <dlfcn.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "stkde_internal.cuh"

using namespace stkde;

#define CK(call)                                                                          \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess) {                                                          \
            set_error("%s failed: %s", #call, cudaGetErrorString(e_));                    \
            return STKDE_ECUDA;                                                           \
        }                                                                                 \
    } while (0)

static const char *const kPhaseName[STKDE_NPHASES] = {"prep", "sort", "scan", "scatter",
                                                      "chords", "worklist", "tiles", "gather"};
static const char *const kNvtxName[STKDE_NPHASES] = {"stkde.prep", "stkde.sort", "stkde.scan",
                                                     "stkde.scatter", "stkde.chords", "stkde.worklist",
                                                     "stkde.tiles", "stkde.gather"};

// ------------------------------------------------------------ phase timing ---
static void phase_harvest(stkde_plan_s *p) {
    if (p->ph_used == 0) return;
    cudaEventSynchronize(p->ph_ev[p->ph_used - 1]);
    for (int k = 1; k < p->ph_used; ++k) {
        const int ph = p->ph_id[k];
        float ms = 0.f;
        if (ph >= 0 && cudaEventElapsedTime(&ms, p->ph_ev[k - 1], p->ph_ev[k]) == cudaSuccess)
            p->ph_ms[ph] += ms;
    }
    p->ph_used = 0;
}

static bool capturing(cudaStream_t st) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    return cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone;
}

static void phase_record(stkde_plan_s *p, cudaStream_t st, int id) {
    if (p->ph_used == p->ph_cap) {          // ring full: fold what is recorded, keep the last mark
        const int8_t last = p->ph_id[p->ph_used - 1];
        phase_harvest(p);
        std::swap(p->ph_ev[0], p->ph_ev[p->ph_cap - 1]);
        p->ph_id[0] = last;
        p->ph_used = 1;
    }
    cudaEventRecord(p->ph_ev[p->ph_used], st);
    p->ph_id[p->ph_used] = (int8_t)id;
    p->ph_used += 1;
}

namespace stkde {
void phase_call_begin(stkde_plan_s *p, cudaStream_t st) {
    if (!p->ph_on || capturing(st)) return;
    phase_record(p, st, -1);
    p->ph_calls += 1;
}

void phase_begin(int ph) { nvtxRangePushA(kNvtxName[ph]); }

void phase_end(stkde_plan_s *p, cudaStream_t st, int ph) {
    nvtxRangePop();
    if (!p->ph_on || p->ph_used == 0 || capturing(st)) return;
    phase_record(p, st, ph);
}
}  // namespace stkde

extern "C" int stkde_plan_enable_phase_timing(stkde_plan_t p, int enable) {
    if (!p) { set_error("plan is NULL"); return STKDE_EINVAL; }
    CK(cudaSetDevice(p->device));
    if (enable && !p->ph_ev) {
        const int cap = 4096;
        p->ph_ev = (cudaEvent_t *)calloc(cap, sizeof(cudaEvent_t));
        p->ph_id = (int8_t *)calloc(cap, 1);
        if (!p->ph_ev || !p->ph_id) { set_error("host allocation failed"); return STKDE_ENOMEM; }
        for (int i = 0; i < cap; ++i) CK(cudaEventCreate(&p->ph_ev[i]));
        p->ph_cap = cap;
    }
    p->ph_used = 0;
    p->ph_on = enable ? 1 : 0;
    for (double &m : p->ph_ms) m = 0.0;
    p->ph_calls = 0;
    return STKDE_OK;
}

extern "C" int stkde_plan_phase_ms(stkde_plan_t p, double *ms, int64_t *calls) {
    if (!p || !ms) { set_error("NULL argument"); return STKDE_EINVAL; }
    CK(cudaSetDevice(p->device));
    if (p->ph_used > 0) {
        // keep the last mark so a call still being enqueued keeps its reference point
        const int8_t last = p->ph_id[p->ph_used - 1];
        const int used = p->ph_used;
        phase_harvest(p);
        std::swap(p->ph_ev[0], p->ph_ev[used - 1]);
        p->ph_id[0] = last;
        p->ph_used = 1;
    }
    for (int i = 0; i < STKDE_NPHASES; ++i) ms[i] = p->ph_ms[i];
    if (calls) *calls = p->ph_calls;
    return STKDE_OK;
}

extern "C" const char *stkde_phase_name(int phase) {
    return (phase >= 0 && phase < STKDE_NPHASES) ? kPhaseName[phase] : nullptr;
}

// ------------------------------------------------------------------- NCCL ---
namespace {
struct Nccl {
    bool tried = false, ok = false;
    char why[256] = "";
    decltype(&ncclGetUniqueId) getUniqueId = nullptr;
    decltype(&ncclCommInitRank) commInitRank = nullptr;
    decltype(&ncclCommDestroy) commDestroy = nullptr;
    decltype(&ncclGroupStart) groupStart = nullptr;
    decltype(&ncclGroupEnd) groupEnd = nullptr;
    decltype(&ncclSend) send = nullptr;
    decltype(&ncclRecv) recv = nullptr;
    decltype(&ncclGetErrorString) errorString = nullptr;
};
Nccl g_nccl;
std::mutex g_nccl_mu;

// resolve NCCL once; the soname already loaded in the process (e.g. torch's) wins
bool nccl_load() {
    std::lock_guard<std::mutex> lk(g_nccl_mu);
    if (g_nccl.tried) return g_nccl.ok;
    g_nccl.tried = true;
    const char *env = getenv("STKDE_NCCL_LIB");
    void *h = dlopen(env && *env ? env : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
        snprintf(g_nccl.why, sizeof g_nccl.why, "NCCL not available: %s", dlerror());
        return false;
    }
#define SYM(field, name)                                                                      \
    g_nccl.field = reinterpret_cast<decltype(g_nccl.field)>(dlsym(h, name));                \
    if (!g_nccl.field) {                                                                      \
        snprintf(g_nccl.why, sizeof g_nccl.why, "NCCL library lacks %s", name);              \
        return false;                                                                         \
    }
    SYM(getUniqueId, "ncclGetUniqueId")
    SYM(commInitRank, "ncclCommInitRank")
    SYM(commDestroy, "ncclCommDestroy")
    SYM(groupStart, "ncclGroupStart")
    SYM(groupEnd, "ncclGroupEnd")
    SYM(send, "ncclSend")
    SYM(recv, "ncclRecv")
    SYM(errorString, "ncclGetErrorString")
#undef SYM
    g_nccl.ok = true;
    return true;
}
}  // namespace

#define NCK(call)                                                                         \
    do {                                                                                  \
        ncclResult_t r_ = (call);                                                         \
        if (r_ != ncclSuccess) {                                                          \
            set_error("%s failed: %s", #call, g_nccl.errorString(r_));                    \
            return STKDE_ENCCL;                                                           \
        }                                                                                 \
    } while (0)

static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");

extern "C" int stkde_nccl_unique_id(void *h_id) {
    if (!h_id) { set_error("h_id is NULL"); return STKDE_EINVAL; }
    if (!nccl_load()) { set_error("%s", g_nccl.why); return STKDE_ENCCL; }
    ncclUniqueId id;
    NCK(g_nccl.getUniqueId(&id));
    memcpy(h_id, &id, sizeof id);
    return STKDE_OK;
}

namespace stkde {
void trace_comm_release(stkde_plan_s *p) {
    if (p->comm && g_nccl.ok) g_nccl.commDestroy((ncclComm_t)p->comm);
    p->comm = nullptr;
    if (p->gather_stage) cudaFree(p->gather_stage);
    p->gather_stage = nullptr;
    p->gather_stage_bytes = 0;
    if (p->ph_ev)
        for (int i = 0; i < p->ph_cap; ++i) cudaEventDestroy(p->ph_ev[i]);
    free(p->ph_ev);
    free(p->ph_id);
    p->ph_ev = nullptr;
    p->ph_id = nullptr;
}
}  // namespace stkde

extern "C" int stkde_plan_comm_init(stkde_plan_t p, int nranks, int rank, const void *h_id) {
    if (!p || !h_id) { set_error("NULL argument"); return STKDE_EINVAL; }
    if (nranks < 1 || rank < 0 || rank >= nranks) {
        set_error("rank %d / nranks %d: need 0 <= rank < nranks", rank, nranks);
        return STKDE_EINVAL;
    }
    if (!nccl_load()) { set_error("%s", g_nccl.why); return STKDE_ENCCL; }
    CK(cudaSetDevice(p->device));
    if (p->comm) {
        g_nccl.commDestroy((ncclComm_t)p->comm);
        p->comm = nullptr;
    }
    ncclUniqueId id;
    memcpy(&id, h_id, sizeof id);
    ncclComm_t c = nullptr;
    NCK(g_nccl.commInitRank(&c, nranks, id, rank));
    p->comm = c;
    p->comm_rank = rank;
    p->comm_nranks = nranks;
    return STKDE_OK;
}

// shared validation of the two gathers; `extent` = Gx (x-slabs) or Gt (time slabs)
static int gather_check(stkde_plan_s *p, const float *d_slab, const int64_t *h_cuts, int root, int64_t extent) {
    if (!p) { set_error("plan is NULL"); return STKDE_EINVAL; }
    if (!p->comm) { set_error("the plan has no communicator (stkde_plan_comm_init)"); return STKDE_EINVAL; }
    if (!h_cuts || !d_slab) { set_error("NULL argument"); return STKDE_EINVAL; }
    const int R = p->comm_nranks;
    if (root < 0 || root >= R) { set_error("root %d outside [0, %d)", root, R); return STKDE_EINVAL; }
    if (h_cuts[0] != 0 || h_cuts[R] != extent) {
        set_error("cuts must run from 0 to %lld", (long long)extent);
        return STKDE_EINVAL;
    }
    for (int r = 0; r < R; ++r)
        if (h_cuts[r + 1] < h_cuts[r]) { set_error("cuts must be ascending"); return STKDE_EINVAL; }
    return STKDE_OK;
}

extern "C" int stkde_gather_xslab(stkde_plan_t p, const float *d_slab, const int64_t *h_cuts, int root,
                                  float *d_full, void *stream) {
    int rc = gather_check(p, d_slab, h_cuts, root, p ? p->g.Gx : 0);
    if (rc) return rc;
    const int R = p->comm_nranks, me = p->comm_rank;
    if (me == root && !d_full) { set_error("d_full is NULL on the root"); return STKDE_EINVAL; }
    cudaStream_t st = (cudaStream_t)stream;
    CK(cudaSetDevice(p->device));
    const size_t row = (size_t)p->g.Gy * p->g.Gt;          // floats per x row
    phase_call_begin(p, st);
    Phase ph_(p, st, STKDE_PHASE_GATHER);
    ncclComm_t c = (ncclComm_t)p->comm;
    const size_t mine = (size_t)(h_cuts[me + 1] - h_cuts[me]) * row;
    NCK(g_nccl.groupStart());
    if (me == root) {
        for (int r = 0; r < R; ++r) {
            const size_t cnt = (size_t)(h_cuts[r + 1] - h_cuts[r]) * row;
            float *dst = d_full + (size_t)h_cuts[r] * row;
            if (cnt == 0 || (r == me && dst == d_slab)) continue;
            if (r == me) {
                if (cudaMemcpyAsync(dst, d_slab, cnt * sizeof(float), cudaMemcpyDeviceToDevice, st) != cudaSuccess) {
                    g_nccl.groupEnd();
                    set_error("root slab copy failed");
                    return STKDE_ECUDA;
                }
            } else {
                NCK(g_nccl.recv(dst, cnt, ncclFloat32, r, c, st));
            }
        }
    } else if (mine > 0) {
        NCK(g_nccl.send(d_slab, mine, ncclFloat32, root, c, st));
    }
    NCK(g_nccl.groupEnd());
    return STKDE_OK;
}

extern "C" int stkde_gather_slab(stkde_plan_t p, const float *d_slab, const int64_t *h_cuts, int root,
                                 float *d_full, void *stream) {
    int rc = gather_check(p, d_slab, h_cuts, root, p ? p->g.Gt : 0);
    if (rc) return rc;
    const int R = p->comm_nranks, me = p->comm_rank;
    if (me == root && !d_full) { set_error("d_full is NULL on the root"); return STKDE_EINVAL; }
    cudaStream_t st = (cudaStream_t)stream;
    CK(cudaSetDevice(p->device));
    const GridParams &g = p->g;
    const size_t plane = (size_t)g.Gx * g.Gy;               // floats per layer of a slab
    ncclComm_t c = (ncclComm_t)p->comm;
    phase_call_begin(p, st);
    Phase ph_(p, st, STKDE_PHASE_GATHER);
    if (me != root) {
        const size_t cnt = (size_t)(h_cuts[me + 1] - h_cuts[me]) * plane;
        if (cnt > 0) {
            NCK(g_nccl.groupStart());
            NCK(g_nccl.send(d_slab, cnt, ncclFloat32, root, c, st));
            NCK(g_nccl.groupEnd());
        }
        return STKDE_OK;
    }
    // root: stage every other slab, then unpack all of them (its own straight from d_slab)
    size_t need = 0;
    for (int r = 0; r < R; ++r)
        if (r != me) need += (size_t)(h_cuts[r + 1] - h_cuts[r]) * plane * sizeof(float);
    if (need > p->gather_stage_bytes) {
        if (p->gather_stage) CK(cudaFree(p->gather_stage));
        p->gather_stage = nullptr;
        p->gather_stage_bytes = 0;
        if (cudaMalloc(&p->gather_stage, need) != cudaSuccess) {
            set_error("gather staging allocation of %zu bytes failed", need);
            return STKDE_ENOMEM;
        }
        p->gather_stage_bytes = need;
    }
    NCK(g_nccl.groupStart());
    size_t off = 0;
    for (int r = 0; r < R; ++r) {
        const size_t cnt = (size_t)(h_cuts[r + 1] - h_cuts[r]) * plane;
        if (r == me || cnt == 0) continue;
        NCK(g_nccl.recv(p->gather_stage + off, cnt, ncclFloat32, r, c, st));
        off += cnt;
    }
    NCK(g_nccl.groupEnd());
    off = 0;
    for (int r = 0; r < R; ++r) {
        const size_t cnt = (size_t)(h_cuts[r + 1] - h_cuts[r]) * plane;
        if (cnt == 0) continue;
        const float *src = r == me ? d_slab : p->gather_stage + off;
        if (launch_gather(src, g.Gx, g.Gy, g.Gt, h_cuts[r], h_cuts[r + 1], d_full, st)) {
            set_error("unpack kernel launch failed");
            return STKDE_ECUDA;
        }
        if (r != me) off += cnt;
    }
    return STKDE_OK;
}

// ---- direct x-slab gather over peer memory (CUDA IPC) ----
// The allocation base of d_ptr comes from the driver's cuMemGetAddressRange (runtime
// driver entry point: no link-time libcuda).
extern "C" int stkde_ipc_get_handle(const void *d_ptr, void *h_handle, int64_t *offset) {
    if (!d_ptr || !h_handle || !offset) { set_error("NULL argument"); return STKDE_EINVAL; }
    typedef int (*range_fn)(unsigned long long *, size_t *, unsigned long long);
    static range_fn range = nullptr;
    if (!range) {
        void *fp = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fp, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !fp) {
            set_error("cuMemGetAddressRange is not available");
            return STKDE_ECUDA;
        }
        range = (range_fn)fp;
    }
    unsigned long long base = 0;
    size_t size = 0;
    if (range(&base, &size, (unsigned long long)(uintptr_t)d_ptr) != 0) {
        set_error("cuMemGetAddressRange failed (not device memory?)");
        return STKDE_ECUDA;
    }
    cudaIpcMemHandle_t h;
    const cudaError_t e = cudaIpcGetMemHandle(&h, (void *)(uintptr_t)base);
    if (e != cudaSuccess) { set_error("cudaIpcGetMemHandle: %s", cudaGetErrorString(e)); return STKDE_ECUDA; }
    memcpy(h_handle, &h, sizeof h);
    *offset = (int64_t)((uintptr_t)d_ptr - (uintptr_t)base);
    return STKDE_OK;
}

extern "C" int stkde_ipc_open(int device, const void *h_handle, void **d_base) {
    if (!h_handle || !d_base) { set_error("NULL argument"); return STKDE_EINVAL; }
    int cur = 0;
    cudaGetDevice(&cur);
    cudaError_t e = cudaSetDevice(device);
    if (e == cudaSuccess) {
        cudaIpcMemHandle_t h;
        memcpy(&h, h_handle, sizeof h);
        e = cudaIpcOpenMemHandle(d_base, h, cudaIpcMemLazyEnablePeerAccess);
    }
    cudaSetDevice(cur);
    if (e != cudaSuccess) { set_error("cudaIpcOpenMemHandle: %s", cudaGetErrorString(e)); return STKDE_ECUDA; }
    return STKDE_OK;
}

extern "C" int stkde_ipc_close(void *d_base) {
    if (!d_base) { set_error("NULL argument"); return STKDE_EINVAL; }
    const cudaError_t e = cudaIpcCloseMemHandle(d_base);
    if (e != cudaSuccess) { set_error("cudaIpcCloseMemHandle: %s", cudaGetErrorString(e)); return STKDE_ECUDA; }
    return STKDE_OK;
}
