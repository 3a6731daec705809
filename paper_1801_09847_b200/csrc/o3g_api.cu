// o3g_api.cu — the C ABI of include/o3g.h: argument validation, the
// context (device buffers, grid build, source ordering), the graph-launched
// iteration loop and the multi-GPU exchange (NCCL, loaded at run time).
#include <dlfcn.h>
#include <nvtx3/nvToolsExt.h>   // header-only; a no-op unless a profiler injects itself
#include <stdio.h>
#include <stdlib.h>
#include <math.h>
#include <string.h>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <cub/iterator/counting_input_iterator.cuh>
#include <algorithm>
#include <string>
#include <vector>

#include "../../include/o3g.h"
#include "o3g_internal.cuh"

using namespace o3g;

// --------------------------------------------------------------- errors
static thread_local std::string g_err;

static o3g_status fail(o3g_status s, const std::string& msg) {
    g_err = msg;
    return s;
}

#define CK(call)                                                                          \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess) {                                                          \
            cudaGetLastError();                                                           \
            return fail(e_ == cudaErrorMemoryAllocation ? O3G_ERR_OUT_OF_MEMORY : O3G_ERR_CUDA, \
                        std::string(#call) + ": " + cudaGetErrorString(e_));              \
        }                                                                                 \
    } while (0)

#define TRY(expr)                          \
    do {                                   \
        o3g_status s_ = (expr);            \
        if (s_ != O3G_OK) return s_;       \
    } while (0)

// --------------------------------------------------------- device buffers
// NVTX phase ranges: one range per API phase on the calling thread
struct PhaseRange {
#ifndef O3G_NO_NVTX
    explicit PhaseRange(const char* name) { nvtxRangePushA(name); }
    ~PhaseRange() { nvtxRangePop(); }
#else
    explicit PhaseRange(const char*) {}
#endif
    PhaseRange(const PhaseRange&) = delete;
    PhaseRange& operator=(const PhaseRange&) = delete;
};

struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    o3g_status ensure(size_t bytes, bool* grew = nullptr) {
        if (bytes <= cap && p) return O3G_OK;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        size_t b = bytes < 256 ? 256 : bytes;
        cudaError_t e = cudaMalloc(&p, b);
        if (e != cudaSuccess) {
            cudaGetLastError();
            return fail(O3G_ERR_OUT_OF_MEMORY, std::string("cudaMalloc: ") + cudaGetErrorString(e));
        }
        cap = b;
        if (grew) *grew = true;
        return O3G_OK;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
    template <class T>
    T* as() const { return (T*)p; }
};

// ------------------------------------------------------------------ NCCL
namespace {
typedef int nccl_result_t;
typedef void* nccl_comm_t;
struct nccl_uid { char internal[128]; };
struct NcclApi {
    bool loaded = false;
    nccl_result_t (*get_unique_id)(nccl_uid*) = nullptr;
    nccl_result_t (*comm_init_rank)(nccl_comm_t*, int, nccl_uid, int) = nullptr;
    nccl_result_t (*all_gather)(const void*, void*, size_t, int, nccl_comm_t, cudaStream_t) = nullptr;
    nccl_result_t (*comm_destroy)(nccl_comm_t) = nullptr;
    const char* (*error_string)(nccl_result_t) = nullptr;
};
constexpr int kNcclFloat64 = 8;

NcclApi& nccl() {
    static NcclApi api;
    if (!api.loaded) {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (h) {
            api.get_unique_id = (decltype(api.get_unique_id))dlsym(h, "ncclGetUniqueId");
            api.comm_init_rank = (decltype(api.comm_init_rank))dlsym(h, "ncclCommInitRank");
            api.all_gather = (decltype(api.all_gather))dlsym(h, "ncclAllGather");
            api.comm_destroy = (decltype(api.comm_destroy))dlsym(h, "ncclCommDestroy");
            api.error_string = (decltype(api.error_string))dlsym(h, "ncclGetErrorString");
            api.loaded = api.get_unique_id && api.comm_init_rank && api.all_gather && api.comm_destroy;
        }
    }
    return api;
}
}  // namespace

// ------------------------------------------------------------------ ctx
struct GraphKey {
    int max_it = -1, search = -1, timing = -1, world = -1, blocks = -1;
    int64_t n_local = -1;
    const void* ptrs[12] = {};
    bool operator==(const GraphKey& o) const {
        return max_it == o.max_it && search == o.search && timing == o.timing && world == o.world &&
               blocks == o.blocks && n_local == o.n_local && !memcmp(ptrs, o.ptrs, sizeof(ptrs));
    }
};

struct o3g_ctx {
    int device = 0;
    int sms = 148;
    cudaStream_t user = nullptr;   // caller's stream (may be the legacy default)
    cudaStream_t exec = nullptr;   // internal capture/execution stream
    cudaEvent_t fence = nullptr;
    // one-shot host inputs: H2D copies on their own stream, overlapped with
    // the grid build (created on first use)
    cudaStream_t copy = nullptr;
    cudaEvent_t ev_copy[4] = {};

    // options
    int search = 1, grid_mode = 0, timing = 0, bps_override = 0, nbr_mask = 1, coop_min = -1;
    int estimation = 0;   // 0 point-to-plane, 1 point-to-point
    int src_order = 0;    // 0 lexicographic cell, 1 brick-Morton
    int target_sort = 1;  // 0 counting sort, 1 stable radix sort (default: measured faster)
    int prune_min = -1;   // variant 1 row pruning: -1 auto, -2 never, >= 0 threshold
    int interleave = -1;  // variant 1 batch interleave: -1 auto, 0 off, 1 on
    int xsort = -1;       // target x-order inside cells: -1 auto, 0 off, 1 on
    double shard_live_weight = 8.0;   // multi-rank split: work of a live query / a dead one
    bool shard_zslab = false;         // multi-rank split by z-major key ranges instead of x-slabs
    int cert_sweep = 0;   // certificate passes: 0 fused into the search kernel, 1 separate sweep kernel
    int cert_opt = -1;    // correspondence certificates in the run loop: -1 auto, 0 off, 1 on (§5.5)
    int trace_pass = -1;  // o3g_icp_run: record the correspondences of this pass
    // certificate goal: searches stage rows up to the previous
    // winner's distance + 2 min(mul x last displacement bound, cap x h);
    // O3G_CERT_GOAL="mul,cap" overrides (experiments only)
    double rhog_mul = 4.0, rhog_cap = 1.0;
    bool xsorted = false;
    bool has_normals = false;

    // target grid
    int64_t m = 0;
    double dmax = 0.0;
    GridDev g{};
    int64_t occupied = 0;
    DevBuf tpos, tnrm, cell_start, counts, nbr_a, nbr_b, nbr_c;   // nbr_c: radius-2 bitmap (dense)
    bool nbr_ready = false;
    int cshift = 0, cnx = 0, cny = 0;   // hashed grid: coarse occupancy bitmap (nbr_a)
    // scratch
    DevBuf keys_a, keys_b, vals_a, vals_b, cub_tmp, stage_a, stage_b, stage_c, misc, misc2;
    // voxel_down_sample / multi-scale scratch
    DevBuf vk_a, vk_b, vflags, vrunid, vstarts, ms_src, ms_tgt, ms_nrm;
    DevBuf ms_in_src, ms_in_tgt, ms_in_nrm;   // multi-scale: host inputs copied once
    DevBuf ev_T, ev_part, ev_out;
    // source
    int64_t n_total = 0, n_local = 0, shard_lo = 0;
    bool src_ready = false;
    DevBuf src4;
    DevBuf prevj;          // run loop: previous pass's winner per local query
    DevBuf cert;           // run loop: per local query certificate (2 x float4, §5.5)
    int32_t cert_epoch = 0;        // the next run's gbase (pass tag base of certificates)
    bool cert_fresh = true;        // the records need a reset (new buffer / tag wrap-around)
    DevBuf need;           // run loop: per local query search flag (sweep -> search)
    DevBuf hist_T, hist_terms, trace_corr;   // run loop: per-pass T / terms, traced corr
    float smax[3] = {0.f, 0.f, 0.f};         // max |source coordinate| per axis
    int32_t last_passes = 0;
    bool trace_valid = false;
    DevBuf tiles, tflag;  // variant 4 tile starts (local shard) and scratch
    DevBuf xk_a, xk_b, xpos, xnrm;   // x-order inside cells (scratch)
    int32_t ntiles = 0;
    // loop
    DevBuf partials, gathered, state, hist_fit, hist_rmse;
    IcpState* h_state = nullptr;   // pinned
    // graph
    cudaGraphExec_t gexec = nullptr;
    GraphKey gkey;
    std::vector<cudaEvent_t> events;
    int graph_launches = 0;        // our kernels per graph launch
    // distributed
    int rank = 0, world = 1;
    bool loopback = false;         // o3g_dist_init_loopback: no communicator (o3g_loopback_run)
    nccl_comm_t comm = nullptr;
    // o3g_set_clouds: the source's keys / sort / gather run on a side stream beside the
    // target build, on their own scratch
    cudaStream_t side = nullptr;
    cudaEvent_t ev_side = nullptr;
    DevBuf s_keys_a, s_keys_b, s_vals_a, s_vals_b, s_cub;
    int64_t pend_src_n = 0, pend_src_lo = 0, pend_src_hi = 0;   // set_source results awaiting source_finish
    // peer-memory exchange (o3g_dist_peer_*): this rank's Xchg, the device array of
    // every rank's Xchg pointer, and the peers' buffers opened through CUDA IPC
    DevBuf xchg, xpeers;
    std::vector<void*> ipc_opened;
    bool peer_xchg = false;
    uint32_t xepoch = 0;           // the next run's IcpState::xbase
    // stats
    int64_t launches = 0;
    double last_k3_ms = 0.0, last_tail_ms = 0.0;
    int32_t last_k3_launches = 0;
};

// ------------------------------------------------------------- helpers
static bool is_device_ptr(const void* p) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

// device memory of ANOTHER device (the kernels would dereference it without
// peer access: a sticky fault): rejected as an invalid argument
static bool foreign_device_ptr(const void* p, int device) {
    cudaPointerAttributes at;
    if (!p || cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeDevice && at.device != device;
}

// the largest float <= v (v > 0)
static float round_down_f(double v) {
    float f = (float)v;
    if ((double)f > v) f = nextafterf(f, 0.0f);
    return f;
}

static bool rigid_ok(const double* T) {
    if (!T) return false;
    for (int i = 0; i < 16; ++i)
        if (!isfinite(T[i])) return false;
    if (T[12] != 0.0 || T[13] != 0.0 || T[14] != 0.0 || T[15] != 1.0) return false;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double s = 0.0;
            for (int k = 0; k < 3; ++k) s += T[4 * k + i] * T[4 * k + j];
            if (fabs(s - (i == j ? 1.0 : 0.0)) > 1e-9) return false;
        }
    const double det = T[0] * (T[5] * T[10] - T[6] * T[9]) - T[1] * (T[4] * T[10] - T[6] * T[8]) +
                       T[2] * (T[4] * T[9] - T[5] * T[8]);
    return fabs(det - 1.0) <= 1e-9;
}

static float ord2f(uint32_t u) {
    uint32_t b = (u & 0x80000000u) ? (u & 0x7fffffffu) : ~u;
    float f;
    memcpy(&f, &b, 4);
    return f;
}

// Fence: work on ctx->exec starts after everything already on the user stream.
static o3g_status enter(o3g_ctx* c) {
    CK(cudaSetDevice(c->device));
    CK(cudaEventRecord(c->fence, c->user));
    CK(cudaStreamWaitEvent(c->exec, c->fence, 0));
    return O3G_OK;
}

// Device view of an input array: the caller's pointer if it is device
// memory, else a copy into a context staging buffer (the e2e path).
static o3g_status device_view(o3g_ctx* c, const float* p, int64_t count, DevBuf& stage,
                              const float** out) {
    if (foreign_device_ptr(p, c->device))
        return fail(O3G_ERR_INVALID_ARGUMENT, "array is device memory of another device than the context's");
    if (is_device_ptr(p)) {
        *out = p;
        return O3G_OK;
    }
    TRY(stage.ensure((size_t)count * sizeof(float)));
    CK(cudaMemcpyAsync(stage.p, p, (size_t)count * sizeof(float), cudaMemcpyHostToDevice, c->exec));
    *out = stage.as<float>();
    return O3G_OK;
}

static int bits_for(uint64_t maxval) {
    int b = 1;
    while (b < 32 && (maxval >> b)) ++b;
    return b;
}

static o3g_status sort_pairs(o3g_ctx* c, int64_t n, int end_bit, int begin_bit = 0) {
    size_t tmp = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, c->keys_a.as<uint32_t>(), c->keys_b.as<uint32_t>(),
                                       c->vals_a.as<int32_t>(), c->vals_b.as<int32_t>(), (int)n, begin_bit,
                                       end_bit, c->exec));
    TRY(c->cub_tmp.ensure(tmp));
    CK(cub::DeviceRadixSort::SortPairs(c->cub_tmp.p, tmp, c->keys_a.as<uint32_t>(), c->keys_b.as<uint32_t>(),
                                       c->vals_a.as<int32_t>(), c->vals_b.as<int32_t>(), (int)n, begin_bit,
                                       end_bit, c->exec));
    return O3G_OK;
}

static void invalidate_graph(o3g_ctx* c) {
    if (c->gexec) cudaGraphExecDestroy(c->gexec);
    c->gexec = nullptr;
    c->gkey = GraphKey{};
}

// ------------------------------------------------------------- C ABI
extern "C" {

const char* o3g_status_string(o3g_status s) {
    switch (s) {
        case O3G_OK: return "ok";
        case O3G_ERR_INVALID_ARGUMENT: return "invalid argument";
        case O3G_ERR_DEGENERATE: return "degenerate input";
        case O3G_ERR_CUDA: return "cuda error";
        case O3G_ERR_OUT_OF_MEMORY: return "out of memory";
        case O3G_ERR_COMM: return "communication error";
        case O3G_ERR_NOT_IMPLEMENTED: return "not implemented";
    }
    return "unknown status";
}

const char* o3g_last_error(void) { return g_err.c_str(); }

o3g_status o3g_create(o3g_ctx** out, int device, void* cuda_stream) {
    if (!out) return fail(O3G_ERR_INVALID_ARGUMENT, "out is NULL");
    *out = nullptr;
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return fail(O3G_ERR_INVALID_ARGUMENT, "bad device index");
    CK(cudaSetDevice(device));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) return fail(O3G_ERR_CUDA, "o3g is built for sm_100a (B200) only");
    o3g_ctx* c = new o3g_ctx();
    c->device = device;
    c->sms = prop.multiProcessorCount;
    if (const char* sw = getenv("O3G_SHARD_LIVE_WEIGHT")) c->shard_live_weight = atof(sw);
    if (const char* sz = getenv("O3G_SHARD_SLAB")) c->shard_zslab = sz[0] == 'z';
    if (const char* gs = getenv("O3G_CERT_GOAL")) sscanf(gs, "%lf,%lf", &c->rhog_mul, &c->rhog_cap);
    c->user = (cudaStream_t)cuda_stream;
    cudaError_t e = cudaStreamCreate(&c->exec);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->fence, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaMallocHost(&c->h_state, sizeof(IcpState));
    if (e != cudaSuccess) {
        cudaGetLastError();
        o3g_destroy(c);
        return fail(O3G_ERR_CUDA, std::string("context setup: ") + cudaGetErrorString(e));
    }
    *out = c;
    return O3G_OK;
}

// drop the peer-memory exchange (IPC mappings and the pointer table; the
// context's own Xchg buffer stays allocated so an exported handle stays valid)
static void peer_disconnect(o3g_ctx* c) {
    for (void* p : c->ipc_opened) cudaIpcCloseMemHandle(p);
    c->ipc_opened.clear();
    c->xpeers.release();
    c->peer_xchg = false;
}

o3g_status o3g_destroy(o3g_ctx* c) {
    if (!c) return O3G_OK;
    cudaSetDevice(c->device);
    if (c->exec) cudaStreamSynchronize(c->exec);
    invalidate_graph(c);
    for (auto ev : c->events) cudaEventDestroy(ev);
    DevBuf* bufs[] = {&c->tpos, &c->tnrm, &c->cell_start, &c->counts, &c->nbr_a, &c->nbr_b, &c->keys_a, &c->keys_b,
                      &c->vals_a, &c->vals_b, &c->cub_tmp, &c->stage_a, &c->stage_b, &c->stage_c, &c->misc, &c->misc2,
                      &c->src4, &c->partials, &c->gathered, &c->state, &c->hist_fit, &c->hist_rmse,
                      &c->vk_a, &c->vk_b, &c->vflags, &c->vrunid, &c->vstarts, &c->ms_src,
                      &c->ms_tgt, &c->ms_nrm, &c->ev_T, &c->ev_part, &c->ev_out, &c->tiles, &c->tflag, &c->prevj, &c->ms_in_src, &c->ms_in_tgt, &c->ms_in_nrm, &c->xk_a, &c->xk_b, &c->xpos, &c->xnrm, &c->cert, &c->hist_T, &c->hist_terms, &c->trace_corr, &c->nbr_c, &c->need};
    for (DevBuf* b : bufs) b->release();
    if (c->comm && nccl().comm_destroy) nccl().comm_destroy(c->comm);
    peer_disconnect(c);
    c->xchg.release();
    for (DevBuf* b : {&c->s_keys_a, &c->s_keys_b, &c->s_vals_a, &c->s_vals_b, &c->s_cub}) b->release();
    if (c->ev_side) cudaEventDestroy(c->ev_side);
    if (c->side) cudaStreamDestroy(c->side);
    if (c->h_state) cudaFreeHost(c->h_state);
    if (c->fence) cudaEventDestroy(c->fence);
    for (cudaEvent_t e : c->ev_copy)
        if (e) cudaEventDestroy(e);
    if (c->copy) cudaStreamDestroy(c->copy);
    if (c->exec) cudaStreamDestroy(c->exec);
    delete c;
    return O3G_OK;
}

o3g_status o3g_set_option(o3g_ctx* c, int option, int64_t value) {
    if (!c) return fail(O3G_ERR_INVALID_ARGUMENT, "ctx is NULL");
    switch (option) {
        case O3G_OPT_SEARCH:
            if (value < 0 || value > 4) return fail(O3G_ERR_INVALID_ARGUMENT, "search must be in [0, 4]");
            c->search = (int)value;
            break;
        case O3G_OPT_GRID:
            if (value < 0 || value > 2) return fail(O3G_ERR_INVALID_ARGUMENT, "grid must be 0, 1 or 2");
            c->grid_mode = (int)value;
            break;
        case O3G_OPT_TIMING: c->timing = value ? 1 : 0; break;
        case O3G_OPT_NBR_MASK: c->nbr_mask = value ? 1 : 0; break;
        case O3G_OPT_SOURCE_ORDER:
            if (value < 0 || value > 1) return fail(O3G_ERR_INVALID_ARGUMENT, "source order must be 0 or 1");
            c->src_order = (int)value;
            break;
        case O3G_OPT_TARGET_SORT:
            if (value < 0 || value > 1) return fail(O3G_ERR_INVALID_ARGUMENT, "target sort must be 0 or 1");
            c->target_sort = (int)value;
            break;
        case O3G_OPT_XSORT:
            if (value < -1 || value > 1) return fail(O3G_ERR_INVALID_ARGUMENT, "xsort must be -1, 0 or 1");
            c->xsort = (int)value;
            break;
        case O3G_OPT_INTERLEAVE:
            if (value < -1 || value > 1) return fail(O3G_ERR_INVALID_ARGUMENT, "interleave must be -1, 0 or 1");
            c->interleave = (int)value;
            break;
        case O3G_OPT_PRUNE_MIN:
            if (value < -2 || value > (1 << 30)) return fail(O3G_ERR_INVALID_ARGUMENT, "prune_min out of range");
            c->prune_min = (int)value;
            break;
        case O3G_OPT_ESTIMATION:
            if (value < 0 || value > 1) return fail(O3G_ERR_INVALID_ARGUMENT, "estimation must be 0 or 1");
            c->estimation = (int)value;
            break;
        case O3G_OPT_COOP_MIN:
            if (value < -1 || value > (1 << 30)) return fail(O3G_ERR_INVALID_ARGUMENT, "coop_min out of range");
            c->coop_min = (int)value;
            break;
        case O3G_OPT_CERT:
            if (value < -1 || value > 2) return fail(O3G_ERR_INVALID_ARGUMENT, "cert must be -1, 0, 1 or 2");
            c->cert_opt = (int)value;
            break;
        case O3G_OPT_CERT_SWEEP:
            if (value < 0 || value > 1) return fail(O3G_ERR_INVALID_ARGUMENT, "cert sweep must be 0 or 1");
            c->cert_sweep = (int)value;
            break;
        case O3G_OPT_TRACE_PASS:
            if (value < -1 || value > 100000) return fail(O3G_ERR_INVALID_ARGUMENT, "trace pass must be in [-1, 100000]");
            c->trace_pass = (int)value;
            break;
        case O3G_OPT_BLOCKS_PER_SM:
            if (value < 0 || value > 64) return fail(O3G_ERR_INVALID_ARGUMENT, "blocks per SM out of range");
            c->bps_override = (int)value;
            break;
        default: return fail(O3G_ERR_INVALID_ARGUMENT, "unknown option");
    }
    invalidate_graph(c);
    return O3G_OK;
}

// normals_ready (nullable): the normals arrive later on another stream; the
// gather waits for it and their finiteness is checked at the final sync
static o3g_status target_finish(o3g_ctx* c, bool normals_late);

// defer_final: return once everything is enqueued (the grid parameters are known and
// stored); the caller runs target_finish after its own work (o3g_set_clouds)
static o3g_status set_target_impl(o3g_ctx* c, const float* xyz, const float* normals, int64_t n,
                                  double dmax, cudaEvent_t normals_ready, bool defer_final = false) {
    PhaseRange nvtx_("o3g:set_target (A0-A1 grid build)");
    if (!c) return fail(O3G_ERR_INVALID_ARGUMENT, "ctx is NULL");
    if (!xyz) return fail(O3G_ERR_INVALID_ARGUMENT, "target xyz is required");
    if (n <= 0 || n > 0x7ffffffeLL) return fail(O3G_ERR_INVALID_ARGUMENT, "n_target must be in [1, 2^31-2]");
    if (!(dmax > 0.0) || !isfinite(dmax)) return fail(O3G_ERR_INVALID_ARGUMENT, "max_correspondence_distance must be finite and > 0");
    TRY(enter(c));
    c->src_ready = false;
    c->m = 0;
    invalidate_graph(c);
    const float *dx, *dn;
    TRY(device_view(c, xyz, 3 * n, c->stage_a, &dx));
    dn = nullptr;
    if (normals) TRY(device_view(c, normals, 3 * n, c->stage_b, &dn));

    // A0/A1: bbox + finiteness (one sync: the grid dims size the table)
    TRY(c->misc.ensure(64));
    uint32_t* mm = c->misc.as<uint32_t>();
    int32_t* bad = (int32_t*)(mm + 6);
    unsigned long long* occ = (unsigned long long*)(mm + 8);
    CK(cudaMemsetAsync(mm, 0xFF, 12, c->exec));
    CK(cudaMemsetAsync(mm + 3, 0x00, 12 + 4 + 4 + 8, c->exec));
    CK(cudaMemsetAsync(mm + 12, 0x00, 4, c->exec));   // fused-tail block counter
    launch_bbox(dx, n, mm, bad, c->sms, c->exec);
    if (dn && !normals_ready) launch_check_finite(dn, 3 * n, bad, c->sms, c->exec);
    c->launches += dn && !normals_ready ? 2 : 1;
    uint32_t h[8];
    CK(cudaMemcpyAsync(h, mm, 32, cudaMemcpyDeviceToHost, c->exec));
    CK(cudaStreamSynchronize(c->exec));
    if (h[6]) return fail(O3G_ERR_INVALID_ARGUMENT, "non-finite target coordinate or normal");

    GridDev g{};
    const double hcell = dmax * (1.0 + 9.5367431640625e-07);  // dmax (1 + 2^-20), R12
    g.inv_h = 1.0 / hcell;
    g.h = hcell;
    double o[3];
    int64_t dims[3];
    for (int a = 0; a < 3; ++a) {
        o[a] = (double)ord2f(h[a]);
        double hi = (double)ord2f(h[3 + a]);
        double cmax = floor((hi - o[a]) * g.inv_h);
        if (!(cmax < 1073741824.0)) return fail(O3G_ERR_INVALID_ARGUMENT, "target extent / dmax exceeds 2^30 cells per axis");
        dims[a] = (int64_t)cmax + 1;
    }
    g.ox = o[0], g.oy = o[1], g.oz = o[2];
    g.nx = (int32_t)dims[0], g.ny = (int32_t)dims[1], g.nz = (int32_t)dims[2];
    const double ncells = (double)dims[0] * (double)dims[1] * (double)dims[2];
    const double dense_cap = fmax(64.0 * (double)n, 16777216.0);
    bool hashed = c->grid_mode == 2 || (c->grid_mode == 0 && ncells > dense_cap) || ncells > 2147483000.0;
    if (hashed) {
        uint64_t t = 1024;
        while (t < 2ull * (uint64_t)n) t <<= 1;
        g.hashed = 1;
        g.hmask = (uint32_t)(t - 1);
        g.table_size = (int64_t)t;
    } else {
        g.hashed = 0;
        g.hmask = 0;
        g.table_size = (int64_t)ncells;
    }

    TRY(c->keys_a.ensure(n * 4));
    TRY(c->keys_b.ensure(n * 4));
    TRY(c->vals_a.ensure(n * 4));
    TRY(c->vals_b.ensure(n * 4));
    TRY(c->cell_start.ensure((g.table_size + 1) * 4));
    if (c->target_sort != 1) TRY(c->counts.ensure((g.table_size + 1) * 4));   // (counting sort only)
    TRY(c->tpos.ensure((n + 2) * sizeof(float4)));   // +pad: pair loads may touch tpos[n]
    TRY(c->tnrm.ensure(n * sizeof(float4)));

    launch_cell_keys(dx, n, g, nullptr, c->keys_a.as<uint32_t>(), c->vals_a.as<int32_t>(), c->exec);
    const bool radix = c->target_sort == 1;
    bool occ_built = false;
    if (radix) {
        TRY(sort_pairs(c, n, bits_for((uint64_t)(g.table_size - 1))));
        // cell starts straight from the sorted keys (one pass, no histogram,
        // memset or scan); dense grids get their occupancy bits here
        uint32_t* obits = nullptr;
        if (!g.hashed) {
            const int64_t nw = (g.table_size + 31) / 32;
            TRY(c->nbr_a.ensure(nw * 4));
            TRY(c->nbr_b.ensure(nw * 4));
            CK(cudaMemsetAsync(c->nbr_a.p, 0, nw * 4, c->exec));
            obits = c->nbr_a.as<uint32_t>();
            occ_built = true;
        }
        launch_cs_fill(c->keys_b.as<uint32_t>(), n, g.table_size, c->cell_start.as<int32_t>(), obits, c->exec);
    } else {
        CK(cudaMemsetAsync(c->counts.p, 0, (g.table_size + 1) * 4, c->exec));
        launch_histogram(c->keys_a.as<uint32_t>(), n, c->counts.as<int32_t>(), occ, c->exec);
        size_t tmp = 0;
        CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, c->counts.as<int32_t>(), c->cell_start.as<int32_t>(),
                                         (int)(g.table_size + 1), c->exec));
        TRY(c->cub_tmp.ensure(tmp));
        CK(cub::DeviceScan::ExclusiveSum(c->cub_tmp.p, tmp, c->counts.as<int32_t>(), c->cell_start.as<int32_t>(),
                                         (int)(g.table_size + 1), c->exec));
    }
    if (normals_ready) {
        CK(cudaStreamWaitEvent(c->exec, normals_ready, 0));
        if (dn) {
            launch_check_finite(dn, 3 * n, bad, c->sms, c->exec);
            c->launches += 1;
        }
    }
    if (radix) {   // stable (key, index) radix sort: cells in original-index order
        launch_gather_target(dx, dn, c->vals_b.as<int32_t>(), c->keys_b.as<uint32_t>(), n,
                             c->tpos.as<float4>(), c->tnrm.as<float4>(), occ, c->exec);
    } else {       // counting sort: one pass, coalesced reads, scattered writes
        CK(cudaMemcpyAsync(c->counts.p, c->cell_start.p, (g.table_size + 1) * 4, cudaMemcpyDeviceToDevice,
                           c->exec));
        launch_scatter_target(dx, dn, c->keys_a.as<uint32_t>(), n, c->counts.as<int32_t>(),
                              c->tpos.as<float4>(), c->tnrm.as<float4>(), c->exec);
    }
    c->launches += 3;
    c->nbr_ready = false;
    if (!g.hashed) {
        const int64_t nw = (g.table_size + 31) / 32;
        TRY(c->nbr_a.ensure(nw * 4));
        TRY(c->nbr_b.ensure(nw * 4));
        if (occ_built) {   // occupancy bits already set from the sorted keys: dilate only
            launch_dilate3(c->nbr_a.as<uint32_t>(), c->nbr_b.as<uint32_t>(), g.table_size, g.nx,
                           (int64_t)g.nx * g.ny, c->exec);
        } else {
            launch_nbr_bits(c->cell_start.as<int32_t>(), g.table_size, g.nx, (int64_t)g.nx * g.ny,
                            c->nbr_b.as<uint32_t>(), c->nbr_a.as<uint32_t>(), c->exec);
        }
        // dilated once more: empty 5^3 neighbourhoods (the certificates of dead queries)
        TRY(c->nbr_c.ensure(nw * 4));
        CK(cudaMemcpyAsync(c->nbr_c.p, c->nbr_a.p, nw * 4, cudaMemcpyDeviceToDevice, c->exec));
        launch_dilate3(c->nbr_c.as<uint32_t>(), c->nbr_b.as<uint32_t>(), g.table_size, g.nx,
                       (int64_t)g.nx * g.ny, c->exec);
        c->launches += 7;
        c->nbr_ready = true;
    } else {
        // hashed grid: coarse occupancy bitmap (<= 2^30 bits) for the live test
        int sh = 0;
        while ((double)(((int64_t)g.nx + (1 << sh) - 1) >> sh) * (double)(((int64_t)g.ny + (1 << sh) - 1) >> sh) *
                   (double)(((int64_t)g.nz + (1 << sh) - 1) >> sh) > 1073741824.0)
            ++sh;
        c->cshift = sh;
        c->cnx = (int)(((int64_t)g.nx + (1 << sh) - 1) >> sh);
        c->cny = (int)(((int64_t)g.ny + (1 << sh) - 1) >> sh);
        const int64_t cnz = ((int64_t)g.nz + (1 << sh) - 1) >> sh;
        const int64_t ncc = (int64_t)c->cnx * c->cny * cnz, nw = (ncc + 31) / 32;
        TRY(c->nbr_a.ensure(nw * 4));
        TRY(c->nbr_b.ensure(nw * 4));
        CK(cudaMemsetAsync(c->nbr_a.p, 0, nw * 4, c->exec));
        launch_coarse_bits(c->tpos.as<float4>(), n, g, sh, c->cnx, c->cny, c->nbr_a.as<uint32_t>(), c->exec);
        launch_dilate3(c->nbr_a.as<uint32_t>(), c->nbr_b.as<uint32_t>(), ncc, c->cnx, (int64_t)c->cnx * c->cny,
                       c->exec);
        c->launches += 4;
        c->nbr_ready = true;
    }
    c->g = g;
    c->m = n;
    c->dmax = dmax;
    c->has_normals = dn != nullptr;
    c->xsorted = false;
    if (defer_final) return O3G_OK;
    return target_finish(c, normals_ready != nullptr);
}

// the end of o3g_set_target: wait for the build, read the occupied-cell count (and the
// late normals' finiteness flag), then the x-order inside cells for dense targets
static o3g_status target_finish(o3g_ctx* c, bool normals_late) {
    PhaseRange nvtx_("o3g:set_target finish");
    const GridDev g = c->g;
    const int64_t n = c->m;
    uint32_t* mm = c->misc.as<uint32_t>();
    int32_t* bad = (int32_t*)(mm + 6);
    unsigned long long* occ = (unsigned long long*)(mm + 8);
    unsigned long long h_occ = 0;
    int32_t h_bad2 = 0;
    c->m = 0;   // (until the build is known to be good)
    CK(cudaMemcpyAsync(&h_occ, occ, 8, cudaMemcpyDeviceToHost, c->exec));
    if (normals_late) CK(cudaMemcpyAsync(&h_bad2, bad, 4, cudaMemcpyDeviceToHost, c->exec));
    CK(cudaStreamSynchronize(c->exec));
    CK(cudaGetLastError());
    if (h_bad2) return fail(O3G_ERR_INVALID_ARGUMENT, "non-finite target coordinate or normal");
    c->m = n;
    c->occupied = (int64_t)h_occ;
    // x-order inside cells for dense targets (the cooperative path's x-windows):
    // auto when the target averages >= 32 points per occupied cell
    c->xsorted = false;
    const bool xs = !g.hashed && (c->xsort == 1 || (c->xsort == -1 && (double)n >= 32.0 * (double)(h_occ ? h_occ : 1)));
    if (xs) {
        TRY(c->xk_a.ensure((size_t)n * 8));
        TRY(c->xk_b.ensure((size_t)n * 8));
        TRY(c->xpos.ensure((size_t)n * sizeof(float4)));
        TRY(c->xnrm.ensure((size_t)n * sizeof(float4)));
        launch_xkeys(c->tpos.as<float4>(), n, g, (uint64_t*)c->xk_a.p, c->vals_a.as<int32_t>(), c->exec);
        const int eb = 32 + bits_for((uint64_t)(g.table_size - 1));
        size_t tmp = 0;
        CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, (uint64_t*)c->xk_a.p, (uint64_t*)c->xk_b.p,
                                           c->vals_a.as<int32_t>(), c->vals_b.as<int32_t>(), (int)n, 0, eb,
                                           c->exec));
        TRY(c->cub_tmp.ensure(tmp));
        CK(cub::DeviceRadixSort::SortPairs(c->cub_tmp.p, tmp, (uint64_t*)c->xk_a.p, (uint64_t*)c->xk_b.p,
                                           c->vals_a.as<int32_t>(), c->vals_b.as<int32_t>(), (int)n, 0, eb,
                                           c->exec));
        launch_permute_target(c->tpos.as<float4>(), c->tnrm.as<float4>(), c->vals_b.as<int32_t>(), n,
                              c->xpos.as<float4>(), c->xnrm.as<float4>(), c->exec);
        std::swap(c->tpos, c->xpos);
        std::swap(c->tnrm, c->xnrm);
        c->launches += 4;
        CK(cudaStreamSynchronize(c->exec));
        CK(cudaGetLastError());
        c->xsorted = true;
    }
    return O3G_OK;
}

o3g_status o3g_set_target(o3g_ctx* c, const float* xyz, const float* normals, int64_t n,
                          double dmax) {
    return set_target_impl(c, xyz, normals, n, dmax, nullptr);
}

static o3g_status source_finish(o3g_ctx* c);

// defer: enqueue only, on c->exec as the caller set it (no wait for the user stream, no
// final sync); the caller runs source_finish afterwards (o3g_set_clouds)
static o3g_status set_source_impl(o3g_ctx* c, const float* xyz, int64_t n, const double order_T[16], bool defer) {
    PhaseRange nvtx_("o3g:set_source (A2 ordering)");
    if (!c) return fail(O3G_ERR_INVALID_ARGUMENT, "ctx is NULL");
    if (!xyz) return fail(O3G_ERR_INVALID_ARGUMENT, "source xyz is required");
    // (the kernels' 32-bit batch cursors step by up to 2^24 past the last query)
    if (n <= 0 || n > 0x7effffffLL) return fail(O3G_ERR_INVALID_ARGUMENT, "n_source must be in [1, 2^31 - 2^24]");
    if (c->m <= 0) return fail(O3G_ERR_INVALID_ARGUMENT, "o3g_set_target must be called first");
    if (order_T && !rigid_ok(order_T)) return fail(O3G_ERR_INVALID_ARGUMENT, "order_T is not a rigid transform");
    if (!defer) TRY(enter(c));
    c->src_ready = false;
    invalidate_graph(c);
    const float* dx;
    TRY(device_view(c, xyz, 3 * n, c->stage_a, &dx));
    TRY(c->misc.ensure(128));
    int32_t* bad = (int32_t*)(c->misc.as<uint32_t>() + 6);
    uint32_t* smm = c->misc.as<uint32_t>() + 24;   // source bbox (ordered uint32 min[3], max[3])
    CK(cudaMemsetAsync(bad, 0, 4, c->exec));
    CK(cudaMemsetAsync(smm, 0xFF, 12, c->exec));
    CK(cudaMemsetAsync(smm + 3, 0x00, 12, c->exec));
    // bbox + finiteness; the bbox bounds |s| for the certificates' displacement
    // test (the flag is read at the final sync: a non-finite point only yields
    // a clamped ordering key meanwhile, and the call then fails)
    launch_bbox(dx, n, smm, bad, c->sms, c->exec);

    TRY(c->keys_a.ensure(n * 4));
    TRY(c->keys_b.ensure(n * 4));
    TRY(c->vals_a.ensure(n * 4));
    TRY(c->vals_b.ensure(n * 4));
    double T12[12];
    if (order_T) memcpy(T12, order_T, sizeof(T12));
    // order: 8^3-cell brick Morton for the staged-tile kernel (variant 4),
    // 4^3 bricks for O3G_OPT_SOURCE_ORDER = 1, else by cell; brick keys must
    // fit 32 bits (3 * bits(dim >> b) + 3 b)
    int brick = c->g.hashed ? 0 : c->search == 4 ? 3 : c->src_order == 1 ? 2 : 0;
    if (brick) {
        const int dmaxc = std::max(c->g.nx, std::max(c->g.ny, c->g.nz));
        if (3 * bits_for((uint64_t)(dmaxc >> brick)) + 3 * brick > 32) brick = 0;
    }
    launch_cell_keys(dx, n, c->g, order_T ? T12 : nullptr, c->keys_a.as<uint32_t>(),
                     c->vals_a.as<int32_t>(), c->exec, brick);
    const int kbits = brick ? 32 : bits_for((uint64_t)(c->g.table_size - 1));
    const int sbits = 0;   // (a 24-bit order of 8-cell x-runs: one sort pass fewer, K3 0.7 % slower, step no faster)
    int64_t lo = (int64_t)c->rank * n / c->world, hi = (int64_t)(c->rank + 1) * n / c->world;
    int64_t base = 0;   // sorted position of the first sorted (selected) key
    if (c->world > 1 && !brick && c->search != 4) {
        // this rank's shard without sorting all n: a histogram
        // of the top 12 key bits with, per bucket, the queries whose stencil
        // holds a target at order_T (they run the full search); the ranks
        // split the bucket sequence into contiguous ranges of equal estimated
        // work (live 8, dead 1: equal counts left the densest slab's rank with
        // 1.8x the mean work at 8 ranks), then select (stably) and sort only
        // their own buckets. Every rank derives the same split.
        const int shift = kbits > 12 ? kbits - 12 : 0;
        // dense grid: x-slabs (O3G_SHARD_SLAB=z: z-major key ranges)
        const int xdiv = c->g.hashed || c->shard_zslab ? 0 : c->g.nx;
        TRY(c->misc2.ensure(2 * kShardBuckets * sizeof(uint32_t)));
        const uint32_t* live = (!c->g.hashed && c->nbr_ready) ? c->nbr_a.as<uint32_t>() : nullptr;
        launch_key_hist(c->keys_a.as<uint32_t>(), n, shift, xdiv, live, c->misc2.as<uint32_t>(), c->sms, c->exec);
        std::vector<uint32_t> hist(2 * kShardBuckets);
        CK(cudaMemcpyAsync(hist.data(), c->misc2.p, hist.size() * sizeof(uint32_t), cudaMemcpyDeviceToHost, c->exec));
        CK(cudaStreamSynchronize(c->exec));
        const double wl = c->shard_live_weight - 1.0;
        double wtot = 0.0;
        for (int b = 0; b < kShardBuckets; ++b) wtot += (double)hist[b] + wl * (double)hist[kShardBuckets + b];
        // rank r owns buckets [B_r, B_(r+1)): B_r = first bucket whose preceding
        // weight reaches r/world of the total
        auto first_bucket = [&](int r) {
            if (r <= 0) return 0;
            if (r >= c->world) return kShardBuckets;
            const double goal = wtot * (double)r / (double)c->world;
            double cw = 0.0;
            for (int b = 0; b < kShardBuckets; ++b) {
                if (cw >= goal) return b;
                cw += (double)hist[b] + wl * (double)hist[kShardBuckets + b];
            }
            return kShardBuckets;
        };
        const int blo = first_bucket(c->rank), bhi = first_bucket(c->rank + 1) - 1;
        int64_t before = 0, nsel = 0;
        for (int b = 0; b < blo; ++b) before += hist[b];
        for (int b = blo; b <= bhi; ++b) nsel += hist[b];
        lo = before, hi = before + nsel, base = before;
        if (nsel > 0) {
            TRY(c->tflag.ensure((size_t)n + 64));
            launch_key_flags(c->keys_a.as<uint32_t>(), n, shift, xdiv, (uint32_t)blo, (uint32_t)bhi,
                             c->tflag.as<uint8_t>(), c->exec);
            TRY(c->misc.ensure(128));
            int32_t* d_nsel = (int32_t*)(c->misc.as<uint32_t>() + 20);
            size_t tmp = 0;
            CK(cub::DeviceSelect::Flagged(nullptr, tmp, c->keys_a.as<uint32_t>(), c->tflag.as<uint8_t>(),
                                          c->keys_b.as<uint32_t>(), d_nsel, (int)n, c->exec));
            TRY(c->cub_tmp.ensure(tmp));
            CK(cub::DeviceSelect::Flagged(c->cub_tmp.p, tmp, c->keys_a.as<uint32_t>(), c->tflag.as<uint8_t>(),
                                          c->keys_b.as<uint32_t>(), d_nsel, (int)n, c->exec));
            CK(cub::DeviceSelect::Flagged(c->cub_tmp.p, tmp, c->vals_a.as<int32_t>(), c->tflag.as<uint8_t>(),
                                          c->vals_b.as<int32_t>(), d_nsel, (int)n, c->exec));
            CK(cudaMemcpyAsync(c->keys_a.p, c->keys_b.p, (size_t)nsel * 4, cudaMemcpyDeviceToDevice, c->exec));
            CK(cudaMemcpyAsync(c->vals_a.p, c->vals_b.p, (size_t)nsel * 4, cudaMemcpyDeviceToDevice, c->exec));
            TRY(sort_pairs(c, nsel, kbits, sbits));
            c->launches += 7;
        }
    } else {
        TRY(sort_pairs(c, n, kbits, sbits));
    }
    TRY(c->src4.ensure((size_t)(hi - lo > 0 ? hi - lo : 1) * sizeof(float4)));
    if (hi > lo) launch_gather_source(dx, c->vals_b.as<int32_t>(), lo - base, hi - base, c->src4.as<float4>(), c->exec);
    c->launches += 3;
    c->ntiles = 0;
    if (c->search == 4 && !c->g.hashed && hi > lo) {
        // variant 4 tiles: a new tile at every 8^3-brick change and every
        // kTileQ queries inside a brick (deterministic: scan + stable select)
        const int64_t nl = hi - lo;
        int32_t* mark = c->vals_a.as<int32_t>();
        int32_t* run_start = (int32_t*)c->keys_a.p;
        TRY(c->tflag.ensure((size_t)nl + 64));
        TRY(c->tiles.ensure((size_t)(nl + 1) * 4));
        launch_run_marks(c->keys_b.as<uint32_t>() + lo, nl, brick == 3 ? 9 : 32, mark, c->exec);
        size_t tmp = 0;
        CK(cub::DeviceScan::InclusiveScan(nullptr, tmp, mark, run_start, cub::Max(), (int)nl, c->exec));
        TRY(c->cub_tmp.ensure(tmp));
        CK(cub::DeviceScan::InclusiveScan(c->cub_tmp.p, tmp, mark, run_start, cub::Max(), (int)nl, c->exec));
        uint8_t* flag = c->tflag.as<uint8_t>();
        launch_tile_flags(run_start, nl, kTileQ, flag, c->exec);
        TRY(c->misc.ensure(128));
        int32_t* nsel = (int32_t*)(c->misc.as<uint32_t>() + 20);
        tmp = 0;
        CK(cub::DeviceSelect::Flagged(nullptr, tmp, cub::CountingInputIterator<int32_t>(0), flag,
                                      c->tiles.as<int32_t>(), nsel, (int)nl, c->exec));
        TRY(c->cub_tmp.ensure(tmp));
        CK(cub::DeviceSelect::Flagged(c->cub_tmp.p, tmp, cub::CountingInputIterator<int32_t>(0), flag,
                                      c->tiles.as<int32_t>(), nsel, (int)nl, c->exec));
        CK(cudaMemcpyAsync(&c->ntiles, nsel, 4, cudaMemcpyDeviceToHost, c->exec));
        c->launches += 5;
    }
    c->pend_src_n = n, c->pend_src_lo = lo, c->pend_src_hi = hi;
    if (defer) return O3G_OK;
    return source_finish(c);
}

// the end of o3g_set_source: wait, read the finiteness flag and the source bbox
static o3g_status source_finish(o3g_ctx* c) {
    PhaseRange nvtx_("o3g:set_source finish");
    const uint32_t* smm = c->misc.as<uint32_t>() + 24;
    int32_t h_bad = 0;
    uint32_t h_mm[6];
    CK(cudaMemcpyAsync(&h_bad, (int32_t*)(c->misc.as<uint32_t>() + 6), 4, cudaMemcpyDeviceToHost, c->exec));
    CK(cudaMemcpyAsync(h_mm, smm, 24, cudaMemcpyDeviceToHost, c->exec));
    CK(cudaStreamSynchronize(c->exec));
    CK(cudaGetLastError());
    if (h_bad) return fail(O3G_ERR_INVALID_ARGUMENT, "non-finite source coordinate");
    for (int a = 0; a < 3; ++a) c->smax[a] = fmaxf(fabsf(ord2f(h_mm[a])), fabsf(ord2f(h_mm[3 + a])));
    c->n_total = c->pend_src_n;
    c->n_local = c->pend_src_hi - c->pend_src_lo;
    c->shard_lo = c->pend_src_lo;
    c->src_ready = true;
    return O3G_OK;
}

o3g_status o3g_set_source(o3g_ctx* c, const float* xyz, int64_t n, const double order_T[16]) {
    return set_source_impl(c, xyz, n, order_T, false);
}

static int coop_min_of(const o3g_ctx* c) {
    // auto (-1): warp-cooperative scans only where cells are dense (measured:
    // LiDAR, 226 points per occupied cell, gains 2.3x; sparse configs lose);
    // threshold 32 (with the warm start and x-windows, LiDAR K3 0.240 ms for
    // thresholds 1-32 vs 0.250 at 256)
    return c->coop_min >= 0 ? c->coop_min
                            : ((double)c->m >= 32.0 * (double)(c->occupied > 0 ? c->occupied : 1) ? 32 : 0);
}

// row pruning (variant 1, dense grid): the per-query candidate threshold, or
// -1 for the plain instantiation (before the warm start, the pre-scan form
// gained 21% K3 on depth and 8% on fragment; with it, it costs ~2%)
static int prune_of(const o3g_ctx* c) {
    if (c->g.hashed || c->prune_min == -2) return -1;
    if (c->prune_min >= 0) return c->prune_min;
    const double rho = (double)c->m / (double)(c->occupied > 0 ? c->occupied : 1);
    // >= 4 per cell: the pruning instantiation without the light pre-scan
    // (the warm start supersedes it), for its warm-start cell cuts and, at
    // >= 32 per cell, the cooperative path's row pruning (depth K3 0.044 ->
    // 0.041 ms, LiDAR 0.240 -> 0.189; the sparse large16m loses: off there)
    return rho >= 4.0 ? (1 << 30) : -1;
}

// point-to-point runs on the two-pass kernel
// (variant 4 stages a dense-table halo: a hashed grid runs variant 1)
static int k3_variant(const o3g_ctx* c) {
    return c->estimation || (c->search == 4 && (c->g.hashed || c->ntiles <= 0)) ? 1 : c->search;
}

static int k3_blocks(o3g_ctx* c, bool write_corr) {
    const int nt = k3_balanced_threads(c->n_local);
    int bps = c->bps_override ? c->bps_override : k3_max_blocks_per_sm(k3_variant(c), write_corr, c->g.hashed, prune_of(c) >= 0, nt);
    if (bps < 1) bps = 1;
    const int tpb = k3_threads(k3_variant(c), nt);
    int64_t need = (c->n_local + tpb - 1) / tpb;
    int64_t b = (int64_t)c->sms * bps;
    if (need < b) b = need;
    return (int)(b < 1 ? 1 : b);
}

static o3g_status loop_buffers(o3g_ctx* c, int blocks, int hist_cap) {
    TRY(c->partials.ensure((size_t)blocks * kTermStride * sizeof(double)));
    TRY(c->gathered.ensure((size_t)c->world * kTermStride * sizeof(double)));
    TRY(c->state.ensure(sizeof(IcpState)));
    TRY(c->hist_fit.ensure((size_t)(hist_cap > 0 ? hist_cap : 1) * sizeof(double)));
    TRY(c->hist_rmse.ensure((size_t)(hist_cap > 0 ? hist_cap : 1) * sizeof(double)));
    TRY(c->hist_T.ensure((size_t)(hist_cap > 0 ? hist_cap : 1) * 16 * sizeof(double)));
    TRY(c->hist_terms.ensure((size_t)(hist_cap > 0 ? hist_cap : 1) * kTermStride * sizeof(double)));
    return O3G_OK;
}

static K3Args k3_args(o3g_ctx* c, int32_t* corr) {
    K3Args a;
    a.src = c->src4.as<float4>();
    a.n = (int32_t)c->n_local;
    a.tpos = c->tpos.as<float4>();
    a.tnrm = c->tnrm.as<float4>();
    a.cell_start = c->cell_start.as<int32_t>();
    a.g = c->g;
    a.r2 = c->dmax * c->dmax;
    a.dmax = c->dmax;
    a.inv_dmax = 1.0 / c->dmax;
    a.st = c->state.as<IcpState>();
    a.block_partials = c->partials.as<double>();
    a.corr_out = corr;
    a.nbr_bits = (c->nbr_mask && c->nbr_ready) ? c->nbr_a.as<uint32_t>() : nullptr;
    a.cshift = c->cshift, a.cnx = c->cnx, a.cny = c->cny;
    a.p2p = c->estimation;
    a.eval_T = nullptr;
    a.n_eval = 0;
    a.coop_min = coop_min_of(c);
    a.tiles = c->tiles.as<int32_t>();
    a.ntiles = c->ntiles;
    // interleave: auto with the cooperative path (dense targets: heavy
    // queries cluster in the ordered source and would serialise a few warps)
    const bool ilv = c->interleave == 1 || (c->interleave == -1 && coop_min_of(c) > 0);
    a.ilv = ilv ? (int)((c->n_local + 31) / 32) : 0;
    a.xsorted = c->xsorted ? 1 : 0;
    a.nt = k3_balanced_threads(c->n_local);
    a.prev_j = nullptr;   // (set by the run loop: o3g_icp_run)
    a.cert = nullptr;     // (idem)
    a.need = nullptr;
    a.part_off = 0;
    a.part_total = 0;
    a.rhog_mul = c->rhog_mul;
    a.rhog_cap = c->rhog_cap;
    a.pass_expect = -1;
    a.nbr2_bits = (a.nbr_bits && !c->g.hashed) ? c->nbr_c.as<uint32_t>() : nullptr;
    a.hist_Tr = c->hist_T.as<double>();
    for (int k = 0; k < 3; ++k) a.smax[k] = c->smax[k];
    a.h_rd = round_down_f(c->g.h);
    a.inv_h_rd = round_down_f(1.0 / c->g.h);
    a.hist_T = a.hist_terms = nullptr;
    a.prune_min = prune_of(c);
    a.prune = a.prune_min >= 0;
    if (!a.prune) a.prune_min = 0;
    a.fuse_mode = 0;
    a.counter = nullptr;
    a.st_rw = nullptr;
    a.hist_fit = a.hist_rmse = nullptr;
    return a;
}

// One pass: K3 (with certificates: the sweep, then the search over the flagged
// queries), then the tail (with the rank exchange when distributed). sblocks:
// the sweep's grid (0 = no certificates); block partials [0, sblocks) are the
// sweep's, [sblocks, sblocks + blocks) the search's.
// phase (world > 1): 0 = the whole pass (NCCL all-gather); 1 = up to this rank's
// TAIL_WRITE_RANK; 2 = only the TAIL_SUM_RANKS tail (the loopback transport
// exchanges the slots between the two).
static o3g_status enqueue_pass(o3g_ctx* c, int blocks, bool write_corr, int32_t* corr,
                               int tail_mode, cudaEvent_t ev0, cudaEvent_t ev1, int* nlaunch,
                               int32_t* prev_j = nullptr, float4* cert = nullptr, int sblocks = 0,
                               int phase = 0, int pass = -1) {
    const TailHist hist{c->hist_fit.as<double>(), c->hist_rmse.as<double>(), c->hist_T.as<double>(),
                        c->hist_terms.as<double>()};
    // (timing events: external event nodes inside the run graph's capture,
    // plain records on the loopback's uncaptured stream)
    cudaStreamCaptureStatus capst = cudaStreamCaptureStatusNone;
    CK(cudaStreamIsCapturing(c->exec, &capst));
    const unsigned evflags = capst == cudaStreamCaptureStatusActive ? cudaEventRecordExternal : cudaEventRecordDefault;
    if (ev0) CK(cudaEventRecordWithFlags(ev0, c->exec, evflags));
    // variant 1 ends its pass in its last block: the A8 epilogue on one GPU,
    // the rank's slot for the exchange when distributed
    const bool fused = k3_variant(c) == 1 && c->n_local > 0;
    if (c->estimation) tail_mode |= TAIL_P2P;
    // rank exchange through peer memory (o3g_dist_peer_connect / the loopback's
    // peer transport): K3's last block publishes to every rank, the tail waits
    // (a world-1 communicator, o3g_dist_init's self-test form, runs the distributed pass too)
    const bool distp = c->world > 1 || c->comm != nullptr;
    const bool peer = c->world > 1 && c->peer_xchg;
    Xchg* const* xp = peer ? c->xpeers.as<Xchg*>() : nullptr;
    const int xmode = peer ? TAIL_PEER : 0;
    if (phase == 2) {
        launch_tail(nullptr, 0, c->gathered.as<double>(), c->world, c->rank, c->state.as<IcpState>(), hist,
                    TAIL_SUM_RANKS | tail_mode | xmode, c->exec, xp);
        ++*nlaunch;
        return O3G_OK;
    }
    if (c->n_local > 0) {
        K3Args ka = k3_args(c, corr);
        ka.prev_j = prev_j;
        ka.cert = cert;
        ka.pass_expect = pass;
        ka.part_total = blocks;
        if (cert && sblocks > 0 && c->cert_sweep) {
            ka.need = c->need.as<uint8_t>();
            launch_k3_sweep(ka, sblocks, write_corr, c->exec);
            ++*nlaunch;
            ka.part_off = sblocks;
            ka.part_total = sblocks + blocks;
        }
        if (fused) {
            ka.fuse_mode = distp ? (TAIL_WRITE_RANK | xmode) : tail_mode;
            ka.gathered = c->gathered.as<double>();
            ka.rank = c->rank;
            ka.xpeers = xp;
            ka.world = c->world;
            ka.counter = c->misc.as<unsigned int>() + 12;   // see set_target's misc layout
            ka.st_rw = c->state.as<IcpState>();
            ka.hist_fit = hist.fit;
            ka.hist_rmse = hist.rmse;
            ka.hist_T = hist.T;
            ka.hist_terms = hist.terms;
        }
        launch_k3(ka, blocks, k3_variant(c), write_corr, c->exec);
        *nlaunch += (ka.cert && k3_variant(c) == 1) ? 2 : 1;   // (both search instantiations)
    }
    if (ev1) CK(cudaEventRecordWithFlags(ev1, c->exec, evflags));
    const int nb = c->n_local > 0 ? blocks + (cert && c->cert_sweep ? sblocks : 0) : 0;
    double* gat = c->gathered.as<double>();
    IcpState* st = c->state.as<IcpState>();
    if (fused && !distp) {
        // A6/A8 ran in the last K3 block
    } else if (!distp) {
        launch_tail(c->partials.as<double>(), nb, gat, 1, 0, st, hist, TAIL_REDUCE_BLOCKS | tail_mode, c->exec);
        ++*nlaunch;
    } else {
        if (!fused) {   // (an empty shard still contributes its zero slot)
            launch_tail(c->partials.as<double>(), nb, gat, c->world, c->rank, st, TailHist{},
                        TAIL_REDUCE_BLOCKS | TAIL_WRITE_RANK | (tail_mode & TAIL_STEP) | xmode, c->exec, xp);
            ++*nlaunch;
        }
        if (phase == 1) return O3G_OK;
        if (!peer) {
            if (!c->comm) return fail(O3G_ERR_COMM, "no communicator (a loopback context runs through o3g_loopback_run)");
            nccl_result_t r = nccl().all_gather(gat + (size_t)c->rank * kTermStride, gat, kTermStride,
                                                kNcclFloat64, c->comm, c->exec);
            if (r != 0) return fail(O3G_ERR_COMM, std::string("ncclAllGather: ") +
                                                      (nccl().error_string ? nccl().error_string(r) : "?"));
        }
        launch_tail(nullptr, 0, gat, c->world, c->rank, st, hist, TAIL_SUM_RANKS | tail_mode | xmode, c->exec, xp);
        *nlaunch += 1;
    }
    return O3G_OK;
}

static void init_state(o3g_ctx* c, const double* T, int max_it, double ef, double er, int cap) {
    IcpState* s = c->h_state;
    memset(s, 0, sizeof(IcpState));
    memcpy(s->T, T, 16 * sizeof(double));
    s->max_it = max_it;
    s->rel_fit = ef;
    s->rel_rmse = er;
    s->n_total = (double)c->n_total;
    s->hist_cap = cap;
    s->cforce = c->cert_opt == 2 ? 1 : 0;
    // certificate pass tags: this run uses gbase .. gbase + max_it (mod 2^16);
    // records tagged by an earlier run are then older than any usable age. A
    // fresh buffer or a wrap-around within 64 tags resets them all.
    if (c->cert_fresh || c->cert_epoch + max_it + 1 + 64 > 65535) {
        c->cert_epoch = 0;
        s->creset = 1;
        c->cert_fresh = false;
    }
    s->gbase = c->cert_epoch;
    c->cert_epoch += max_it + 1;
    // peer-memory exchange: pass p of this run carries epoch xbase + p + 1 (never 0,
    // the cleared flag value; every rank makes the same calls, so the same epochs)
    s->xbase = c->xepoch;
    c->xepoch += (uint32_t)max_it + 2u;
}

o3g_status o3g_icp_step(o3g_ctx* c, const double T_in[16], int32_t* corr_out, double JTJ_out[36],
                        double JTr_out[6], double* inlier_count, double* sum_sq_dist,
                        double* terms_out) {
    PhaseRange nvtx_("o3g:icp_step (A3-A6, A9)");
    if (!c) return fail(O3G_ERR_INVALID_ARGUMENT, "ctx is NULL");
    if (!rigid_ok(T_in)) return fail(O3G_ERR_INVALID_ARGUMENT, "T_in is not a rigid transform");
    if (!c->src_ready) return fail(O3G_ERR_INVALID_ARGUMENT, "o3g_set_target and o3g_set_source must be called first");
    if (!c->estimation && !c->has_normals) return fail(O3G_ERR_INVALID_ARGUMENT, "point-to-plane needs target normals");
    if (corr_out && (!is_device_ptr(corr_out) || foreign_device_ptr(corr_out, c->device)))
        return fail(O3G_ERR_INVALID_ARGUMENT, "corr_out must be device memory of the context's device");
    TRY(enter(c));
    const bool wc = corr_out != nullptr;
    const int blocks = k3_blocks(c, wc);
    TRY(loop_buffers(c, blocks, 1));
    init_state(c, T_in, 0, 0.0, 0.0, 1);
    CK(cudaMemcpyAsync(c->state.p, c->h_state, sizeof(IcpState), cudaMemcpyHostToDevice, c->exec));
    int nl = 0;
    TRY(enqueue_pass(c, blocks, wc, corr_out, TAIL_STEP, nullptr, nullptr, &nl));
    c->launches += nl;
    CK(cudaMemcpyAsync(c->h_state, c->state.p, sizeof(IcpState), cudaMemcpyDeviceToHost, c->exec));
    CK(cudaStreamSynchronize(c->exec));
    CK(cudaGetLastError());
    const double* t = c->h_state->terms;
    if (JTJ_out) {
        int k = 0;
        for (int i = 0; i < 6; ++i)
            for (int j = i; j < 6; ++j) {
                JTJ_out[6 * i + j] = t[k];
                JTJ_out[6 * j + i] = t[k];
                ++k;
            }
    }
    if (JTr_out) memcpy(JTr_out, t + 21, 6 * sizeof(double));
    if (inlier_count) *inlier_count = t[27];
    if (sum_sq_dist) *sum_sq_dist = t[28];
    if (terms_out) memcpy(terms_out, t, kTerms * sizeof(double));
    return O3G_OK;
}

// certificates: variant 1's run loop, pass indices < 2^16;
// auto (-1): shards of >= 2^20 queries (on the small L2-resident configs the
// extra sweep launch and the certificate searches cost more than they save:
// depth 0.042 -> 0.117 ms per pass, tiny 0.022 -> 0.023)
static bool cert_on(const o3g_ctx* c, int max_it) {
    const bool want = c->cert_opt >= 1 || (c->cert_opt == -1 && c->n_local >= (1 << 20));
    return want && k3_variant(c) == 1 && max_it + 1 < 65535 && c->n_local > 0;
}

static int sweep_blocks(const o3g_ctx* c) {
    int bps = k3_sweep_blocks_per_sm();
    if (bps < 1) bps = 1;
    int64_t need = (c->n_local + 255) / 256;
    int64_t b = (int64_t)c->sms * bps;
    if (need < b) b = need;
    return (int)(b < 1 ? 1 : b);
}

// Per-run state (enqueued on c->exec): the first pass has no previous winners
// or certificates, every entry starts at -1 (a certificate of all ones is
// invalid; only the first 16 bytes of each 32-byte record);
// the traced correspondences start at -2 (not this rank's).
static o3g_status run_state_buffers(o3g_ctx* c, bool certm, bool trace) {
    TRY(c->prevj.ensure((size_t)(c->n_local > 0 ? c->n_local : 1) * 4));
    if (certm) {
        bool grew = false;
        TRY(c->cert.ensure((size_t)c->n_local * 2 * sizeof(float4), &grew));
        if (grew) c->cert_fresh = true;
        TRY(c->need.ensure((size_t)c->n_local + 256));   // (+ a zero tail: flags are read 8 at a time)
    }
    if (trace) TRY(c->trace_corr.ensure((size_t)c->n_total * 4));
    return O3G_OK;
}
static o3g_status run_prologue(o3g_ctx* c, bool certm, bool trace) {
    if (c->n_local > 0) CK(cudaMemsetAsync(c->prevj.p, 0xFF, (size_t)c->n_local * 4, c->exec));
    if (c->n_local > 0 && certm) launch_cert_reset(c->cert.as<float4>(), c->n_local, c->state.as<IcpState>(), c->exec);
    if (certm) CK(cudaMemsetAsync(c->need.as<uint8_t>() + c->n_local, 0, 256, c->exec));
    if (trace) launch_fill_i32(c->trace_corr.as<int32_t>(), c->n_total, -2, c->exec);
    return O3G_OK;
}

static o3g_status build_graph(o3g_ctx* c, int max_it, int blocks, int sblocks) {
    PhaseRange nvtx_("o3g:build_graph");
    GraphKey key;
    key.max_it = max_it + 1000000 * c->estimation;
    key.search = c->search;
    key.timing = c->timing;
    key.world = c->world;
    key.blocks = blocks + 100000 * sblocks;
    key.n_local = c->n_local;
    const bool certm = cert_on(c, max_it) && sblocks > 0;
    const bool trace = c->trace_pass >= 0 && c->trace_pass <= max_it;
    // the run loop's per-query state: the previous winner (warm start) and,
    // with certificates, the 32-byte records and the sweep's search flags
    TRY(run_state_buffers(c, certm, trace));
    const void* ptrs[12] = {c->src4.p, c->tpos.p, c->tnrm.p, c->cell_start.p, c->partials.p,
                            c->state.p, c->hist_fit.p, c->gathered.p, c->hist_T.p, c->hist_terms.p,
                            certm ? c->cert.p : c->prevj.p, trace ? c->trace_corr.p : c->need.p};
    memcpy(key.ptrs, ptrs, sizeof(ptrs));
    if (c->gexec && c->gkey == key) return O3G_OK;
    invalidate_graph(c);
    const size_t nev = c->timing ? 2 * (size_t)(max_it + 1) : 0;
    while (c->events.size() < nev) {
        cudaEvent_t ev;
        CK(cudaEventCreate(&ev));
        c->events.push_back(ev);
    }
    CK(cudaStreamBeginCapture(c->exec, cudaStreamCaptureModeThreadLocal));
    o3g_status st0 = run_prologue(c, certm, trace);
    if (st0 != O3G_OK) {
        cudaGraph_t g0 = nullptr;
        cudaStreamEndCapture(c->exec, &g0);
        if (g0) cudaGraphDestroy(g0);
        return st0;
    }
    int nl = (trace ? 1 : 0) + (certm && c->n_local > 0 ? 1 : 0);
    o3g_status st = O3G_OK;
    for (int p = 0; p <= max_it && st == O3G_OK; ++p) {
        const bool wc = trace && p == c->trace_pass;
        st = enqueue_pass(c, blocks, wc, wc ? c->trace_corr.as<int32_t>() : nullptr, TAIL_SOLVE,
                          c->timing ? c->events[2 * p] : nullptr,
                          c->timing ? c->events[2 * p + 1] : nullptr, &nl,
                          c->prevj.as<int32_t>(), certm ? c->cert.as<float4>() : nullptr,
                          certm ? sblocks : 0, 0, p);
    }
    cudaGraph_t graph = nullptr;
    cudaError_t e = cudaStreamEndCapture(c->exec, &graph);
    if (st != O3G_OK) {
        if (graph) cudaGraphDestroy(graph);
        return st;
    }
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(O3G_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(e));
    }
    e = cudaGraphInstantiate(&c->gexec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) {
        cudaGetLastError();
        c->gexec = nullptr;
        return fail(O3G_ERR_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(e));
    }
    c->gkey = key;
    c->graph_launches = nl;
    return O3G_OK;
}

o3g_status o3g_icp_run(o3g_ctx* c, const double init_T[16], int32_t max_iterations,
                       double relative_fitness, double relative_rmse, double T_out[16],
                       double* fitness, double* inlier_rmse, o3g_icp_info* info,
                       double* hist_fitness, double* hist_rmse) {
    PhaseRange nvtx_("o3g:icp_run (A3-A8 loop)");
    if (!c) return fail(O3G_ERR_INVALID_ARGUMENT, "ctx is NULL");
    if (!rigid_ok(init_T)) return fail(O3G_ERR_INVALID_ARGUMENT, "init_T is not a rigid transform");
    if (max_iterations < 0 || max_iterations > 100000) return fail(O3G_ERR_INVALID_ARGUMENT, "max_iterations must be in [0, 100000]");
    if (!(relative_fitness >= 0.0) || !(relative_rmse >= 0.0)) return fail(O3G_ERR_INVALID_ARGUMENT, "criteria must be >= 0");
    if (!c->src_ready) return fail(O3G_ERR_INVALID_ARGUMENT, "o3g_set_target and o3g_set_source must be called first");
    if (!T_out || !fitness || !inlier_rmse) return fail(O3G_ERR_INVALID_ARGUMENT, "T_out, fitness and inlier_rmse are required");
    if (!c->estimation && !c->has_normals) return fail(O3G_ERR_INVALID_ARGUMENT, "point-to-plane needs target normals");
    if (c->loopback) return fail(O3G_ERR_INVALID_ARGUMENT, "a loopback context runs through o3g_loopback_run");
    TRY(enter(c));
    const int blocks = k3_blocks(c, false);
    const int sblocks = cert_on(c, max_iterations) ? sweep_blocks(c) : 0;
    TRY(loop_buffers(c, blocks + sblocks, max_iterations + 1));
    // (buffers first: a new certificate buffer requests the reset in init_state)
    TRY(run_state_buffers(c, sblocks > 0, c->trace_pass >= 0 && c->trace_pass <= max_iterations));
    init_state(c, init_T, max_iterations, relative_fitness, relative_rmse, max_iterations + 1);
    CK(cudaMemcpyAsync(c->state.p, c->h_state, sizeof(IcpState), cudaMemcpyHostToDevice, c->exec));
    TRY(build_graph(c, max_iterations, blocks, sblocks));
    CK(cudaGraphLaunch(c->gexec, c->exec));
    c->launches += c->graph_launches;
    CK(cudaMemcpyAsync(c->h_state, c->state.p, sizeof(IcpState), cudaMemcpyDeviceToHost, c->exec));
    CK(cudaStreamSynchronize(c->exec));
    CK(cudaGetLastError());
    const IcpState* s = c->h_state;
    const int passes = s->passes;
    c->last_passes = passes;
    c->trace_valid = c->trace_pass >= 0 && c->trace_pass < passes;
    if (hist_fitness && passes > 0)
        CK(cudaMemcpy(hist_fitness, c->hist_fit.p, passes * sizeof(double), cudaMemcpyDeviceToHost));
    if (hist_rmse && passes > 0)
        CK(cudaMemcpy(hist_rmse, c->hist_rmse.p, passes * sizeof(double), cudaMemcpyDeviceToHost));
    memcpy(T_out, s->T, 16 * sizeof(double));
    *fitness = s->fit;
    *inlier_rmse = s->rmse;
    if (info) {
        info->iterations = s->it;
        info->passes = passes;
        info->converged = s->converged;
        info->flags = s->flags;
        info->fitness = s->fit;
        info->inlier_rmse = s->rmse;
        info->inlier_count = s->terms[27];
    }
    c->last_k3_ms = 0.0;
    c->last_tail_ms = 0.0;
    c->last_k3_launches = 0;
    if (c->timing) {
        for (int p = 0; p < passes; ++p) {
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, c->events[2 * p], c->events[2 * p + 1]));
            c->last_k3_ms += ms;
            if (p + 1 < passes) {
                CK(cudaEventElapsedTime(&ms, c->events[2 * p + 1], c->events[2 * p + 2]));
                c->last_tail_ms += ms;
            }
        }
        c->last_k3_launches = passes;
    }
    return O3G_OK;
}

o3g_status o3g_last_run_trace(o3g_ctx* c, double* T_hist, double* terms_hist, int32_t* corr_out,
                              double* stats_hist) {
    if (!c) return fail(O3G_ERR_INVALID_ARGUMENT, "ctx is NULL");
    CK(cudaSetDevice(c->device));
    const int np = c->last_passes;
    if (np > 0 && T_hist)
        CK(cudaMemcpy(T_hist, c->hist_T.p, (size_t)np * 16 * sizeof(double), cudaMemcpyDeviceToHost));
    if (np > 0 && (terms_hist || stats_hist)) {
        std::vector<double> t((size_t)np * kTermStride);
        CK(cudaMemcpy(t.data(), c->hist_terms.p, t.size() * sizeof(double), cudaMemcpyDeviceToHost));
        for (int p = 0; p < np; ++p) {
            if (terms_hist) memcpy(terms_hist + (size_t)p * kTerms, &t[(size_t)p * kTermStride], kTerms * sizeof(double));
            if (stats_hist) {
                stats_hist[3 * p] = t[(size_t)p * kTermStride + kStatSearched];
                stats_hist[3 * p + 1] = t[(size_t)p * kTermStride + kStatCandidates];
                stats_hist[3 * p + 2] = t[(size_t)p * kTermStride + kStatCertified];
            }
        }
    }
    if (corr_out && c->trace_valid)
        CK(cudaMemcpy(corr_out, c->trace_corr.p, (size_t)c->n_total * 4, cudaMemcpyDefault));
    return O3G_OK;
}

o3g_status o3g_last_run_kernel_ms(o3g_ctx* c, double* k3_ms, int32_t* k3_launches, double* tail_ms) {
    if (!c) return fail(O3G_ERR_INVALID_ARGUMENT, "ctx is NULL");
    if (k3_ms) *k3_ms = c->last_k3_ms;
    if (k3_launches) *k3_launches = c->last_k3_launches;
    if (tail_ms) *tail_ms = c->last_tail_ms;
    return O3G_OK;
}

o3g_status o3g_grid_info(o3g_ctx* c, int64_t dims[3], int64_t* table_size, int32_t* hashed,
                         int64_t* occupied_cells) {
    if (!c) return fail(O3G_ERR_INVALID_ARGUMENT, "ctx is NULL");
    if (c->m <= 0) return fail(O3G_ERR_INVALID_ARGUMENT, "no target set");
    if (dims) dims[0] = c->g.nx, dims[1] = c->g.ny, dims[2] = c->g.nz;
    if (table_size) *table_size = c->g.table_size;
    if (hashed) *hashed = c->g.hashed;
    if (occupied_cells) *occupied_cells = c->occupied;
    return O3G_OK;
}

int64_t o3g_launch_count(const o3g_ctx* c) { return c ? c->launches : 0; }

o3g_status o3g_nccl_unique_id(void* id_out) {
    if (!id_out) return fail(O3G_ERR_INVALID_ARGUMENT, "id_out is NULL");
    if (!nccl().loaded) return fail(O3G_ERR_COMM, "libnccl.so.2 not loadable");
    nccl_uid id;
    nccl_result_t r = nccl().get_unique_id(&id);
    if (r != 0) return fail(O3G_ERR_COMM, "ncclGetUniqueId failed");
    memcpy(id_out, &id, sizeof(id));
    return O3G_OK;
}

o3g_status o3g_dist_init(o3g_ctx* c, int rank, int world, const void* id) {
    if (!c) return fail(O3G_ERR_INVALID_ARGUMENT, "ctx is NULL");
    if (world < 1 || rank < 0 || rank >= world) return fail(O3G_ERR_INVALID_ARGUMENT, "bad rank/world");
    if (world > 1 && !id) return fail(O3G_ERR_INVALID_ARGUMENT, "nccl unique id required");
    CK(cudaSetDevice(c->device));
    invalidate_graph(c);
    c->src_ready = false;
    c->loopback = false;
    peer_disconnect(c);
    if (c->comm && nccl().comm_destroy) nccl().comm_destroy(c->comm);
    c->comm = nullptr;
    c->rank = rank;
    c->world = world;
    // world 1 with an id: a one-rank communicator (self-test of the NCCL leg on a
    // single GPU: every pass then runs K3 -> rank slot -> ncclAllGather -> rank-order tail)
    if (world == 1 && !id) return O3G_OK;
    if (!nccl().loaded) return fail(O3G_ERR_COMM, "libnccl.so.2 not loadable");
    nccl_uid uid;
    memcpy(&uid, id, sizeof(uid));
    nccl_result_t r = nccl().comm_init_rank(&c->comm, world, uid, rank);
    if (r != 0) {
        c->comm = nullptr;
        c->world = 1;
        c->rank = 0;
        return fail(O3G_ERR_COMM, std::string("ncclCommInitRank: ") +
                                      (nccl().error_string ? nccl().error_string(r) : "?"));
    }
    return O3G_OK;
}

o3g_status o3g_dist_init_loopback(o3g_ctx* c, int rank, int world) {
    if (!c) return fail(O3G_ERR_INVALID_ARGUMENT, "ctx is NULL");
    if (world < 1 || rank < 0 || rank >= world) return fail(O3G_ERR_INVALID_ARGUMENT, "bad rank/world");
    TRY(o3g_dist_init(c, 0, 1, nullptr));
    c->rank = rank;
    c->world = world;
    c->loopback = world > 1;
    return O3G_OK;
}

// this rank's exchange buffer: allocated once, zeroed (flag 0 = no epoch)
static o3g_status xchg_ensure(o3g_ctx* c) {
    if (c->xchg.p) return O3G_OK;
    TRY(c->xchg.ensure(sizeof(Xchg)));
    CK(cudaMemset(c->xchg.p, 0, sizeof(Xchg)));
    CK(cudaDeviceSynchronize());   // (cleared before any peer can learn the handle)
    return O3G_OK;
}

// install the table of every rank's Xchg pointer and switch the exchange over
static o3g_status peer_install(o3g_ctx* c, const std::vector<Xchg*>& table) {
    TRY(c->xpeers.ensure(table.size() * sizeof(Xchg*)));
    CK(cudaMemcpy(c->xpeers.p, table.data(), table.size() * sizeof(Xchg*), cudaMemcpyHostToDevice));
    invalidate_graph(c);
    // (epochs keep growing over the context's life, so flags left by earlier
    // runs are always below the next run's: no reset, hence no race with a
    // peer that already publishes into this rank's buffer)
    c->peer_xchg = true;
    return O3G_OK;
}

o3g_status o3g_dist_peer_handle(o3g_ctx* c, void* handle_out_64) {
    if (!c || !handle_out_64) return fail(O3G_ERR_INVALID_ARGUMENT, "ctx or handle_out is NULL");
    static_assert(sizeof(cudaIpcMemHandle_t) == O3G_PEER_HANDLE_BYTES, "IPC handle size");
    CK(cudaSetDevice(c->device));
    TRY(xchg_ensure(c));
    cudaIpcMemHandle_t h;
    CK(cudaIpcGetMemHandle(&h, c->xchg.p));
    memcpy(handle_out_64, &h, sizeof(h));
    return O3G_OK;
}

o3g_status o3g_dist_peer_connect(o3g_ctx* c, const void* handles) {
    if (!c) return fail(O3G_ERR_INVALID_ARGUMENT, "ctx is NULL");
    if (c->world < 2 || c->loopback) return fail(O3G_ERR_INVALID_ARGUMENT, "o3g_dist_init with world > 1 first");
    if (c->world > kMaxWorld) return fail(O3G_ERR_INVALID_ARGUMENT, "peer exchange supports up to 64 ranks");
    if (!handles) return fail(O3G_ERR_INVALID_ARGUMENT, "handles is NULL");
    CK(cudaSetDevice(c->device));
    TRY(xchg_ensure(c));
    peer_disconnect(c);
    std::vector<Xchg*> table(c->world);
    for (int r = 0; r < c->world; ++r) {
        if (r == c->rank) {
            table[r] = c->xchg.as<Xchg>();
            continue;
        }
        cudaIpcMemHandle_t h;
        memcpy(&h, (const char*)handles + (size_t)r * sizeof(h), sizeof(h));
        void* p = nullptr;
        cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) {
            cudaGetLastError();
            peer_disconnect(c);
            return fail(O3G_ERR_COMM, std::string("cudaIpcOpenMemHandle (rank ") + std::to_string(r) + "): " +
                                          cudaGetErrorString(e));
        }
        c->ipc_opened.push_back(p);
        table[r] = (Xchg*)p;
    }
    return peer_install(c, table);
}

o3g_status o3g_loopback_peer_connect(o3g_ctx* const* ctxs, int world) {
    if (!ctxs || world < 2 || world > kMaxWorld) return fail(O3G_ERR_INVALID_ARGUMENT, "need 2 <= world <= 64 contexts");
    std::vector<Xchg*> table(world);
    for (int r = 0; r < world; ++r) {
        o3g_ctx* c = ctxs[r];
        if (!c || c->rank != r || c->world != world || !c->loopback)
            return fail(O3G_ERR_INVALID_ARGUMENT, "ctxs[r] must be loopback rank r of world");
        if (c->device != ctxs[0]->device) return fail(O3G_ERR_INVALID_ARGUMENT, "loopback contexts share one device");
        CK(cudaSetDevice(c->device));
        TRY(xchg_ensure(c));
        table[r] = c->xchg.as<Xchg>();
    }
    for (int r = 0; r < world; ++r) {
        peer_disconnect(ctxs[r]);
        TRY(peer_install(ctxs[r], table));
    }
    return O3G_OK;
}

o3g_status o3g_loopback_run(o3g_ctx* const* ctxs, int world, const double init_T[16], int32_t max_iterations,
                            double relative_fitness, double relative_rmse, double T_out[16], double* fitness,
                            double* inlier_rmse, o3g_icp_info* info) {
    if (!ctxs || world < 1 || world > 64) return fail(O3G_ERR_INVALID_ARGUMENT, "need 1 <= world <= 64 contexts");
    if (!rigid_ok(init_T)) return fail(O3G_ERR_INVALID_ARGUMENT, "init_T is not a rigid transform");
    if (max_iterations < 0 || max_iterations > 100000) return fail(O3G_ERR_INVALID_ARGUMENT, "max_iterations must be in [0, 100000]");
    if (!(relative_fitness >= 0.0) || !(relative_rmse >= 0.0)) return fail(O3G_ERR_INVALID_ARGUMENT, "criteria must be >= 0");
    if (!T_out || !fitness || !inlier_rmse) return fail(O3G_ERR_INVALID_ARGUMENT, "T_out, fitness and inlier_rmse are required");
    for (int r = 0; r < world; ++r) {
        o3g_ctx* c = ctxs[r];
        if (!c || c->rank != r || c->world != world || (world > 1 && !c->loopback))
            return fail(O3G_ERR_INVALID_ARGUMENT, "ctxs[r] must be loopback rank r of world");
        if (!c->src_ready) return fail(O3G_ERR_INVALID_ARGUMENT, "o3g_set_target and o3g_set_source must be called first");
        if (!c->estimation && !c->has_normals) return fail(O3G_ERR_INVALID_ARGUMENT, "point-to-plane needs target normals");
        if (c->device != ctxs[0]->device) return fail(O3G_ERR_INVALID_ARGUMENT, "loopback contexts share one device");
    }
    TRY(enter(ctxs[0]));
    // every rank's work goes on ctxs[0]'s stream, in lockstep
    std::vector<cudaStream_t> saved(world);
    for (int r = 0; r < world; ++r) saved[r] = ctxs[r]->exec, ctxs[r]->exec = ctxs[0]->exec;
    auto body = [&]() -> o3g_status {
        std::vector<int> blocks(world), sblocks(world);
        std::vector<bool> certm(world), trace(world);
        for (int r = 0; r < world; ++r) {
            o3g_ctx* c = ctxs[r];
            invalidate_graph(c);
            blocks[r] = k3_blocks(c, false);
            sblocks[r] = cert_on(c, max_iterations) ? sweep_blocks(c) : 0;
            certm[r] = sblocks[r] > 0;
            trace[r] = c->trace_pass >= 0 && c->trace_pass <= max_iterations;
            TRY(loop_buffers(c, blocks[r] + sblocks[r], max_iterations + 1));
            TRY(run_state_buffers(c, certm[r], trace[r]));
            init_state(c, init_T, max_iterations, relative_fitness, relative_rmse, max_iterations + 1);
            CK(cudaMemcpyAsync(c->state.p, c->h_state, sizeof(IcpState), cudaMemcpyHostToDevice, c->exec));
            CK(cudaStreamSynchronize(c->exec));   // (h_state is reused below)
            TRY(run_prologue(c, certm[r], trace[r]));
        }
        int nl = 0;
        // O3G_OPT_TIMING on a rank: its correspondence kernels are timed per
        // pass (the ranks run one after another on this device, so each
        // rank's time is its kernels' alone: the per-GPU phase times of a
        // world-P run)
        for (int r = 0; r < world; ++r) {
            o3g_ctx* c = ctxs[r];
            const size_t nev = c->timing ? 2 * (size_t)(max_iterations + 1) : 0;
            while (c->events.size() < nev) {
                cudaEvent_t ev;
                CK(cudaEventCreate(&ev));
                c->events.push_back(ev);
            }
        }
        for (int p = 0; p <= max_iterations; ++p) {
            for (int r = 0; r < world; ++r) {
                o3g_ctx* c = ctxs[r];
                const bool wc = trace[r] && p == c->trace_pass;
                TRY(enqueue_pass(c, blocks[r], wc, wc ? c->trace_corr.as<int32_t>() : nullptr, TAIL_SOLVE,
                                 c->timing ? c->events[2 * p] : nullptr, c->timing ? c->events[2 * p + 1] : nullptr,
                                 &nl, c->prevj.as<int32_t>(), certm[r] ? c->cert.as<float4>() : nullptr,
                                 certm[r] ? sblocks[r] : 0, world > 1 ? 1 : 0, p));
            }
            if (world == 1) continue;
            // the transport: rank r's slot of its gathered buffer -> every other rank's
            // (peer transport: every rank's K3 already stored its slot into every
            // rank's Xchg and released its flag, so the tails below never spin)
            for (int r = 0; r < world && !ctxs[0]->peer_xchg; ++r)
                for (int q = 0; q < world; ++q)
                    if (q != r)
                        CK(cudaMemcpyAsync(ctxs[q]->gathered.as<double>() + (size_t)r * kTermStride,
                                           ctxs[r]->gathered.as<double>() + (size_t)r * kTermStride,
                                           kTermStride * sizeof(double), cudaMemcpyDeviceToDevice, ctxs[0]->exec));
            for (int r = 0; r < world; ++r) {
                o3g_ctx* c = ctxs[r];
                TRY(enqueue_pass(c, blocks[r], false, nullptr, TAIL_SOLVE, nullptr, nullptr, &nl, nullptr, nullptr,
                                 0, 2));
            }
        }
        for (int r = 0; r < world; ++r) ctxs[r]->launches += nl / world;
        return O3G_OK;
    };
    o3g_status st = body();
    for (int r = 0; r < world; ++r) ctxs[r]->exec = saved[r];
    TRY(st);
    CK(cudaStreamSynchronize(ctxs[0]->exec));
    CK(cudaGetLastError());
    IcpState s0;
    for (int r = 0; r < world; ++r) {
        o3g_ctx* c = ctxs[r];
        IcpState sr;
        CK(cudaMemcpy(&sr, c->state.p, sizeof(IcpState), cudaMemcpyDeviceToHost));
        if (r == 0) s0 = sr;
        else if (memcmp(sr.T, s0.T, sizeof(s0.T)) || sr.passes != s0.passes || sr.flags != s0.flags)
            return fail(O3G_ERR_CUDA, "loopback ranks diverged");
        c->last_passes = sr.passes;
        c->trace_valid = c->trace_pass >= 0 && c->trace_pass < sr.passes;
        c->last_k3_ms = 0.0;
        c->last_tail_ms = 0.0;
        c->last_k3_launches = 0;
        if (c->timing) {
            for (int p = 0; p < sr.passes; ++p) {
                float ms = 0.f;
                CK(cudaEventElapsedTime(&ms, c->events[2 * p], c->events[2 * p + 1]));
                c->last_k3_ms += ms;
            }
            c->last_k3_launches = sr.passes;
        }
    }
    memcpy(T_out, s0.T, 16 * sizeof(double));
    *fitness = s0.fit;
    *inlier_rmse = s0.rmse;
    if (info) {
        info->iterations = s0.it;
        info->passes = s0.passes;
        info->converged = s0.converged;
        info->flags = s0.flags;
        info->fitness = s0.fit;
        info->inlier_rmse = s0.rmse;
        info->inlier_count = s0.terms[27];
    }
    return O3G_OK;
}

// ------------------------------------------------------ estimate_normals
extern "C" o3g_status o3g_estimate_normals(o3g_ctx* c, const float* xyz, int64_t n, double radius,
                                           int32_t max_nn, float* out_normals, int32_t* nbr_count,
                                           int64_t* n_fallback) {
    if (!c) return fail(O3G_ERR_INVALID_ARGUMENT, "ctx is NULL");
    if (n < 3) return fail(O3G_ERR_INVALID_ARGUMENT, "estimate_normals needs at least 3 points (S:71)");
    if (max_nn < 1 || max_nn > 64) return fail(O3G_ERR_INVALID_ARGUMENT, "max_nn must be in [1, 64]");
    if (!out_normals || !is_device_ptr(out_normals) || foreign_device_ptr(out_normals, c->device))
        return fail(O3G_ERR_INVALID_ARGUMENT, "out_normals must be device memory of the context's device");
    if (nbr_count && (!is_device_ptr(nbr_count) || foreign_device_ptr(nbr_count, c->device)))
        return fail(O3G_ERR_INVALID_ARGUMENT, "nbr_count must be device memory of the context's device");
    TRY(o3g_set_target(c, xyz, nullptr, n, radius));   // the cloud's own grid, cell = radius
    c->src_ready = false;
    TRY(c->misc.ensure(64));
    unsigned long long* fb = (unsigned long long*)(c->misc.as<uint32_t>() + 14);
    CK(cudaMemsetAsync(fb, 0, 8, c->exec));
    launch_normals(c->tpos.as<float4>(), (int)n, c->cell_start.as<int32_t>(), c->g, radius * radius,
                   max_nn, out_normals, nbr_count, fb, c->exec);
    c->launches += 1;
    unsigned long long h = 0;
    CK(cudaMemcpyAsync(&h, fb, 8, cudaMemcpyDeviceToHost, c->exec));
    CK(cudaStreamSynchronize(c->exec));
    CK(cudaGetLastError());
    if (n_fallback) *n_fallback = (int64_t)h;
    return O3G_OK;
}

// ---------------------------------------- batched evaluate_registration
extern "C" o3g_status o3g_evaluate_registration(o3g_ctx* c, const double* Ts, int32_t k,
                                                double* fitness, double* inlier_rmse) {
    if (!c) return fail(O3G_ERR_INVALID_ARGUMENT, "ctx is NULL");
    if (!Ts || !fitness || !inlier_rmse || k <= 0 || k > 65535)
        return fail(O3G_ERR_INVALID_ARGUMENT, "need 1 <= k <= 65535 transforms and output arrays");
    for (int i = 0; i < k; ++i)
        if (!rigid_ok(Ts + 16 * (size_t)i)) return fail(O3G_ERR_INVALID_ARGUMENT, "a transform is not rigid");
    if (!c->src_ready) return fail(O3G_ERR_INVALID_ARGUMENT, "o3g_set_target and o3g_set_source must be called first");
    if (c->world != 1) return fail(O3G_ERR_NOT_IMPLEMENTED, "batched evaluation is single-GPU");
    TRY(enter(c));
    const int blocks = k3_blocks(c, false);
    // transforms go in chunks of <= 1024 per launch: the partials buffer stays
    // bounded (1024 x blocks x 256 B, ~155 MB at 592 blocks) for any k
    constexpr int kEvalChunk = 1024;
    const int kc = k < kEvalChunk ? k : kEvalChunk;
    TRY(c->ev_T.ensure((size_t)k * 16 * sizeof(double)));
    TRY(c->ev_part.ensure((size_t)kc * blocks * kTermStride * sizeof(double)));
    TRY(c->ev_out.ensure((size_t)k * 2 * sizeof(double)));
    TRY(c->state.ensure(sizeof(IcpState)));
    CK(cudaMemcpyAsync(c->ev_T.p, Ts, (size_t)k * 16 * sizeof(double), cudaMemcpyHostToDevice, c->exec));
    K3Args a = k3_args(c, nullptr);
    a.p2p = 1;                       // count and sum d^2 ride in the point-to-point record
    a.block_partials = c->ev_part.as<double>();
    if (c->n_local > 0) {
        for (int k0 = 0; k0 < k; k0 += kEvalChunk) {
            const int kn = k - k0 < kEvalChunk ? k - k0 : kEvalChunk;
            a.eval_T = c->ev_T.as<double>() + 16 * (size_t)k0;
            a.n_eval = kn;
            launch_k3(a, blocks, 1, false, c->exec);
            launch_eval_reduce(c->ev_part.as<double>(), blocks, kn, (double)c->n_total, c->ev_out.as<double>() + k0,
                               c->ev_out.as<double>() + k + k0, c->exec);
            c->launches += 2;
        }
    } else {
        CK(cudaMemsetAsync(c->ev_out.p, 0, (size_t)k * 2 * sizeof(double), c->exec));
    }
    CK(cudaMemcpyAsync(fitness, c->ev_out.p, (size_t)k * sizeof(double), cudaMemcpyDeviceToHost, c->exec));
    CK(cudaMemcpyAsync(inlier_rmse, c->ev_out.as<double>() + k, (size_t)k * sizeof(double),
                       cudaMemcpyDeviceToHost, c->exec));
    CK(cudaStreamSynchronize(c->exec));
    CK(cudaGetLastError());
    return O3G_OK;
}

// ------------------------------------------------- voxel downsample
static o3g_status voxel_impl(o3g_ctx* c, const float* xyz, const float* normals, int64_t n,
                             double voxel, float* out_xyz, float* out_nrm, int64_t* n_out) {
    if (n <= 0 || n > 0x7ffffffeLL) return fail(O3G_ERR_INVALID_ARGUMENT, "n must be in [1, 2^31-2]");
    if (!(voxel > 0.0) || !isfinite(voxel)) return fail(O3G_ERR_INVALID_ARGUMENT, "voxel must be finite and > 0");
    if (!xyz || !out_xyz || !n_out) return fail(O3G_ERR_INVALID_ARGUMENT, "xyz, out_xyz and n_out are required");
    TRY(enter(c));
    const float *dx, *dn = nullptr;
    TRY(device_view(c, xyz, 3 * n, c->stage_a, &dx));
    if (normals) TRY(device_view(c, normals, 3 * n, c->stage_b, &dn));
    TRY(c->misc.ensure(64));
    uint32_t* mm = c->misc.as<uint32_t>();
    int32_t* bad = (int32_t*)(mm + 6);
    CK(cudaMemsetAsync(mm, 0xFF, 12, c->exec));
    CK(cudaMemsetAsync(mm + 3, 0x00, 12 + 4, c->exec));
    launch_bbox(dx, n, mm, bad, c->sms, c->exec);
    if (dn) launch_check_finite(dn, 3 * n, bad, c->sms, c->exec);
    c->launches += dn ? 2 : 1;
    uint32_t h[7];
    CK(cudaMemcpyAsync(h, mm, 28, cudaMemcpyDeviceToHost, c->exec));
    CK(cudaStreamSynchronize(c->exec));
    if (h[6]) return fail(O3G_ERR_INVALID_ARGUMENT, "non-finite coordinate or normal");
    double mn[3];
    double cells = 1.0;
    uint64_t dims[3];
    for (int a = 0; a < 3; ++a) {
        mn[a] = (double)ord2f(h[a]);
        const double d = floor(((double)ord2f(h[3 + a]) - mn[a]) / voxel) + 1.0;
        dims[a] = (uint64_t)d;
        cells *= d;
    }
    if (!(cells < 9.0e18)) return fail(O3G_ERR_INVALID_ARGUMENT, "too many voxels in the bounding box");
    TRY(c->vk_a.ensure(n * 8));
    TRY(c->vk_b.ensure(n * 8));
    TRY(c->vals_a.ensure(n * 4));
    TRY(c->vals_b.ensure(n * 4));
    TRY(c->vflags.ensure(n * 4));
    TRY(c->vrunid.ensure(n * 4));
    TRY(c->vstarts.ensure((n + 1) * 4));
    launch_vox_keys(dx, n, mn, voxel, dims[1], dims[2], c->vk_a.as<uint64_t>(), c->vals_a.as<int32_t>(), c->exec);
    int bits = 1;
    while (bits < 64 && ((uint64_t)(cells - 1.0) >> bits)) ++bits;
    size_t tmp = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, c->vk_a.as<uint64_t>(), c->vk_b.as<uint64_t>(),
                                       c->vals_a.as<int32_t>(), c->vals_b.as<int32_t>(), (int)n, 0, bits, c->exec));
    TRY(c->cub_tmp.ensure(tmp));
    CK(cub::DeviceRadixSort::SortPairs(c->cub_tmp.p, tmp, c->vk_a.as<uint64_t>(), c->vk_b.as<uint64_t>(),
                                       c->vals_a.as<int32_t>(), c->vals_b.as<int32_t>(), (int)n, 0, bits, c->exec));
    launch_run_flags(c->vk_b.as<uint64_t>(), n, c->vflags.as<int32_t>(), c->exec);
    tmp = 0;
    CK(cub::DeviceScan::InclusiveSum(nullptr, tmp, c->vflags.as<int32_t>(), c->vrunid.as<int32_t>(), (int)n, c->exec));
    TRY(c->cub_tmp.ensure(tmp));
    CK(cub::DeviceScan::InclusiveSum(c->cub_tmp.p, tmp, c->vflags.as<int32_t>(), c->vrunid.as<int32_t>(), (int)n, c->exec));
    launch_run_starts(c->vflags.as<int32_t>(), c->vrunid.as<int32_t>(), n, c->vstarts.as<int32_t>(), c->exec);
    int32_t nruns = 0;
    CK(cudaMemcpyAsync(&nruns, c->vrunid.as<int32_t>() + (n - 1), 4, cudaMemcpyDeviceToHost, c->exec));
    CK(cudaStreamSynchronize(c->exec));
    launch_vox_mean(dx, dn, c->vals_b.as<int32_t>(), c->vstarts.as<int32_t>(), nruns, out_xyz,
                    dn ? out_nrm : nullptr, c->exec);
    c->launches += 4;
    CK(cudaStreamSynchronize(c->exec));
    CK(cudaGetLastError());
    *n_out = nruns;
    return O3G_OK;
}

extern "C" o3g_status o3g_voxel_down_sample(o3g_ctx* c, const float* xyz, const float* normals, int64_t n,
                                            double voxel, float* out_xyz, float* out_normals,
                                            int64_t* n_out) {
    if (!c) return fail(O3G_ERR_INVALID_ARGUMENT, "ctx is NULL");
    if (out_xyz && (!is_device_ptr(out_xyz) || foreign_device_ptr(out_xyz, c->device)))
        return fail(O3G_ERR_INVALID_ARGUMENT, "out_xyz must be device memory of the context's device");
    if (out_normals && (!is_device_ptr(out_normals) || foreign_device_ptr(out_normals, c->device)))
        return fail(O3G_ERR_INVALID_ARGUMENT, "out_normals must be device memory of the context's device");
    return voxel_impl(c, xyz, normals, n, voxel, out_xyz, out_normals, n_out);
}

extern "C" o3g_status o3g_icp_multiscale(o3g_ctx* c, const float* src, int64_t n, const float* tgt,
                                         const float* nrm, int64_t m, const double init_T[16],
                                         int32_t ns, const double* voxel, const double* dmax,
                                         const int32_t* iters, double rel_fit, double rel_rmse,
                                         double T_out[16], double* fit_s, double* rmse_s,
                                         int32_t* it_s, int64_t* n_s) {
    if (!c) return fail(O3G_ERR_INVALID_ARGUMENT, "ctx is NULL");
    if (ns <= 0 || !voxel || !dmax || !iters) return fail(O3G_ERR_INVALID_ARGUMENT, "need n_scales > 0 and per-scale arrays");
    if (!init_T || !rigid_ok(init_T)) return fail(O3G_ERR_INVALID_ARGUMENT, "init_T is not a rigid transform");
    if (!T_out) return fail(O3G_ERR_INVALID_ARGUMENT, "T_out is required");
    if (!src || !tgt || !nrm) return fail(O3G_ERR_INVALID_ARGUMENT, "source, target and normals are required");
    for (int s = 0; s < ns; ++s)
        if (iters[s] < 0 || !(dmax[s] > 0.0) || !(voxel[s] > 0.0))
            return fail(O3G_ERR_INVALID_ARGUMENT, "invalid per-scale parameters");
    if (n <= 0 || m <= 0) return fail(O3G_ERR_INVALID_ARGUMENT, "empty cloud");
    TRY(c->ms_src.ensure((size_t)n * 12));
    TRY(c->ms_tgt.ensure((size_t)m * 12));
    TRY(c->ms_nrm.ensure((size_t)m * 12));
    // host inputs: copied to the device once (not once per scale), on the copy
    // stream, target first, so the first target downsample overlaps the source copy
    const bool host = !is_device_ptr(src) || !is_device_ptr(tgt) || !is_device_ptr(nrm);
    if (host) {
        CK(cudaSetDevice(c->device));
        if (!c->copy) {
            CK(cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking));
            for (cudaEvent_t& e : c->ev_copy) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        }
        TRY(c->ms_in_src.ensure((size_t)n * 12));
        TRY(c->ms_in_tgt.ensure((size_t)m * 12));
        TRY(c->ms_in_nrm.ensure((size_t)m * 12));
        TRY(enter(c));
        CK(cudaEventRecord(c->ev_copy[3], c->exec));
        CK(cudaStreamWaitEvent(c->copy, c->ev_copy[3], 0));
        CK(cudaMemcpyAsync(c->ms_in_tgt.p, tgt, (size_t)m * 12, cudaMemcpyDefault, c->copy));
        CK(cudaMemcpyAsync(c->ms_in_nrm.p, nrm, (size_t)m * 12, cudaMemcpyDefault, c->copy));
        CK(cudaEventRecord(c->ev_copy[0], c->copy));
        CK(cudaMemcpyAsync(c->ms_in_src.p, src, (size_t)n * 12, cudaMemcpyDefault, c->copy));
        CK(cudaEventRecord(c->ev_copy[2], c->copy));
        CK(cudaStreamWaitEvent(c->exec, c->ev_copy[0], 0));
        src = c->ms_in_src.as<float>();
        tgt = c->ms_in_tgt.as<float>();
        nrm = c->ms_in_nrm.as<float>();
    }
    double T[16];
    memcpy(T, init_T, sizeof(T));
    for (int s = 0; s < ns; ++s) {
        int64_t nsrc = 0, ntgt = 0;
        TRY(voxel_impl(c, tgt, nrm, m, voxel[s], c->ms_tgt.as<float>(), c->ms_nrm.as<float>(), &ntgt));
        TRY(o3g_set_target(c, c->ms_tgt.as<float>(), c->ms_nrm.as<float>(), ntgt, dmax[s]));
        if (host && s == 0) CK(cudaStreamWaitEvent(c->exec, c->ev_copy[2], 0));
        TRY(voxel_impl(c, src, nullptr, n, voxel[s], c->ms_src.as<float>(), nullptr, &nsrc));
        TRY(o3g_set_source(c, c->ms_src.as<float>(), nsrc, T));
        double fit = 0, rmse = 0, Tn[16];
        o3g_icp_info info;
        TRY(o3g_icp_run(c, T, iters[s], rel_fit, rel_rmse, Tn, &fit, &rmse, &info, nullptr, nullptr));
        memcpy(T, Tn, sizeof(T));
        if (fit_s) fit_s[s] = fit;
        if (rmse_s) rmse_s[s] = rmse;
        if (it_s) it_s[s] = info.iterations;
        if (n_s) n_s[s] = nsrc;
    }
    memcpy(T_out, T, sizeof(T));
    return O3G_OK;
}

// Host inputs: the three H2D copies run in order on the copy stream (target
// xyz, normals, source) while the exec stream builds the grid as soon as the
// target xyz has landed (the gather waits for the normals, the source
// ordering for the source), so about 2/3 of the PCIe time hides the build.
static o3g_status set_inputs(o3g_ctx* c, const float* src, int64_t ns, const float* tgt,
                             const float* nrm, int64_t nt, double dmax, const double order_T[16]) {
    const bool host = !is_device_ptr(src) && !is_device_ptr(tgt) && !(nrm && is_device_ptr(nrm));
    // device-resident clouds on one GPU: the source's bbox / keys / sort / gather need
    // only the grid's dimensions, so they run on a side stream (own scratch) beside the
    // target's sort, cell table, gather and bitmaps; one final wait for both
    const bool dev3 = src && tgt && is_device_ptr(src) && is_device_ptr(tgt) && (!nrm || is_device_ptr(nrm)) &&
                      !foreign_device_ptr(src, c->device) && !foreign_device_ptr(tgt, c->device) &&
                      !(nrm && foreign_device_ptr(nrm, c->device));
    if (dev3 && c->world == 1 && c->search != 4 && c->target_sort == 1 && ns > 0 && nt > 0 &&
        ns <= 0x7effffffLL && nt <= 0x7ffffffeLL && (!order_T || rigid_ok(order_T))) {
        CK(cudaSetDevice(c->device));
        if (!c->side) {
            CK(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
            CK(cudaEventCreateWithFlags(&c->ev_side, cudaEventDisableTiming));
        }
        TRY(c->s_keys_a.ensure((size_t)ns * 4));
        TRY(c->s_keys_b.ensure((size_t)ns * 4));
        TRY(c->s_vals_a.ensure((size_t)ns * 4));
        TRY(c->s_vals_b.ensure((size_t)ns * 4));
        TRY(set_target_impl(c, tgt, nrm, nt, dmax, nullptr, /*defer_final=*/true));
        // (the side stream starts from the caller's stream position, as exec did in enter())
        CK(cudaStreamWaitEvent(c->side, c->fence, 0));
        auto swap_scratch = [&]() {
            std::swap(c->keys_a, c->s_keys_a), std::swap(c->keys_b, c->s_keys_b);
            std::swap(c->vals_a, c->s_vals_a), std::swap(c->vals_b, c->s_vals_b);
            std::swap(c->cub_tmp, c->s_cub), std::swap(c->exec, c->side);
        };
        swap_scratch();
        o3g_status st = set_source_impl(c, src, ns, order_T, /*defer=*/true);
        cudaError_t e = st == O3G_OK ? cudaEventRecord(c->ev_side, c->exec) : cudaSuccess;
        swap_scratch();
        if (st == O3G_OK && e == cudaSuccess) e = cudaStreamWaitEvent(c->exec, c->ev_side, 0);
        if (st != O3G_OK || e != cudaSuccess) {
            cudaStreamSynchronize(c->side);
            cudaStreamSynchronize(c->exec);
            c->m = 0;
            if (st != O3G_OK) return st;
            return fail(O3G_ERR_CUDA, cudaGetErrorString(e));
        }
        TRY(target_finish(c, false));
        return source_finish(c);
    }
    if (!host || ns <= 0 || nt <= 0 || ns > 0x7ffffffeLL || nt > 0x7ffffffeLL) {
        TRY(o3g_set_target(c, tgt, nrm, nt, dmax));
        return o3g_set_source(c, src, ns, order_T);
    }
    CK(cudaSetDevice(c->device));
    if (!c->copy) {
        CK(cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking));
        for (cudaEvent_t& e : c->ev_copy) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    TRY(c->stage_a.ensure((size_t)nt * 12));
    if (nrm) TRY(c->stage_b.ensure((size_t)nt * 12));
    TRY(c->stage_c.ensure((size_t)ns * 12));
    // the staging buffers may still be read by earlier work on exec / user
    TRY(enter(c));
    CK(cudaEventRecord(c->ev_copy[3], c->exec));
    CK(cudaStreamWaitEvent(c->copy, c->ev_copy[3], 0));
    CK(cudaMemcpyAsync(c->stage_a.p, tgt, (size_t)nt * 12, cudaMemcpyHostToDevice, c->copy));
    CK(cudaEventRecord(c->ev_copy[0], c->copy));
    if (nrm) CK(cudaMemcpyAsync(c->stage_b.p, nrm, (size_t)nt * 12, cudaMemcpyHostToDevice, c->copy));
    CK(cudaEventRecord(c->ev_copy[1], c->copy));
    CK(cudaMemcpyAsync(c->stage_c.p, src, (size_t)ns * 12, cudaMemcpyHostToDevice, c->copy));
    CK(cudaEventRecord(c->ev_copy[2], c->copy));
    CK(cudaStreamWaitEvent(c->exec, c->ev_copy[0], 0));
    TRY(set_target_impl(c, c->stage_a.as<float>(), nrm ? c->stage_b.as<float>() : nullptr, nt, dmax,
                        c->ev_copy[1]));
    CK(cudaStreamWaitEvent(c->exec, c->ev_copy[2], 0));
    return o3g_set_source(c, c->stage_c.as<float>(), ns, order_T);
}

o3g_status o3g_set_clouds(o3g_ctx* c, const float* source_xyz, int64_t n_source, const float* target_xyz,
                          const float* target_normals, int64_t n_target, double dmax,
                          const double order_T[16]) {
    if (!c) return fail(O3G_ERR_INVALID_ARGUMENT, "ctx is NULL");
    if (!source_xyz || !target_xyz) return fail(O3G_ERR_INVALID_ARGUMENT, "source and target xyz are required");
    return set_inputs(c, source_xyz, n_source, target_xyz, target_normals, n_target, dmax, order_T);
}

o3g_status o3g_icp_point_to_point(const float* source_xyz, int64_t n_source, const float* target_xyz,
                                  int64_t n_target, const double init_T[16], double dmax,
                                  int32_t max_iterations, double relative_fitness,
                                  double relative_rmse, double T_out[16], double* fitness,
                                  double* inlier_rmse, o3g_icp_info* info, void* cuda_stream) {
    static thread_local o3g_ctx* cached[64] = {};
    if (!init_T || !rigid_ok(init_T)) return fail(O3G_ERR_INVALID_ARGUMENT, "init_T is not a rigid transform");
    if (!source_xyz) return fail(O3G_ERR_INVALID_ARGUMENT, "source xyz is required");
    if (n_source <= 0) return fail(O3G_ERR_INVALID_ARGUMENT, "n_source must be > 0");
    int dev = 0;
    CK(cudaGetDevice(&dev));
    if (dev < 0 || dev >= 64) return fail(O3G_ERR_CUDA, "device index out of range");
    o3g_ctx*& c = cached[dev];
    if (!c) TRY(o3g_create(&c, dev, cuda_stream));
    c->user = (cudaStream_t)cuda_stream;
    TRY(o3g_set_option(c, O3G_OPT_ESTIMATION, 1));
    TRY(set_inputs(c, source_xyz, n_source, target_xyz, nullptr, n_target, dmax, init_T));
    return o3g_icp_run(c, init_T, max_iterations, relative_fitness, relative_rmse, T_out, fitness,
                       inlier_rmse, info, nullptr, nullptr);
}

// ---------------------------------------------------------- one-shot
o3g_status o3g_icp_point_to_plane(const float* source_xyz, int64_t n_source, const float* target_xyz,
                                  const float* target_normals, int64_t n_target,
                                  const double init_T[16], double dmax, int32_t max_iterations,
                                  double relative_fitness, double relative_rmse, double T_out[16],
                                  double* fitness, double* inlier_rmse, o3g_icp_info* info,
                                  void* cuda_stream) {
    static thread_local o3g_ctx* cached[64] = {};
    if (!init_T || !rigid_ok(init_T)) return fail(O3G_ERR_INVALID_ARGUMENT, "init_T is not a rigid transform");
    if (!source_xyz) return fail(O3G_ERR_INVALID_ARGUMENT, "source xyz is required");
    if (n_source <= 0) return fail(O3G_ERR_INVALID_ARGUMENT, "n_source must be > 0");
    int dev = 0;
    CK(cudaGetDevice(&dev));
    if (dev < 0 || dev >= 64) return fail(O3G_ERR_CUDA, "device index out of range");
    o3g_ctx*& c = cached[dev];
    if (!c) TRY(o3g_create(&c, dev, cuda_stream));
    c->user = (cudaStream_t)cuda_stream;
    TRY(set_inputs(c, source_xyz, n_source, target_xyz, target_normals, n_target, dmax, init_T));
    return o3g_icp_run(c, init_T, max_iterations, relative_fitness, relative_rmse, T_out, fitness,
                       inlier_rmse, info, nullptr, nullptr);
}

}  // extern "C"
