// capi.cu -- the extern "C" boundary (include/gabp_b200.h) and the host side of the
// solve loop.  The loop itself is device-driven: every sweep launch evaluates the
// convergence test of the sweep two launches back (gabp_internal.cuh, Ctrl), so the
// host only enqueues CUDA-graph chunks of sweeps and polls one flag per chunk, one
// chunk ahead -- no per-sweep host synchronisation.
#include <float.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <dlfcn.h>
#include <chrono>
#include <nccl.h>  // types only: libnccl is loaded at run time (gabp_dist_attach)

#include <atomic>
#include <mutex>
#include <omp.h>
#include <vector>

#include "gabp_internal.cuh"

using gabp::Ctrl;
using gabp::DeviceGraph;
using gabp::SweepArgs;

namespace {
thread_local char g_err[1024] = "";

int fail(int code, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return code;
}

#define CK(call)                                                                             \
    do {                                                                                     \
        cudaError_t _e = (call);                                                             \
        if (_e != cudaSuccess)                                                               \
            return fail(_e == cudaErrorMemoryAllocation ? GABP_ENOMEM : GABP_ECUDA,          \
                        "%s failed: %s (%s:%d)", #call, cudaGetErrorString(_e), __FILE__,    \
                        __LINE__);                                                           \
    } while (0)

}  // namespace

// ---- NCCL, loaded on first use so the library has no link-time NCCL dependency --------
struct NcclApi {
    void *h = nullptr;
    ncclResult_t (*getUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*allReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t,
                              ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*send)(const void *, size_t, ncclDataType_t, int, ncclComm_t,
                         cudaStream_t) = nullptr;
    ncclResult_t (*recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*groupStart)() = nullptr;
    ncclResult_t (*groupEnd)() = nullptr;
    const char *(*errorString)(ncclResult_t) = nullptr;
};

// Multi-rank state of a graph that holds one rank's row block.
struct DistState {
    bool comm_nccl = true;         // false for in-process partitions (device copies)
    int rank = 0, world = 1;
    int64_t n_global = 0;
    double bnorm = 0.0;
    bool local = false;            // in-process partitions (no NCCL): gabp_dist_solve_local
    ncclComm_t comm = nullptr;
    std::vector<int> peers;
    std::vector<int64_t> scount, rcount, soff, roff;  // nodes per peer, offsets
    uint32_t *d_sidx = nullptr, *d_ridx = nullptr;
    double *d_sbuf = nullptr, *d_rbuf = nullptr;       // 4 doubles per node, per-peer blocks
    double *d_stats = nullptr;                          // [0..4] max, [5] sum
    // split sweep (boundary groups, then interior groups under the exchange)
    cudaStream_t xstream = nullptr;  // exchange stream
    cudaEvent_t ev_bnd = nullptr, ev_sweep = nullptr, ev_done = nullptr;
    // launch protocol agreed by every rank (dist_agree): the kernel family (slice layout or
    // recomputing tiles: the statistics' sweep lag) and the split sweep (the NCCL call
    // sequence) must be the same on all ranks, whatever each rank's own layout allows;
    // -1 until agreed
    int use_slices = -1, use_split = -1;
    int64_t split_launches = 0;      // split sweeps run by the last solve (report)
    // diagonal layout across ranks (every rank a stencil graph with the same diagonals):
    // per peer the diagonals whose incoming messages cross the cut, each way
    int use_dia = 0;
    std::vector<gabp::DiaHalo> dsend, drecv;
    int dia_w = 0;                   // doubles per exchanged node: {P, x} + 2 per diagonal
    double *d_dsbuf = nullptr, *d_drbuf = nullptr;
};

// pinned host mirror of a graph's controller and poll flags (capi.cu pinned_get)
struct PinnedBlock {
    Ctrl ctrl;
    int32_t done[4];
};

struct gabp_graph {
    // owner handle + one per live gabp_state: destruction order between a graph and
    // its states does not matter (Python GC may finalise either first)
    std::atomic<int> refs{1};
    DeviceGraph g;
    cudaStream_t stream = nullptr;
    int device = 0;
    int is_dense = 0;
    // solve workspace
    double2 *msg[3] = {nullptr, nullptr, nullptr};
    double2 *agg[3] = {nullptr, nullptr, nullptr};
    gabp::NodeState *rec[3] = {nullptr, nullptr, nullptr};  // slice path node states
    double *x[3] = {nullptr, nullptr, nullptr};
    double *p[3] = {nullptr, nullptr, nullptr};
    double *rsq_part = nullptr;
    double *rsq_grp = nullptr;
    Ctrl *ctrl = nullptr;
    Ctrl *h_ctrl = nullptr;          // pinned mirror
    int32_t *h_done = nullptr;       // pinned, 2 poll slots
    char *ws_base = nullptr;         // the solve workspace block (msg ... ctrl)
    size_t ws_bytes = 0;
    PinnedBlock *pin = nullptr;
    double *change_hist = nullptr, *res_hist = nullptr, *rsq_hist = nullptr;
    int64_t hist_cap = 0;
    uint64_t ws_gen = 0;
    int64_t kernels_launched = 0;  // kernels the last solve loop enqueued (report)
    // cached CUDA graph of a chunk of sweep launches
    cudaGraphExec_t chunk_exec = nullptr;
    int chunk_len = 0, chunk_sched = -1, chunk_gather = -1;
    uint64_t chunk_gen = 0;
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    double *xhist = nullptr;  // device means history (only while a solve asks for it)
    bool slice_order = false;  // the last solve's x / p ring is in slice position order
    int bins_used = 0;         // the last solve ran the row kernel in binned message order
    double *xs = nullptr, *ps = nullptr;  // row-order copies of the returned marginals
    int64_t xhist_rows = 0;
    DistState *dist = nullptr;
    // dense variant (gabp_graph_create_dense): A and the padded message matrix ring
    int64_t K = 0;
    double *dA = nullptr;
    double2 *dmsg[3] = {nullptr, nullptr, nullptr};
    double2 *dnode = nullptr;
    uint32_t *demask = nullptr;      // edge bitmask: initial (-0, +0) non-edge messages
    int64_t Kp = 0;                  // padded dimension (multiple of 32)
    uint2 *dpairs = nullptr;         // tile pairs of the pair-tile kernel
    int64_t dnpairs = 0;
    // serial schedule: dependency levels of the last order (gabp_sweep_serial)
    bool serial_valid = false, serial_ascending = false;
    std::vector<int64_t> serial_order;
    std::vector<int64_t> serial_lvl;       // task offsets per level
    uint2 *d_serial = nullptr;             // tasks {node, order position}, level by level
    int64_t *d_serial_lvl = nullptr;       // level offsets on the device
    double2 *serial_strip = nullptr;       // global term strips of tasks > 256 edges
    int64_t serial_strip_stride = 0;
    int64_t serial_maxw = 0;               // tasks of the widest level
    cudaGraphExec_t serial_exec = nullptr; // the level launches, captured once per order
    uint64_t serial_gen = 0;               // workspace generation of the capture
    double serial_lim = 0.0;               // blow-up limit of the capture
    std::vector<uint32_t> h_rp, h_col;     // host CSR (level build)
    int small_state = 0;                   // small.cu plan: 0 not tried, 1 fits, -1 does not
    gabp::SmallPart small_part = {};
};

struct gabp_state {
    const gabp_graph *g = nullptr;
    double2 *buf[2] = {nullptr, nullptr};
    int cur = 0;
    int64_t iteration = 0;
    int64_t messages_sent = 0;
};

namespace {

NcclApi g_nccl;

int load_nccl() {
    if (g_nccl.h) return GABP_OK;
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return fail(GABP_ECUDA, "cannot load libnccl.so.2: %s", dlerror());
#define NCCL_SYM(field, name)                                                           \
    g_nccl.field = reinterpret_cast<decltype(g_nccl.field)>(dlsym(h, name));             \
    if (!g_nccl.field) return fail(GABP_ECUDA, "libnccl lacks %s", name);
    NCCL_SYM(getUniqueId, "ncclGetUniqueId");
    NCCL_SYM(commInitRank, "ncclCommInitRank");
    NCCL_SYM(commDestroy, "ncclCommDestroy");
    NCCL_SYM(allReduce, "ncclAllReduce");
    NCCL_SYM(send, "ncclSend");
    NCCL_SYM(recv, "ncclRecv");
    NCCL_SYM(groupStart, "ncclGroupStart");
    NCCL_SYM(groupEnd, "ncclGroupEnd");
    NCCL_SYM(errorString, "ncclGetErrorString");
#undef NCCL_SYM
    g_nccl.h = h;
    return GABP_OK;
}

#define NK(call)                                                                          \
    do {                                                                                  \
        ncclResult_t _r = (call);                                                         \
        if (_r != ncclSuccess)                                                            \
            return fail(GABP_ECUDA, "%s failed: %s", #call, g_nccl.errorString(_r));      \
    } while (0)

// GABP_HOST_TIMING=1: host-clock phase times of the drop-in calls on stderr
double host_ms() {
    return std::chrono::duration<double, std::milli>(
               std::chrono::steady_clock::now().time_since_epoch())
        .count();
}
bool host_timing() {
    static const int on = getenv("GABP_HOST_TIMING") ? atoi(getenv("GABP_HOST_TIMING")) : 0;
    return on != 0;
}

// stream-ordered free of a pool block (no-op for NULL)
inline void afree(void *p, cudaStream_t st) {
    if (p) cudaFreeAsync(p, st);
}

// message slots of the solve ring: CSR edges, or slice slots (padding included)
int64_t msg_slots(const DeviceGraph &g) {
    const int64_t ns = g.nslices > 0 ? g.nslots + gabp::kSlotPad : 0;
    int64_t m = g.E > ns ? g.E : ns;
    if ((int64_t)g.dia_D * g.n > m) m = (int64_t)g.dia_D * g.n;  // diagonal layout (dia.cu)
    return m > 0 ? m : 1;
}

// Pinned host mirrors (controller + poll flags) come from a process-wide slab: a
// cudaMallocHost per graph costs about a millisecond of page locking.
std::mutex g_pin_mu;
std::vector<PinnedBlock *> g_pin_free;

PinnedBlock *pinned_get() {
    std::lock_guard<std::mutex> lk(g_pin_mu);
    if (g_pin_free.empty()) {
        constexpr int kPer = 64;
        PinnedBlock *slab = nullptr;
        if (cudaMallocHost(&slab, sizeof(PinnedBlock) * kPer) != cudaSuccess) return nullptr;
        for (int k = 0; k < kPer; ++k) g_pin_free.push_back(slab + k);  // never returned
    }
    PinnedBlock *b = g_pin_free.back();
    g_pin_free.pop_back();
    return b;
}
void pinned_put(PinnedBlock *b) {
    if (!b) return;
    std::lock_guard<std::mutex> lk(g_pin_mu);
    g_pin_free.push_back(b);
}

// Spare large blocks (a released solve workspace, a graph-create staging buffer) are
// kept per device and handed to the next request of a similar size.  Taking them from the
// pool instead costs a re-mapping of the whole range whenever smaller allocations have
// been carved out of the freed block in between (about 1 ms per GB).
struct SpareBlock {
    int device = -1;
    void *p = nullptr;
    size_t bytes = 0;
};
std::mutex g_spare_mu;
SpareBlock g_spare[2][16];  // [kind][slot]: 0 workspace, 1 staging

void *spare_take(int kind, int device, size_t bytes) {
    std::lock_guard<std::mutex> lk(g_spare_mu);
    for (auto &b : g_spare[kind])
        if (b.p && b.device == device && b.bytes >= bytes && b.bytes <= 2 * bytes + (64u << 20)) {
            void *p = b.p;
            b.p = nullptr;
            return p;
        }
    return nullptr;
}
// p must be idle (its stream synchronized); returns false when no slot is free
bool spare_keep(int kind, int device, void *p, size_t bytes) {
    std::lock_guard<std::mutex> lk(g_spare_mu);
    for (auto &b : g_spare[kind])
        if (!b.p) {
            b.device = device;
            b.p = p;
            b.bytes = bytes;
            return true;
        }
    return false;
}

// Frees the spare blocks of a device and trims its pool: the memory of earlier graphs comes
// back to the device (on an allocation failure, and on request: gabp_release_cached).
void release_spares(int device) {
    std::vector<void *> ps;
    {
        std::lock_guard<std::mutex> lk(g_spare_mu);
        for (auto &k : g_spare)
            for (auto &b : k)
                if (b.p && b.device == device) {
                    ps.push_back(b.p);
                    b.p = nullptr;
                }
    }
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(device);
    for (void *p : ps) cudaFreeAsync(p, 0);
    cudaStreamSynchronize(0);
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
    cudaSetDevice(cur);
}

// One stream-ordered block from the retained device pool holds the whole solve workspace
// (a repeated solve, or a new graph of similar size, reuses the cached block).
struct Carve {
    char *base;
    size_t off = 0;
    template <class T>
    T *take(int64_t count) {
        off = (off + 255) & ~(size_t)255;
        T *p = reinterpret_cast<T *>(base ? base + off : nullptr);
        off += sizeof(T) * (size_t)(count > 0 ? count : 1);
        return p;
    }
};

void carve_workspace(gabp_graph *G, Carve &c) {
    const DeviceGraph &g = G->g;
    const int64_t E = msg_slots(g);
    // node arrays: row order (tiles) or position order (slices, padding lanes + halo)
    const int64_t nn = (g.n > g.npos ? g.n : g.npos) + gabp::kNodePad;
    // the diagonal kernel stages ranges shifted by up to the widest offset: pad both sides
    const int64_t pad = g.dia_D > 0 ? gabp::dia_pad(g.dia_O) : 0;
    for (int b = 0; b < 3; ++b) {
        G->msg[b] = c.take<double2>(E + 2 * pad);
        if (G->msg[b]) G->msg[b] += pad;
    }
    for (int b = 0; b < 3; ++b) G->agg[b] = c.take<double2>(nn);
    for (int b = 0; b < 3; ++b) {
        G->x[b] = c.take<double>(nn + 2 * pad);
        G->p[b] = c.take<double>(nn + 2 * pad);
        if (G->x[b]) {
            G->x[b] += pad;
            G->p[b] += pad;
        }
    }
    for (int b = 0; b < 3; ++b)
        G->rec[b] = g.nslices > 0 ? c.take<gabp::NodeState>(g.npos + gabp::kNodePad) : nullptr;
    G->xs = c.take<double>(g.n + 1);
    G->ps = c.take<double>(g.n + 1);
    // one partial per CTA of a persistent launch (either layout)
    G->rsq_part = c.take<double>(g.ntiles > 8192 ? g.ntiles : 8192);
    // one partial per slice group (group TMA kernels: dynamic claims, fixed summation order)
    G->rsq_grp = c.take<double>(g.nslices / 15 + 1);
    G->ctrl = c.take<Ctrl>(1);
}

int ensure_workspace(gabp_graph *G, int64_t max_iter) {
    cudaStream_t st = G->stream;
    const DeviceGraph &g = G->g;
    const double tw0 = host_ms();
    double tw1 = tw0, tw2 = tw0;
    if (!G->ws_base) {
        Carve size{nullptr};
        carve_workspace(G, size);
        G->ws_base = static_cast<char *>(spare_take(0, G->device, size.off));
        if (!G->ws_base && cudaMallocAsync(&G->ws_base, size.off, st) != cudaSuccess) {
            cudaGetLastError();  // out of memory: give the cached spares back, retry once
            G->ws_base = nullptr;
            release_spares(G->device);
            CK(cudaMallocAsync(&G->ws_base, size.off, st));
        }
        G->ws_bytes = size.off;
        tw1 = host_ms();
        Carve c{G->ws_base};
        carve_workspace(G, c);
        const int64_t nn = (g.n > g.npos ? g.n : g.npos) + gabp::kNodePad;
        for (int b = 0; b < 3; ++b) CK(cudaMemsetAsync(G->x[b], 0, sizeof(double) * nn, st));
        G->pin = pinned_get();
        if (!G->pin) return fail(GABP_ENOMEM, "pinned host allocation failed");
        G->h_ctrl = &G->pin->ctrl;
        G->h_done = G->pin->done;
        for (int k = 0; k < 4; ++k) CK(cudaEventCreateWithFlags(&G->ev[k], cudaEventDefault));
        tw2 = host_ms();
        CK(cudaStreamSynchronize(st));  // usable from any stream from here on
        G->ws_gen++;
    }
    if (max_iter > G->hist_cap) {
        afree(G->change_hist, st);
        CK(cudaMallocAsync(&G->change_hist, sizeof(double) * 3 * max_iter, st));
        G->res_hist = G->change_hist + max_iter;
        G->rsq_hist = G->change_hist + 2 * max_iter;
        CK(cudaStreamSynchronize(st));
        G->hist_cap = max_iter;
        G->ws_gen++;
    }
    if (host_timing()) {
        cudaMemPool_t pool;
        cudaDeviceGetMemPool(&pool, G->device);
        uint64_t res = 0, used = 0;
        cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &res);
        cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used);
        fprintf(stderr, "[gabp] workspace: alloc %.2f ms, carve+memset+pin+events %.2f ms, "
                        "syncs + history %.2f ms; pool reserved %.2f GB used %.2f GB\n",
                tw1 - tw0, tw2 - tw1, host_ms() - tw2, res / 1e9, used / 1e9);
    }
    return GABP_OK;
}

SweepArgs make_args(gabp_graph *G) {
    SweepArgs a{};
    const DeviceGraph &g = G->g;
    a.strip = G->serial_strip;
    a.strip_stride = G->serial_strip_stride;
    a.dia_D = g.dia_D;
    a.dia_nl = g.n;
    a.dia_r0 = g.row_lo;
    a.dia_r1 = g.row_hi;
    a.dia_coef = g.dia_coef;
    a.dia_mask = g.dia_mask;
    a.dia_cu = g.dia_cu;
    a.dia_nlc = g.dia_nlc;
    a.dia_O = g.dia_O;
    a.dia_W = g.dia_W;
    for (int k = 0; k < gabp::kDiaMaxD; ++k) {
        a.dia_off[k] = g.dia_off.v[k];
        a.dia_opp[k] = g.dia_opp[k];
    }
    a.n = g.n;
    a.ntiles = g.ntiles;
    a.row_ptr = g.row_ptr;
    a.tile_start = g.tile_start;
    a.tile_info = g.tile_info;
    a.er = g.er;
    a.nd = g.nd;
    a.diag = g.diag;
    a.prior_num = g.prior_num;
    a.rhs = g.rhs;
    for (int b = 0; b < 3; ++b) a.msg[b] = G->msg[b];
    for (int b = 0; b < 3; ++b) a.agg[b] = G->agg[b];
    for (int b = 0; b < 3; ++b) {
        a.x[b] = G->x[b];
        a.p[b] = G->p[b];
    }
    a.rsq_part = G->rsq_part;
    a.rsq_grp = G->rsq_grp;
    a.ctrl = G->ctrl;
    a.change_hist = G->change_hist;
    a.res_hist = G->res_hist;
    a.rsq_hist = G->rsq_hist;
    a.xhist = G->xhist;
    a.xhist_rows = G->xhist_rows;
    a.msg_lag = 0;
    for (int b = 0; b < 3; ++b) a.rec[b] = G->rec[b];
    a.slice_variant = g.slice_variant;
    a.slice_path = 0;
    a.nslices = g.nslices;
    a.slice_info = g.slice_info;
    a.gorder = getenv("GABP_NO_GORDER") ? nullptr : g.gorder;  // (A/B: claim order)
    a.sdeg = g.sdeg;
    a.srow = g.srow;
    a.snd = g.snd;
    a.srhs = g.srhs;
    a.scol = g.scol;
    a.scoef = g.scoef;
    a.stwin = g.stwin;
    {
        // slots per lane of the four-rows-per-warp kernel: the smallest instantiation that
        // leaves at most one row in 1024 to the long-row path (GABP_QUAD_SLOTS: A/B)
        const int64_t few = g.n / 1024;
        a.quad_slots = g.rows_gt16 <= few   ? 2
                       : g.rows_gt32 <= few ? 4
                       : g.rows_gt48 <= few ? 6
                                            : 8;
        if (const char *qs = getenv("GABP_QUAD_SLOTS")) a.quad_slots = atoi(qs);
    }
    if (g.bins > 0 && !getenv("GABP_ROW_NO_BIN")) {  // (A/B: CSR message order)
        a.gidx = g.gidx;
        a.gcoef = g.gcoef;
        a.gout = g.gout;
    }
    a.sl_lo = 0;
    a.sl_hi = g.nslices;
    a.part_base = 0;
    a.exact_primary = 0;
    return a;
}

void release_workspace(gabp_graph *G) {
    cudaStream_t st = G->stream;
    // (graph_release synchronized the stream: the block is idle)
    if (G->ws_base && !spare_keep(0, G->device, G->ws_base, G->ws_bytes)) afree(G->ws_base, st);
    afree(G->change_hist, st);  // (res_hist, rsq_hist live in the same block)
    afree(G->xhist, st);
    pinned_put(G->pin);
    if (G->chunk_exec) cudaGraphExecDestroy(G->chunk_exec);
    cudaFree(G->dA);
    for (int b = 0; b < 3; ++b) cudaFree(G->dmsg[b]);
    cudaFree(G->dnode);
    cudaFree(G->demask);
    cudaFree(G->dpairs);
    if (G->dist) {
        cudaFree(G->dist->d_sidx);
        cudaFree(G->dist->d_ridx);
        cudaFree(G->dist->d_sbuf);
        cudaFree(G->dist->d_rbuf);
        if (G->dist->d_dsbuf) cudaFree(G->dist->d_dsbuf);
        if (G->dist->d_drbuf) cudaFree(G->dist->d_drbuf);
        cudaFree(G->dist->d_stats);
        if (G->dist->xstream) cudaStreamDestroy(G->dist->xstream);
        if (G->dist->ev_bnd) cudaEventDestroy(G->dist->ev_bnd);
        if (G->dist->ev_sweep) cudaEventDestroy(G->dist->ev_sweep);
        if (G->dist->ev_done) cudaEventDestroy(G->dist->ev_done);
        if (G->dist->comm && g_nccl.commDestroy) g_nccl.commDestroy(G->dist->comm);
        delete G->dist;
        G->dist = nullptr;
    }
    for (int k = 0; k < 4; ++k)
        if (G->ev[k]) cudaEventDestroy(G->ev[k]);
}

int check_options(const gabp_options_t *opt) {
    if (!opt) return fail(GABP_EINVAL, "options must not be NULL");
    if (!(opt->epsilon > 0.0)) return fail(GABP_EINVAL, "epsilon must be positive");
    if (opt->max_iter < 1) return fail(GABP_EINVAL, "max_iter must be >= 1");
    if (!(opt->blowup > 1.0)) return fail(GABP_EINVAL, "blowup must exceed 1");
    if (opt->schedule != GABP_SCHED_PARALLEL && opt->schedule != GABP_SCHED_BROADCAST)
        return fail(GABP_EINVAL, "schedule must be parallel (0) or broadcast (2)");
    if (opt->gather_mode < GABP_GATHER_AUTO || opt->gather_mode > GABP_GATHER_ROWS)
        return fail(GABP_EINVAL, "unknown gather mode %d", opt->gather_mode);
    return GABP_OK;
}

int check_slice(const gabp_graph *G, const gabp_options_t *opt) {
    if (opt->gather_mode == GABP_GATHER_SLICE && G->g.nslices == 0)
        return fail(GABP_EINVAL, "graph has no slice layout (max degree %lld)",
                    (long long)G->g.max_degree);
    if (opt->gather_mode == GABP_GATHER_ROWS && opt->schedule == GABP_SCHED_PARALLEL &&
        G->g.max_degree > gabp::kRowParMaxDegree)
        return fail(GABP_EINVAL, "gather mode rows: max degree %lld > %d",
                    (long long)G->g.max_degree, gabp::kRowParMaxDegree);
    return GABP_OK;
}

// kernel family of a multi-rank launch: slice layout when built, else recomputing tiles
int dist_gather(const gabp_graph *G) {
    if (G->dist && G->dist->use_slices >= 0)
        return G->dist->use_slices ? gabp::kGatherSlice : gabp::kGatherRecompute;
    return G->g.nslices > 0 ? gabp::kGatherSlice : gabp::kGatherRecompute;
}

// Gather mode of the broadcast solve: recompute the twin message from the node aggregate
// (L2-resident, contiguous DRAM traffic only) when the twin messages are far away in
// memory; gather the twin message itself when it is near (structured grids).
int pick_gather(const gabp_graph *G, const gabp_options_t *opt) {
    if (opt->schedule != GABP_SCHED_BROADCAST) {
        // parallel schedule: the slice-group kernel (exclusion sums over the row's
        // contiguous incoming slots, scattered twin stores) on whole graphs with slices
        const bool whole = G->g.row_lo == 0 && G->g.row_hi == G->g.n;
        if (opt->gather_mode == GABP_GATHER_ROWS) return gabp::kGatherRowParallel;
        // mean degree >= 7: four rows per warp (rowpar.cu: rowquad_kernel; config 1, mean
        // 32: 0.80 ms/sweep against 1.70 for the slice groups, whose later passes re-stream
        // the row); lower degrees stay on the slice groups (random graphs of 512 k rows,
        // tools/par_degree_probe.py, slice / rows: mean degree 4 0.094 / 0.116 ms, 8
        // 0.190 / 0.167, 12 0.300 / 0.197, 24 0.580 / 0.357)
        if (opt->gather_mode == GABP_GATHER_AUTO && whole && G->g.n > 0 &&
            G->g.E >= 7 * G->g.n && G->g.max_degree <= gabp::kRowParMaxDegree)
            return gabp::kGatherRowParallel;
        if (opt->gather_mode == GABP_GATHER_SLICE ||
            (opt->gather_mode == GABP_GATHER_AUTO && G->g.nslices > 0 && whole))
            return gabp::kGatherSliceParallel;
        return gabp::kGatherMessage;
    }
    if (opt->gather_mode == GABP_GATHER_MESSAGE) return gabp::kGatherMessage;
    if (opt->gather_mode == GABP_GATHER_RECOMPUTE) return gabp::kGatherRecompute;
    if (G->g.nslices > 0) return gabp::kGatherSlice;  // AUTO or SLICE
    return G->g.twin_span * 16.0 > 4.0e6 ? gabp::kGatherRecompute : gabp::kGatherMessage;
}

int auto_chunk(const gabp_graph *G) {
    // aim for ~1.5 ms of sweeps between host polls (sweep ~ 72 B/edge + 52 B/node)
    const double bytes = 72.0 * (double)G->g.E + 52.0 * (double)G->g.n;
    const double us = fmax(4.0, bytes / 6.5e6);
    int c = (int)(1500.0 / us);
    if (c < 2) c = 2;
    if (c > 64) c = 64;
    return c;
}

bool chunk_exec_ready(const gabp_graph *G, int sched, int gather, int len) {
    return G->chunk_exec && G->chunk_len == len && G->chunk_sched == sched &&
           G->chunk_gather == gather && G->chunk_gen == G->ws_gen;
}

int get_chunk_exec(gabp_graph *G, int sched, int gather, int len) {
    if (chunk_exec_ready(G, sched, gather, len)) return GABP_OK;
    if (G->chunk_exec) {
        cudaGraphExecDestroy(G->chunk_exec);
        G->chunk_exec = nullptr;
    }
    SweepArgs a = make_args(G);
    cudaGraph_t graph;
    CK(cudaStreamBeginCapture(G->stream, cudaStreamCaptureModeThreadLocal));
    for (int k = 0; k < len; ++k) {
        cudaError_t e = gabp::launch_sweep(a, sched, gabp::kModeSolve, gather, G->stream);
        if (e != cudaSuccess) {
            cudaStreamEndCapture(G->stream, &graph);
            return fail(GABP_ECUDA, "capture: %s", cudaGetErrorString(e));
        }
    }
    CK(cudaStreamEndCapture(G->stream, &graph));
    cudaError_t e = cudaGraphInstantiate(&G->chunk_exec, graph, 0);
    cudaGraphDestroy(graph);
    CK(e);
    G->chunk_len = len;
    G->chunk_sched = sched;
    G->chunk_gather = gather;
    G->chunk_gen = G->ws_gen;
    return GABP_OK;
}

// Common setup of a solve: options, workspace, controller, S_0 = 0.
int solve_setup(gabp_graph *G, const gabp_options_t *opt) {
    int rc = check_options(opt);
    if (rc) return rc;
    if (G->dist) G->dist->split_launches = 0;
    CK(cudaSetDevice(G->device));
    rc = ensure_workspace(G, opt->max_iter);
    if (rc) return rc;
    const DeviceGraph &g = G->g;
    const int64_t rows = opt->h_means_history ? opt->means_history_rows : 0;
    if (rows != G->xhist_rows) {
        afree(G->xhist, G->stream);
        G->xhist = nullptr;
        G->xhist_rows = 0;
        if (rows > 0) CK(cudaMallocAsync(&G->xhist, sizeof(double) * rows * g.n, G->stream));
        G->xhist_rows = rows;
        G->ws_gen++;
    }
    Ctrl c = gabp::fresh_ctrl();
    c.next_sweep = 1;
    c.epsilon = opt->epsilon;
    c.blowup = opt->blowup;
    c.rel_tol = opt->rel_residual_tol;
    c.bnorm = G->dist ? G->dist->bnorm : g.rhs_norm;
    c.max_iter = opt->max_iter;
    c.n = G->dist ? G->dist->n_global : g.n;
    *G->h_ctrl = c;
    cudaStream_t st = G->stream;
    CK(cudaMemcpyAsync(G->ctrl, G->h_ctrl, sizeof(Ctrl), cudaMemcpyHostToDevice, st));
    CK(cudaMemsetAsync(G->msg[0], 0, sizeof(double2) * msg_slots(g), st));  // S_0 = 0
    return GABP_OK;
}

// Poll bookkeeping shared by the loops: the done flag of chunk k is read after chunk k+1
// has been enqueued, so the device never idles on the host.
struct Poller {
    gabp_graph *G;
    int poll = 0;
    bool pending = false;
    // returns 1 when the previous chunk's flag says done
    int after_chunk(cudaStream_t st, int *rc) {
        const int slot = poll & 1;
        cudaError_t e = cudaMemcpyAsync(&G->h_done[slot], &G->ctrl->done, sizeof(int32_t),
                                        cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaEventRecord(G->ev[slot], st);
        int done = 0;
        if (e == cudaSuccess && pending) {
            e = cudaEventSynchronize(G->ev[slot ^ 1]);
            done = G->h_done[slot ^ 1];
        }
        pending = true;
        poll++;
        if (e != cudaSuccess) *rc = fail(GABP_ECUDA, "poll: %s", cudaGetErrorString(e));
        return done;
    }
};

// Plans the one-launch cluster solve of a small graph once per graph (small.cu): the row
// offsets come to the host (<= 64 KB) and the cluster's row blocks are cut there.
bool small_graph(gabp_graph *G) {
    if (G->small_state == 0) {
        G->small_state = -1;
        if (gabp::small_candidate(G->g.n, G->g.E)) {
            std::vector<uint32_t> rp((size_t)G->g.n + 1);
            if (cudaMemcpyAsync(rp.data(), G->g.row_ptr, sizeof(uint32_t) * rp.size(),
                                cudaMemcpyDeviceToHost, G->stream) == cudaSuccess &&
                cudaStreamSynchronize(G->stream) == cudaSuccess &&
                gabp::small_plan(G->g.n, rp.data(), &G->small_part))
                G->small_state = 1;
        }
    }
    return G->small_state > 0;
}

int finish_loop(gabp_graph *G, double *device_ms) {
    cudaStream_t st = G->stream;
    CK(cudaEventRecord(G->ev[3], st));
    CK(cudaMemcpyAsync(G->h_ctrl, G->ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (device_ms) {  // (partitions other than rank 0 never record the start event)
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, G->ev[2], G->ev[3]));
        *device_ms = ms;
    }
    if (!G->h_ctrl->done)
        return fail(GABP_ECUDA, "solve loop ended without a decision (internal error)");
    if (host_timing())
        fprintf(stderr, "[gabp] solve: %lld sweeps, %lld launched, %d residual probes\n",
                (long long)G->h_ctrl->iterations, (long long)(G->h_ctrl->next_sweep - 1),
                (int)G->h_ctrl->probes);
    return GABP_OK;
}

constexpr int kReserveSms = 2;  // SMs the interior part leaves to the exchange kernels

int dist_ensure_comm(DistState *D) {
    if (D->xstream) return GABP_OK;
    CK(cudaStreamCreateWithFlags(&D->xstream, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&D->ev_bnd, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&D->ev_sweep, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&D->ev_done, cudaEventDisableTiming));
    return GABP_OK;
}

// Split sweep of a multi-rank slice-path launch: the leading bnd_groups groups hold every
// row a peer needs.  Worth it when they are a minority (structured partitions); for a
// random graph nearly every row is a boundary row and the sweep stays whole.
int64_t split_slices_local(const gabp_graph *G) {
    const DeviceGraph &g = G->g;
    if (g.nslices == 0 || g.slice_variant == 1 || g.bnd_groups <= 0) return 0;
    const int64_t ng = g.nslices / 15;  // (kGroup; the split is at whole groups)
    if (2 * g.bnd_groups > ng) return 0;
    return g.bnd_groups * 15;
}

// the split of this rank's sweep under the agreed protocol (0: whole sweeps on every rank)
int64_t split_slices(const gabp_graph *G) {
    if (G->dist && G->dist->use_split == 0) return 0;
    if (G->dist && G->dist->use_slices == 0) return 0;
    return split_slices_local(G);
}

// Signature of a rank's diagonal layout (0: none): ranks run it together only when every
// rank has the same diagonals.
int64_t dia_signature(const gabp_graph *G) {
    const DeviceGraph &g = G->g;
    if (g.dia_D <= 0 || getenv("GABP_NO_DIST_DIA")) return 0;
    uint64_t h = 1469598103934665603ull ^ (uint64_t)g.dia_D;
    for (int k = 0; k < g.dia_D; ++k) h = (h ^ (uint64_t)g.dia_off.v[k]) * 1099511628211ull;
    h ^= g.dia_mask ? 0x5bd1e995ull : 0ull;  // (the same kernel specialization too)
    return (int64_t)(h & 0x3fffffffffffffffull) | 1;
}

// What this rank's layout allows: bit 0 the slice layout, bit 1 the split sweep.
int dist_local_caps(const gabp_graph *G) {
    const int sl = G->g.nslices > 0 ? 1 : 0;
    const bool nosplit = getenv("GABP_NO_SPLIT") != nullptr;  // (A/B: whole sweeps)
    return sl | ((sl && !nosplit && split_slices_local(G) > 0) ? 2 : 0);
}

// Fixes the agreed protocol (caps = the AND over the ranks of dist_local_caps; dia = every
// rank has the same diagonal layout) and maps the halo lists into position numbering when
// the slice path runs.  The diagonal layout runs on local row numbering: to the peer above a
// rank sends its boundary rows' incoming messages on the positive diagonals (the peer's rows
// read them as twins), to the peer below those on the negative ones.
int dist_agree(gabp_graph *G, int caps, bool dia) {
    DistState *D = G->dist;
    D->use_slices = caps & 1;
    D->use_split = (caps & 2) ? 1 : 0;
    D->use_dia = dia ? 1 : 0;
    if (dia) {
        const DeviceGraph &g = G->g;
        D->dsend.assign(D->peers.size(), gabp::DiaHalo{});
        D->drecv.assign(D->peers.size(), gabp::DiaHalo{});
        for (size_t q = 0; q < D->peers.size(); ++q) {
            const bool up = D->peers[q] > D->rank;
            for (int k = 0; k < g.dia_D; ++k) {
                const bool pos = g.dia_off.v[k] > 0;
                gabp::DiaHalo &s = D->dsend[q], &r = D->drecv[q];
                if (pos == up) s.diag[s.nd++] = k;
                else r.diag[r.nd++] = k;
            }
        }
        D->dia_w = 2 + g.dia_D;  // {P, x} + 2 x (D / 2) message doubles
        int64_t ns = 0, nr = 0;
        for (size_t q = 0; q < D->peers.size(); ++q) {
            ns += (D->scount[q] + 1) & ~1ll;
            nr += (D->rcount[q] + 1) & ~1ll;
        }
        CK(cudaMalloc(&D->d_dsbuf, sizeof(double) * D->dia_w * (ns > 0 ? ns : 1)));
        CK(cudaMalloc(&D->d_drbuf, sizeof(double) * D->dia_w * (nr > 0 ? nr : 1)));
        return GABP_OK;  // (halo lists stay in row numbering)
    }
    if (D->use_slices) {
        int64_t ns = 0, nr = 0;
        for (size_t q = 0; q < D->peers.size(); ++q) {
            ns += (D->scount[q] + 1) & ~1ll;
            nr += (D->rcount[q] + 1) & ~1ll;
        }
        CK(gabp::slice_map_index(G->g, D->d_sidx, ns, G->stream));
        CK(gabp::slice_map_index(G->g, D->d_ridx, nr, G->stream));
        CK(cudaStreamSynchronize(G->stream));
    }
    return GABP_OK;
}

// Launches of one split sweep: boundary part (exact) on st, then the interior part (fast +
// twin) on st; the halo of the boundary part moves on the comm stream meanwhile (pack,
// grouped send/recv, unpack), and the statistics are reduced and the decision taken after
// both.  The next launch waits for all of it.
int dist_launch_split(gabp_graph *G, const SweepArgs &a, int64_t nbs, cudaStream_t st,
                      cudaStream_t cs) {
    DistState *D = G->dist;
    SweepArgs b = a;
    b.sl_lo = 0;
    b.sl_hi = nbs;
    int64_t gb = 0;
    CK(gabp::launch_slice_boundary(b, &gb, st));
    CK(cudaEventRecord(D->ev_bnd, st));
    SweepArgs in = a;
    in.sl_lo = nbs;
    in.part_base = gb;
    CK(gabp::launch_slice_part(in, kReserveSms, st));
    CK(cudaEventRecord(D->ev_sweep, st));
    // exchange of the boundary rows' new states, under the interior part
    CK(cudaStreamWaitEvent(cs, D->ev_bnd, 0));
    for (size_t q = 0; q < D->peers.size(); ++q)
        CK(gabp::launch_halo_pack(a, D->d_sidx + D->soff[q], D->scount[q],
                                  D->d_sbuf + 4 * D->soff[q], cs, 1));
    if (D->comm_nccl) {
        NK(g_nccl.groupStart());
        for (size_t q = 0; q < D->peers.size(); ++q) {
            if (D->scount[q])
                NK(g_nccl.send(D->d_sbuf + 4 * D->soff[q], 4 * D->scount[q], ncclFloat64,
                               D->peers[q], D->comm, cs));
            if (D->rcount[q])
                NK(g_nccl.recv(D->d_rbuf + 4 * D->roff[q], 4 * D->rcount[q], ncclFloat64,
                               D->peers[q], D->comm, cs));
        }
        NK(g_nccl.groupEnd());
    }
    return GABP_OK;
}

int dist_finish_split(gabp_graph *G, const SweepArgs &a, cudaStream_t st, cudaStream_t cs) {
    DistState *D = G->dist;
    for (size_t q = 0; q < D->peers.size(); ++q)
        CK(gabp::launch_halo_unpack(a, D->d_ridx + D->roff[q], D->rcount[q],
                                    D->d_rbuf + 4 * D->roff[q], cs, 1));
    CK(cudaStreamWaitEvent(cs, D->ev_sweep, 0));
    if (D->world > 1 && D->comm_nccl) {  // (one group: one NCCL launch)
        NK(g_nccl.groupStart());
        NK(g_nccl.allReduce(D->d_stats, D->d_stats, 5, ncclFloat64, ncclMax, D->comm, cs));
        NK(g_nccl.allReduce(D->d_stats + 5, D->d_stats + 5, 1, ncclFloat64, ncclSum, D->comm,
                            cs));
        NK(g_nccl.groupEnd());
    }
    CK(gabp::launch_finish(a, cs));
    CK(cudaEventRecord(D->ev_done, cs));
    CK(cudaStreamWaitEvent(st, D->ev_done, 0));
    return GABP_OK;
}

// One multi-rank launch on this rank, NCCL transport: sweep, all-reduce of the launch's
// statistics, decision, halo exchange of the node aggregates and marginals.
int dist_launch_nccl(gabp_graph *G, const SweepArgs &a, cudaStream_t st) {
    DistState *D0 = G->dist;
    if (const int64_t nbs = split_slices(G)) {
        D0->split_launches++;
        int rc = dist_ensure_comm(D0);
        if (rc) return rc;
        rc = dist_launch_split(G, a, nbs, st, D0->xstream);
        if (rc) return rc;
        return dist_finish_split(G, a, st, D0->xstream);
    }
    DistState *D = G->dist;
    CK(gabp::launch_sweep(a, GABP_SCHED_BROADCAST, gabp::kModeSolve, dist_gather(G), st));
    // the halo is packed straight after the sweep (before the decision: pre_finish), so the
    // statistics all-reduce and the halo send/recv go out as one NCCL group and the
    // all-reduce's latency hides under the exchange; the decision and the unpack follow
    for (size_t q = 0; q < D->peers.size(); ++q)
        CK(gabp::launch_halo_pack(a, D->d_sidx + D->soff[q], D->scount[q],
                                  D->d_sbuf + 4 * D->soff[q], st, 1));
    if (D->world <= 1 || D->peers.empty()) {
        if (D->world > 1) {
            NK(g_nccl.groupStart());
            NK(g_nccl.allReduce(D->d_stats, D->d_stats, 5, ncclFloat64, ncclMax, D->comm, st));
            NK(g_nccl.allReduce(D->d_stats + 5, D->d_stats + 5, 1, ncclFloat64, ncclSum,
                                D->comm, st));
            NK(g_nccl.groupEnd());
        }
        CK(gabp::launch_finish(a, st));
        return GABP_OK;
    }
    NK(g_nccl.groupStart());
    NK(g_nccl.allReduce(D->d_stats, D->d_stats, 5, ncclFloat64, ncclMax, D->comm, st));
    NK(g_nccl.allReduce(D->d_stats + 5, D->d_stats + 5, 1, ncclFloat64, ncclSum, D->comm, st));
    for (size_t q = 0; q < D->peers.size(); ++q) {
        if (D->scount[q])
            NK(g_nccl.send(D->d_sbuf + 4 * D->soff[q], 4 * D->scount[q], ncclFloat64,
                           D->peers[q], D->comm, st));
        if (D->rcount[q])
            NK(g_nccl.recv(D->d_rbuf + 4 * D->roff[q], 4 * D->rcount[q], ncclFloat64,
                           D->peers[q], D->comm, st));
    }
    NK(g_nccl.groupEnd());
    CK(gabp::launch_finish(a, st));
    for (size_t q = 0; q < D->peers.size(); ++q)
        CK(gabp::launch_halo_unpack(a, D->d_ridx + D->roff[q], D->rcount[q],
                                    D->d_rbuf + 4 * D->roff[q], st, 0));
    return GABP_OK;
}

// ---- diagonal layout across ranks --------------------------------------------------------
int dia_pack_all(gabp_graph *G, const SweepArgs &a, int64_t s_fix, int post, cudaStream_t st) {
    DistState *D = G->dist;
    for (size_t q = 0; q < D->peers.size(); ++q)
        CK(gabp::launch_dia_pack(a, D->d_sidx + D->soff[q], D->scount[q],
                                 D->d_dsbuf + D->dia_w * D->soff[q], D->dsend[q], s_fix, post,
                                 st));
    return GABP_OK;
}
int dia_unpack_all(gabp_graph *G, const SweepArgs &a, int64_t s_fix, int post,
                   cudaStream_t st) {
    DistState *D = G->dist;
    for (size_t q = 0; q < D->peers.size(); ++q)
        CK(gabp::launch_dia_unpack(a, D->d_ridx + D->roff[q], D->rcount[q],
                                   D->d_drbuf + D->dia_w * D->roff[q], D->drecv[q], s_fix,
                                   post, st));
    return GABP_OK;
}
// the halo's point-to-point part, inside an open NCCL group
int dia_p2p(gabp_graph *G, cudaStream_t st) {
    DistState *D = G->dist;
    for (size_t q = 0; q < D->peers.size(); ++q) {
        if (D->scount[q])
            NK(g_nccl.send(D->d_dsbuf + D->dia_w * D->soff[q], D->dia_w * D->scount[q],
                           ncclFloat64, D->peers[q], D->comm, st));
        if (D->rcount[q])
            NK(g_nccl.recv(D->d_drbuf + D->dia_w * D->roff[q], D->dia_w * D->rcount[q],
                           ncclFloat64, D->peers[q], D->comm, st));
    }
    return GABP_OK;
}
// S_0's aggregates of the owned rows, then the halo rows' from the peers (their local
// priors are placeholders)
int dia_start_nccl(gabp_graph *G, const SweepArgs &a, cudaStream_t st) {
    DistState *D = G->dist;
    CK(gabp::launch_dia_init(a, st));
    int rc = dia_pack_all(G, a, 0, 0, st);
    if (rc) return rc;
    if (D->world > 1 && !D->peers.empty()) {
        NK(g_nccl.groupStart());
        rc = dia_p2p(G, st);
        if (rc) return rc;
        NK(g_nccl.groupEnd());
    }
    return dia_unpack_all(G, a, 0, 0, st);
}
// One launch: the sweep (its last CTA publishes the rank's statistics of sweep s-1), the
// halo of S_s packed at once, then one NCCL group with the statistics all-reduce and the
// point-to-point halo, the decision, the unpack.
int dia_launch_nccl(gabp_graph *G, const SweepArgs &a, cudaStream_t st) {
    DistState *D = G->dist;
    CK(gabp::launch_dia_sweep(a, st));
    int rc = dia_pack_all(G, a, -1, 0, st);
    if (rc) return rc;
    if (D->world > 1) {
        NK(g_nccl.groupStart());
        NK(g_nccl.allReduce(D->d_stats, D->d_stats, 5, ncclFloat64, ncclMax, D->comm, st));
        NK(g_nccl.allReduce(D->d_stats + 5, D->d_stats + 5, 1, ncclFloat64, ncclSum, D->comm,
                            st));
        rc = dia_p2p(G, st);
        if (rc) return rc;
        NK(g_nccl.groupEnd());
    }
    CK(gabp::launch_dia_finish(a, st));
    return dia_unpack_all(G, a, -1, 1, st);
}

SweepArgs make_dist_args(gabp_graph *G) {
    SweepArgs a = make_args(G);
    a.dist = 1;
    a.dstats = G->dist->d_stats;
    a.msg_lag = dist_gather(G) == gabp::kGatherSlice ? 1 : 0;
    a.slice_path = a.msg_lag;
    if (G->dist->use_dia) a.msg_lag = a.slice_path = 0;
    return a;
}

// Runs the device-driven loop; on return G->h_ctrl holds the final controller.
int run_solve(gabp_graph *G, const gabp_options_t *opt, double *device_ms) {
    const double t_setup = host_ms();
    int rc = solve_setup(G, opt);
    if (rc) return rc;
    G->kernels_launched = 0;
    G->bins_used = 0;
    cudaStream_t st = G->stream;
    // max_iter + 2 sweep launches, plus at most one residual-only launch per sweep (slice
    // path, probe_next) -- the loop normally stops on the polled done flag long before
    const int64_t total = 2 * opt->max_iter + 4;
    int64_t launched = 0;
    Poller P{G};
    if (G->dist) {
        if (G->dist->local)
            return fail(GABP_EINVAL, "in-process partition: use gabp_dist_solve_local");
        if (opt->schedule != GABP_SCHED_BROADCAST)
            return fail(GABP_EINVAL, "the multi-rank solve runs the broadcast schedule");
        SweepArgs a = make_dist_args(G);
        G->slice_order = !G->dist->use_dia && dist_gather(G) == gabp::kGatherSlice;
        const int C = opt->sweeps_per_poll > 0 ? opt->sweeps_per_poll : auto_chunk(G);
        CK(cudaEventRecord(G->ev[2], st));
        if (G->dist->use_dia) {
            rc = dia_start_nccl(G, a, st);
            if (rc) return rc;
        }
        while (launched < total) {
            const int64_t k = total - launched < C ? total - launched : C;
            for (int64_t q = 0; q < k; ++q) {
                rc = G->dist->use_dia ? dia_launch_nccl(G, a, st) : dist_launch_nccl(G, a, st);
                if (rc) return rc;
            }
            launched += k;
            if (P.after_chunk(st, &rc)) break;
            if (rc) return rc;
        }
        return finish_loop(G, device_ms);
    }
    const int sched = opt->schedule;
    if (G->is_dense && sched == GABP_SCHED_BROADCAST && opt->gather_mode == GABP_GATHER_AUTO) {
        // dense variant: column walk + edge tiles (dense.cu), same controller protocol
        G->slice_order = false;
        const int64_t K = G->K, Kp = G->Kp;
        for (int b = 0; b < 3; ++b)
            if (!G->dmsg[b]) CK(cudaMalloc(&G->dmsg[b], sizeof(double2) * Kp * Kp));
        if (!G->dnode) {
            CK(cudaMalloc(&G->dnode, sizeof(double2) * Kp));
            CK(cudaMemset(G->dnode, 0, sizeof(double2) * Kp));  // padding rows stay zero
        }
        // S_0: +0 messages on the edges, (-0, +0) on the non-edges (dense.cu: adding them is
        // the exact identity, so the column walk needs no edge test)
        CK(gabp::launch_dense_init(G->demask, Kp, G->dmsg[0], st));
        G->kernels_launched = 0;
        gabp::DenseArgs d{};
        d.K = K;
        d.ld = Kp;
        d.A = G->dA;
        for (int b = 0; b < 3; ++b) d.msg[b] = G->dmsg[b];
        d.node = G->dnode;
        d.pairs = G->dpairs;
        d.emask = G->demask;

        d.npairs = G->dnpairs;
        SweepArgs a = make_args(G);
        const int C = opt->sweeps_per_poll > 0 ? opt->sweeps_per_poll : 8;
        if (!getenv("GABP_DENSE_TWO_KERNELS")) {
            // one fused kernel per sweep (dense.cu: dense_fused_kernel), decision of sweep
            // s-1 in launch s like the diagonal layout
            CK(gabp::launch_dense_fused_init(a, d, st));
            const int64_t dtotal = opt->max_iter + 2;
            G->kernels_launched = 1;
            CK(cudaEventRecord(G->ev[2], st));
            while (launched < dtotal) {
                const int64_t k = dtotal - launched < C ? dtotal - launched : C;
                for (int64_t q = 0; q < k; ++q) CK(gabp::launch_dense_fused_sweep(a, d, st));
                launched += k;
                G->kernels_launched += k;
                if (P.after_chunk(st, &rc)) break;
                if (rc) return rc;
            }
            return finish_loop(G, device_ms);
        }
        CK(cudaEventRecord(G->ev[2], st));
        while (launched < total) {
            const int64_t k = total - launched < C ? total - launched : C;
            for (int64_t q = 0; q < k; ++q) CK(gabp::launch_dense_sweep(a, d, st));
            launched += k;
            G->kernels_launched += 2 * k;  // column walk + pair tiles
            if (P.after_chunk(st, &rc)) break;
            if (rc) return rc;
        }
        return finish_loop(G, device_ms);
    }
    if ((sched == GABP_SCHED_BROADCAST || sched == GABP_SCHED_PARALLEL) &&
        opt->gather_mode == GABP_GATHER_AUTO && !G->dist &&
        G->g.row_lo == 0 && G->g.row_hi == G->g.n && small_graph(G) &&
        !getenv("GABP_NO_SMALL")) {
        // small graph: the whole solve loop in one launch of one thread-block cluster
        // (small.cu) -- sweeps of a few thousand edges are bound by launch and decision
        // latency, not by HBM
        SweepArgs a = make_args(G);
        G->slice_order = false;
        G->kernels_launched = 1;
        CK(cudaEventRecord(G->ev[2], st));
        CK(gabp::launch_small_solve(a, G->small_part, sched == GABP_SCHED_PARALLEL, st));
        return finish_loop(G, device_ms);
    }
    if (sched == GABP_SCHED_BROADCAST && opt->gather_mode == GABP_GATHER_AUTO &&
        G->g.dia_D > 0) {
        // stencil graph: the diagonal layout (dia.cu), one launch per sweep, decision of
        // sweep s-1 at the end of launch s
        SweepArgs a = make_args(G);
        G->slice_order = false;
        CK(gabp::launch_dia_init(a, st));
        const int C = opt->sweeps_per_poll > 0 ? opt->sweeps_per_poll : auto_chunk(G);
        const int64_t dtotal = opt->max_iter + 2;
        G->kernels_launched = 1;
        CK(cudaEventRecord(G->ev[2], st));
        while (launched < dtotal) {
            const int64_t k = dtotal - launched < C ? dtotal - launched : C;
            for (int64_t q = 0; q < k; ++q) CK(gabp::launch_dia_sweep(a, st));
            G->kernels_launched += k;
            launched += k;
            if (P.after_chunk(st, &rc)) break;
            if (rc) return rc;
        }
        return finish_loop(G, device_ms);
    }
    if (sched == GABP_SCHED_PARALLEL && opt->gather_mode == GABP_GATHER_AUTO &&
        G->g.dia_D > 0 && G->g.row_lo == 0 && G->g.row_hi == G->g.n &&
        !getenv("GABP_NO_DIA_PAR")) {
        // stencil graph, the reference's default schedule: exclusion sums over the row's own
        // slots, outgoing messages into the neighbours' shifted slots (dia.cu)
        SweepArgs a = make_args(G);
        G->slice_order = false;
        const int C = opt->sweeps_per_poll > 0 ? opt->sweeps_per_poll : auto_chunk(G);
        const int64_t ptotal = opt->max_iter + 2;
        G->kernels_launched = 0;
        CK(cudaEventRecord(G->ev[2], st));
        while (launched < ptotal) {
            const int64_t k = ptotal - launched < C ? ptotal - launched : C;
            for (int64_t q = 0; q < k; ++q) CK(gabp::launch_dia_par_sweep(a, st));
            G->kernels_launched += k;
            launched += k;
            if (P.after_chunk(st, &rc)) break;
            if (rc) return rc;
        }
        return finish_loop(G, device_ms);
    }
    rc = check_slice(G, opt);
    if (rc) return rc;
    const int gather = pick_gather(G, opt);
    if (gather == gabp::kGatherSliceParallel && !G->g.stwin) {
        rc = gabp::build_stwin(G->g, st, g_err, sizeof(g_err));
        if (rc) return rc;
        G->ws_gen++;  // captured sweeps hold the slot pointers
    }
    if (gather == gabp::kGatherRowParallel && G->g.bins == 0 && !G->dist) {
        // four rows per warp: messages in binned order when they exceed L2 (build_bins)
        rc = gabp::build_bins(G->g, st, g_err, sizeof(g_err));
        if (rc) return rc;
        G->ws_gen++;  // captured sweeps hold the index pointers
    }
    G->slice_order = gather == gabp::kGatherSlice || gather == gabp::kGatherSliceParallel;
    {
        const SweepArgs ab = make_args(G);
        G->bins_used = gather == gabp::kGatherRowParallel && ab.gout && !getenv("GABP_ROW_NO_QUAD")
                           ? G->g.bins
                           : 0;
    }
    const int C = opt->sweeps_per_poll > 0 ? opt->sweeps_per_poll : auto_chunk(G);
    // The chunks run as one CUDA graph each (one host call per chunk).  Capturing and
    // instantiating it costs ~0.2 ms, which a short solve on a fresh graph (the one-shot
    // gabp_solve_system) never earns back: its first sweeps are launched directly and the
    // chunk graph is built only if the solve is still running after them.
    constexpr int64_t kDirectSweeps = 16;
    const double tc0 = host_ms();
    bool have_exec = chunk_exec_ready(G, sched, gather, C);
    if (host_timing())
        fprintf(stderr, "[gabp] run_solve: setup %.2f ms, chunk graph (%d sweeps) %s\n",
                tc0 - t_setup, C, have_exec ? "cached" : "deferred");
    SweepArgs a = make_args(G);
    // kernels per sweep launch: the fast kernel (exact twins, host- or tail-launched, count
    // themselves on the device: Ctrl.twin_launches)
    const int kps = 1;
    G->kernels_launched = 0;
    CK(cudaEventRecord(G->ev[2], st));
    while (launched < total) {
        const int64_t k = total - launched < C ? total - launched : C;
        G->kernels_launched += kps * k;
        if (k == C && !have_exec && launched >= kDirectSweeps) {
            rc = get_chunk_exec(G, sched, gather, C);
            if (rc) return rc;
            have_exec = true;
        }
        if (k == C && have_exec) {
            CK(cudaGraphLaunch(G->chunk_exec, st));
        } else {
            for (int64_t q = 0; q < k; ++q)
                CK(gabp::launch_sweep(a, sched, gabp::kModeSolve, gather, st));
        }
        launched += k;
        if (P.after_chunk(st, &rc)) break;
        if (rc) return rc;
    }
    return finish_loop(G, device_ms);
}

void fill_report(gabp_graph *G, const gabp_options_t *opt, double ms, double rsq_last,
                 gabp_report_t *rep) {
    if (!rep) return;
    const Ctrl &c = *G->h_ctrl;
    rep->converged = c.converged;
    rep->diverged = c.diverged;
    rep->iterations = c.iterations;
    rep->n_hist = c.n_hist;
    rep->sweeps_launched = c.next_sweep - 1;
    rep->messages_sent =
        c.iterations * (opt->schedule == GABP_SCHED_BROADCAST ? G->g.n : G->g.E);
    rep->device_ms = ms;
    rep->residual_probes = c.probes;
    rep->kernel_launches = G->kernels_launched + c.twin_launches;
    rep->split_sweeps = G->dist ? G->dist->split_launches : 0;
    rep->dist_layout = !G->dist ? 0 : G->dist->use_dia ? 3 : G->dist->use_slices ? 1 : 2;
    rep->message_bins = G->bins_used;
    rep->final_rel_residual =
        (c.n_hist >= 1 && G->g.rhs_norm > 0.0) ? sqrt(rsq_last) / G->g.rhs_norm : NAN;
}

// ---- packed index upload (gabp_graph_create_ex) -----------------------------------------
// The pair indices are two thirds of a system's bytes as int64 (config 1: 268 of 420 MB over
// PCIe).  For n < 2^32 the host packs them to 32 bits chunk by chunk (OpenMP threads) into a
// cached pinned buffer while the previous chunk and the values are on the wire, and the
// device widens them again -- half the index bytes cross the link.
__global__ void widen_u32_kernel(int64_t cnt, const uint32_t *in, int64_t *out) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < cnt;
         k += (int64_t)gridDim.x * blockDim.x)
        out[k] = (int64_t)in[k];
}

std::mutex g_pack_mu;
uint32_t *g_pack_buf = nullptr;  // pinned, 2 x g_pack_cap entries
int64_t g_pack_cap = 0;

// packs [lo, hi) of both index arrays; false when a value does not fit 32 bits (the plain
// int64 path then lets the device validation report it as the reference does)
bool pack_chunk(const int64_t *pi, const int64_t *pj, int64_t lo, int64_t hi, uint32_t *oi,
                uint32_t *oj) {
    int bad = 0;
#pragma omp parallel for schedule(static) reduction(| : bad)
    for (int64_t k = lo; k < hi; ++k) {
        const int64_t a = pi[k], b = pj[k];
        bad |= ((uint64_t)a > 0xffffffffull) | ((uint64_t)b > 0xffffffffull);
        oi[k] = (uint32_t)a;
        oj[k] = (uint32_t)b;
    }
    return bad == 0;
}

gabp_graph *new_graph(int device, int *rc) {
    gabp_graph *G = new gabp_graph();
    G->device = device;
    cudaError_t e = cudaSetDevice(device);
    if (e == cudaSuccess) e = gabp::prepare_sweep_kernels();
    if (e == cudaSuccess) e = gabp::prepare_rowpar_kernels();
    if (e == cudaSuccess) e = gabp::prepare_slice_kernels();
    if (e == cudaSuccess) e = gabp::prepare_dia_kernels();
    if (e == cudaSuccess) {
        // keep freed blocks in the device pool (graphs, workspaces and build scratch are
        // stream-ordered allocations): no re-mapping on the next build or solve
        cudaMemPool_t pool;
        e = cudaDeviceGetDefaultMemPool(&pool, device);
        uint64_t keep = UINT64_MAX;
        if (e == cudaSuccess)
            e = cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&G->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
        *rc = fail(GABP_ECUDA, "device %d: %s", device, cudaGetErrorString(e));
        delete G;
        return nullptr;
    }
    *rc = GABP_OK;
    return G;
}

}  // namespace

extern "C" {

const char *gabp_last_error(void) { return g_err; }

int gabp_version(void) { return 10000; }

int gabp_device_count(int32_t *count) {
    int c = 0;
    cudaError_t e = cudaGetDeviceCount(&c);
    if (e != cudaSuccess) {
        *count = 0;
        return fail(GABP_ECUDA, "cudaGetDeviceCount: %s", cudaGetErrorString(e));
    }
    *count = c;
    return GABP_OK;
}

static int create_device_range(int64_t n, int64_t npairs, const double *d_diag,
                               const double *d_rhs, const int64_t *d_pair_i,
                               const int64_t *d_pair_j, const double *d_pair_v, int64_t row_lo,
                               int64_t row_hi, int32_t device, gabp_graph_t **out,
                               cudaEvent_t idx_ready = nullptr,
                               cudaEvent_t val_ready = nullptr) {
    if (!out) return fail(GABP_EINVAL, "out must not be NULL");
    *out = nullptr;
    int rc;
    gabp_graph *G = new_graph(device, &rc);
    if (!G) return rc;
    rc = gabp::build_graph_device(G->g, n, npairs, d_diag, d_rhs, d_pair_i, d_pair_j, d_pair_v,
                                  row_lo, row_hi, G->stream, g_err, sizeof(g_err), idx_ready,
                                  val_ready);
    if (rc == GABP_ENOMEM) {  // the cached spares of earlier graphs back to the device, once
        cudaStreamSynchronize(G->stream);
        gabp::free_graph(G->g, G->stream);
        cudaStreamSynchronize(G->stream);
        cudaGetLastError();
        release_spares(device);
        rc = gabp::build_graph_device(G->g, n, npairs, d_diag, d_rhs, d_pair_i, d_pair_j,
                                      d_pair_v, row_lo, row_hi, G->stream, g_err,
                                      sizeof(g_err), idx_ready, val_ready);
    }
    if (rc != GABP_OK) {
        cudaStreamSynchronize(G->stream);
        gabp::free_graph(G->g, G->stream);
        cudaStreamSynchronize(G->stream);
        cudaStreamDestroy(G->stream);
        delete G;
        return rc;
    }
    *out = G;
    return GABP_OK;
}

int gabp_release_cached(int32_t device) {
    int count = 0;
    CK(cudaGetDeviceCount(&count));
    if (device < 0 || device >= count) return fail(GABP_EINVAL, "no device %d", device);
    release_spares(device);
    return GABP_OK;
}

int gabp_graph_create_device(int64_t n, int64_t npairs, const double *d_diag,
                             const double *d_rhs, const int64_t *d_pair_i,
                             const int64_t *d_pair_j, const double *d_pair_v, int32_t device,
                             gabp_graph_t **out) {
    return create_device_range(n, npairs, d_diag, d_rhs, d_pair_i, d_pair_j, d_pair_v, 0, n,
                               device, out);
}

int gabp_graph_create_device_ex(int64_t n, int64_t npairs, const double *d_diag,
                                const double *d_rhs, const int64_t *d_pair_i,
                                const int64_t *d_pair_j, const double *d_pair_v,
                                int64_t row_lo, int64_t row_hi, int32_t device,
                                gabp_graph_t **out) {
    if (row_lo < 0 || row_hi > n || row_lo >= row_hi)
        return fail(GABP_EINVAL, "swept rows [%lld, %lld) outside [0, %lld)", (long long)row_lo,
                    (long long)row_hi, (long long)n);
    return create_device_range(n, npairs, d_diag, d_rhs, d_pair_i, d_pair_j, d_pair_v, row_lo,
                               row_hi, device, out);
}

int gabp_graph_create(int64_t n, int64_t npairs, const double *h_diag, const double *h_rhs,
                      const int64_t *h_pair_i, const int64_t *h_pair_j, const double *h_pair_v,
                      int32_t device, gabp_graph_t **out) {
    return gabp_graph_create_ex(n, npairs, h_diag, h_rhs, h_pair_i, h_pair_j, h_pair_v, 0, n,
                                device, out);
}

int gabp_graph_create_ex(int64_t n, int64_t npairs, const double *h_diag, const double *h_rhs,
                         const int64_t *h_pair_i, const int64_t *h_pair_j,
                         const double *h_pair_v, int64_t row_lo, int64_t row_hi,
                         int32_t device, gabp_graph_t **out) {
    if (!out) return fail(GABP_EINVAL, "out must not be NULL");
    *out = nullptr;
    if (n < 1) return fail(GABP_EINVAL, "diag must be a non-empty vector");
    if (npairs < 0) return fail(GABP_EINVAL, "negative pair count");
    const double t_start = host_ms();
    CK(cudaSetDevice(device));
    // Two copy streams: the pair indices first (the structural passes of the build -- degree
    // count, scan, scatter, row sort -- need only them), the values and node vectors
    // behind them on a second stream; the build waits on their events.
    cudaStream_t st, sv;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&sv, cudaStreamNonBlocking));
    cudaEvent_t ev_buf, ev_idx, ev_val;
    CK(cudaEventCreateWithFlags(&ev_buf, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ev_idx, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ev_val, cudaEventDisableTiming));
    const size_t nb = sizeof(double) * n, pb = sizeof(int64_t) * (npairs > 0 ? npairs : 1);
    // (packing runs at host memory bandwidth only with several threads: a process limited
    // to one or two -- torchrun exports OMP_NUM_THREADS=1 -- sends the int64 indices as is)
    bool pack = npairs >= (1 << 20) && n <= 0xffffffffll && omp_get_max_threads() >= 4 &&
                !getenv("GABP_NO_PACK");
    const size_t sbytes = 2 * nb + 3 * pb + (pack ? pb : 0);  // (+ two packed index arrays)
    char *buf = static_cast<char *>(spare_take(1, device, sbytes));
    cudaError_t e = buf ? cudaSuccess : cudaMallocAsync(&buf, sbytes, st);
    if (e != cudaSuccess) {
        cudaStreamDestroy(st);
        cudaStreamDestroy(sv);
        return fail(GABP_ENOMEM, "staging allocation: %s", cudaGetErrorString(e));
    }
    cudaEventRecord(ev_buf, st);
    cudaStreamWaitEvent(sv, ev_buf, 0);
    double *d_diag = (double *)buf, *d_rhs = (double *)(buf + nb);
    int64_t *d_pi = (int64_t *)(buf + 2 * nb), *d_pj = (int64_t *)(buf + 2 * nb + pb);
    double *d_pv = (double *)(buf + 2 * nb + 2 * pb);
    // values and node vectors first on their stream: the link is busy while chunk 0 packs
    // (sending the values only after the indices was measured: 0.7 ms slower per call)
    if (npairs > 0)
        cudaMemcpyAsync(d_pv, h_pair_v, sizeof(double) * npairs, cudaMemcpyHostToDevice, sv);
    cudaMemcpyAsync(d_diag, h_diag, nb, cudaMemcpyHostToDevice, sv);
    cudaMemcpyAsync(d_rhs, h_rhs, nb, cudaMemcpyHostToDevice, sv);
    double t_pack = 0.0;
    // (held to the end of the call: the pinned pack buffer is shared, and its copies have
    // left it only after the stream synchronisations below)
    std::unique_lock<std::mutex> pack_lk(g_pack_mu, std::defer_lock);
    if (pack) {
        pack_lk.lock();
        if (g_pack_cap < npairs) {
            if (g_pack_buf) cudaFreeHost(g_pack_buf);
            g_pack_buf = nullptr;
            g_pack_cap = 0;
            if (cudaHostAlloc(&g_pack_buf, sizeof(uint32_t) * 2 * (size_t)npairs,
                              cudaHostAllocPortable) == cudaSuccess)
                g_pack_cap = npairs;
            else
                cudaGetLastError();
        }
        pack = g_pack_cap >= npairs;
        if (pack) {
            uint32_t *hi32 = g_pack_buf, *hj32 = g_pack_buf + g_pack_cap;
            uint32_t *di32 = (uint32_t *)(buf + 2 * nb + 3 * pb), *dj32 = di32 + npairs;
            constexpr int kChunks = 8;
            for (int c = 0; c < kChunks && pack; ++c) {
                const int64_t lo = npairs * c / kChunks, hi = npairs * (c + 1) / kChunks;
                const double tp0 = host_ms();
                pack = pack_chunk(h_pair_i, h_pair_j, lo, hi, hi32, hj32);
                t_pack += host_ms() - tp0;
                if (!pack) break;
                cudaMemcpyAsync(di32 + lo, hi32 + lo, sizeof(uint32_t) * (hi - lo),
                                cudaMemcpyHostToDevice, st);
                cudaMemcpyAsync(dj32 + lo, hj32 + lo, sizeof(uint32_t) * (hi - lo),
                                cudaMemcpyHostToDevice, st);
                widen_u32_kernel<<<296, 256, 0, st>>>(hi - lo, di32 + lo, d_pi + lo);
                widen_u32_kernel<<<296, 256, 0, st>>>(hi - lo, dj32 + lo, d_pj + lo);
            }
        }
    }
    if (!pack && npairs > 0) {
        cudaMemcpyAsync(d_pi, h_pair_i, sizeof(int64_t) * npairs, cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(d_pj, h_pair_j, sizeof(int64_t) * npairs, cudaMemcpyHostToDevice, st);
    }
    cudaEventRecord(ev_idx, st);
    e = cudaEventRecord(ev_val, sv);
    int rc = GABP_OK;
    if (e != cudaSuccess) {
        rc = fail(GABP_ECUDA, "H2D copy: %s", cudaGetErrorString(e));
    } else {
        rc = create_device_range(n, npairs, d_diag, d_rhs, d_pi, d_pj, d_pv, row_lo, row_hi,
                                 device, out, ev_idx, ev_val);
    }
    const cudaError_t e1 = cudaStreamSynchronize(st), e2 = cudaStreamSynchronize(sv);
    if (rc == GABP_OK && (e1 != cudaSuccess || e2 != cudaSuccess))
        rc = fail(GABP_ECUDA, "H2D copy: %s", cudaGetErrorString(e1 != cudaSuccess ? e1 : e2));
    if (host_timing())
        fprintf(stderr, "[gabp] graph_create: H2D + device build %.2f ms (core %.2f on device; "
                "index packing %.2f ms on the host)\n",
                host_ms() - t_start, rc == GABP_OK ? (*out)->g.build_ms : 0.0, t_pack);
    if (!spare_keep(1, device, buf, sbytes)) {  // both streams and the build are idle
        cudaFreeAsync(buf, st);
        cudaStreamSynchronize(st);
    }
    cudaEventDestroy(ev_buf);
    cudaEventDestroy(ev_idx);
    cudaEventDestroy(ev_val);
    cudaStreamDestroy(st);
    cudaStreamDestroy(sv);
    return rc;
}

int gabp_graph_create_dense(int64_t n, const double *h_a, const double *h_rhs, int32_t device,
                            gabp_graph_t **out) {
    if (!out || !h_a || !h_rhs) return fail(GABP_EINVAL, "NULL argument");
    if (n < 1) return fail(GABP_EINVAL, "matrix must be non-empty");
    std::vector<double> diag(n);
    std::vector<int64_t> pi, pj;
    std::vector<double> pv;
    for (int64_t i = 0; i < n; ++i) {
        diag[i] = h_a[i * n + i];
        for (int64_t j = i + 1; j < n; ++j) {
            const double v = h_a[i * n + j];
            if (v != h_a[j * n + i])
                return fail(GABP_EINVAL, "matrix not symmetric at (%lld, %lld)", (long long)i,
                            (long long)j);
            if (v != 0.0) {
                pi.push_back(i);
                pj.push_back(j);
                pv.push_back(v);
            }
        }
    }
    int rc = gabp_graph_create(n, (int64_t)pv.size(), diag.data(), h_rhs, pi.data(), pj.data(),
                               pv.data(), device, out);
    if (rc != GABP_OK) return rc;
    gabp_graph *G = *out;
    G->is_dense = 1;
    G->K = n;
    G->Kp = (n + 31) / 32 * 32;  // padded rows/columns: whole 32 x 32 tiles, zero A
    const int64_t Kp = G->Kp;
    CK(cudaMalloc(&G->dA, sizeof(double) * Kp * Kp));
    CK(cudaMemset(G->dA, 0, sizeof(double) * Kp * Kp));
    CK(cudaMemcpy2D(G->dA, sizeof(double) * Kp, h_a, sizeof(double) * n, sizeof(double) * n, n,
                    cudaMemcpyHostToDevice));
    const int64_t nt = Kp / 32;
    std::vector<uint2> tp;
    tp.reserve(nt * (nt + 1) / 2);
    for (int64_t I = 0; I < nt; ++I)
        for (int64_t J = I; J < nt; ++J) tp.push_back(make_uint2((unsigned)I, (unsigned)J));
    G->dnpairs = (int64_t)tp.size();
    CK(cudaMalloc(&G->demask, sizeof(uint32_t) * Kp * (Kp / 32)));
    CK(gabp::launch_dense_mask(G->dA, Kp, G->demask, 0));
    CK(cudaDeviceSynchronize());
    CK(cudaMalloc(&G->dpairs, sizeof(uint2) * tp.size()));
    CK(cudaMemcpy(G->dpairs, tp.data(), sizeof(uint2) * tp.size(), cudaMemcpyHostToDevice));
    return GABP_OK;
}

static void graph_release(gabp_graph *G) {
    if (G->refs.fetch_sub(1) != 1) return;
    cudaSetDevice(G->device);
    cudaStreamSynchronize(G->stream);
    if (G->d_serial) cudaFree(G->d_serial);
    if (G->d_serial_lvl) cudaFree(G->d_serial_lvl);
    if (G->serial_strip) cudaFree(G->serial_strip);
    if (G->serial_exec) cudaGraphExecDestroy(G->serial_exec);
    release_workspace(G);
    gabp::free_graph(G->g, G->stream);
    cudaStreamSynchronize(G->stream);
    cudaStreamDestroy(G->stream);
    delete G;
}

void gabp_graph_destroy(gabp_graph_t *G) {
    if (!G) return;
    graph_release(G);
}

int gabp_graph_info(const gabp_graph_t *G, gabp_graph_info_t *info) {
    if (!G || !info) return fail(GABP_EINVAL, "NULL argument");
    info->n = G->g.n;
    info->num_edges = G->g.E;
    info->num_tiles = G->g.ntiles;
    info->max_degree = G->g.max_degree;
    info->device = G->device;
    info->is_dense = G->is_dense;
    info->rhs_norm = G->g.rhs_norm;
    info->build_ms = G->g.build_ms;
    info->twin_span = G->g.twin_span;
    info->num_slices = G->g.nslices;
    info->num_slots = G->g.nslots;
    info->slice_variant = G->g.slice_variant;
    info->dia_diagonals = G->g.dia_D;
    return GABP_OK;
}

int gabp_graph_export(const gabp_graph_t *G, int64_t *h_row_ptr, int64_t *h_col,
                      int64_t *h_rev, double *h_coeff) {
    if (!G) return fail(GABP_EINVAL, "NULL graph");
    CK(cudaSetDevice(G->device));
    const DeviceGraph &g = G->g;
    if (h_row_ptr) {
        std::vector<uint32_t> rp(g.n + 1);
        CK(cudaMemcpyAsync(rp.data(), g.row_ptr, sizeof(uint32_t) * (g.n + 1),
                           cudaMemcpyDeviceToHost, G->stream));
        CK(cudaStreamSynchronize(G->stream));
        for (int64_t i = 0; i <= g.n; ++i) h_row_ptr[i] = rp[i];
    }
    if ((h_col || h_rev || h_coeff) && g.E > 0) {
        std::vector<gabp::EdgeRec> er(g.E);
        CK(cudaMemcpyAsync(er.data(), g.er, sizeof(gabp::EdgeRec) * g.E, cudaMemcpyDeviceToHost,
                           G->stream));
        CK(cudaStreamSynchronize(G->stream));
        for (int64_t e = 0; e < g.E; ++e) {
            if (h_rev) h_rev[e] = er[e].rev;
            if (h_col) h_col[e] = er[e].col;
            if (h_coeff) h_coeff[e] = er[e].coeff;
        }
    }
    return GABP_OK;
}

int gabp_graph_set_rhs(gabp_graph_t *G, const double *h_rhs) {
    if (!G || !h_rhs) return fail(GABP_EINVAL, "NULL argument");
    CK(cudaSetDevice(G->device));
    CK(cudaMemcpyAsync(G->g.rhs, h_rhs, sizeof(double) * G->g.n, cudaMemcpyHostToDevice,
                       G->stream));
    return gabp::compute_priors(G->g, G->stream, g_err, sizeof(g_err));
}

void *gabp_graph_stream(const gabp_graph_t *G) { return G ? (void *)G->stream : nullptr; }

// ---- message state ---------------------------------------------------------------------

int gabp_state_create(const gabp_graph_t *G, gabp_state_t **out) {
    if (!G || !out) return fail(GABP_EINVAL, "NULL argument");
    CK(cudaSetDevice(G->device));
    gabp_state *S = new gabp_state();
    S->g = G;
    const_cast<gabp_graph *>(G)->refs.fetch_add(1);
    const int64_t E = G->g.E > 0 ? G->g.E : 1;
    for (int b = 0; b < 2; ++b) {  // (stream-ordered pool blocks: a state per sweep is cheap)
        cudaError_t e = cudaMallocAsync(&S->buf[b], sizeof(double2) * E, G->stream);
        if (e != cudaSuccess) {
            if (S->buf[0]) cudaFreeAsync(S->buf[0], G->stream);
            graph_release(const_cast<gabp_graph *>(G));
            delete S;
            return fail(GABP_ENOMEM, "state allocation: %s", cudaGetErrorString(e));
        }
    }
    *out = S;
    return gabp_state_reset(S);
}

int gabp_state_clone(const gabp_state_t *S, gabp_state_t **out) {
    if (!S || !out) return fail(GABP_EINVAL, "NULL argument");
    int rc = gabp_state_create(S->g, out);
    if (rc) return rc;
    gabp_state *D = *out;
    const int64_t E = S->g->g.E > 0 ? S->g->g.E : 1;
    CK(cudaMemcpyAsync(D->buf[0], S->buf[S->cur], sizeof(double2) * E, cudaMemcpyDeviceToDevice,
                       S->g->stream));
    CK(cudaStreamSynchronize(S->g->stream));
    D->cur = 0;
    D->iteration = S->iteration;
    D->messages_sent = S->messages_sent;
    return GABP_OK;
}

void gabp_state_destroy(gabp_state_t *S) {
    if (!S) return;
    cudaSetDevice(S->g->device);
    cudaFreeAsync(S->buf[0], S->g->stream);
    cudaFreeAsync(S->buf[1], S->g->stream);
    cudaStreamSynchronize(S->g->stream);
    graph_release(const_cast<gabp_graph *>(S->g));
    delete S;
}

int gabp_state_reset(gabp_state_t *S) {
    if (!S) return fail(GABP_EINVAL, "NULL state");
    CK(cudaSetDevice(S->g->device));
    const int64_t E = S->g->g.E > 0 ? S->g->g.E : 1;
    CK(cudaMemsetAsync(S->buf[0], 0, sizeof(double2) * E, S->g->stream));
    CK(cudaStreamSynchronize(S->g->stream));
    S->cur = 0;
    S->iteration = 0;
    S->messages_sent = 0;
    return GABP_OK;
}

int gabp_state_read(const gabp_state_t *S, double *h_prec, double *h_mean) {
    if (!S) return fail(GABP_EINVAL, "NULL state");
    const int64_t E = S->g->g.E;
    if (E == 0) return GABP_OK;
    CK(cudaSetDevice(S->g->device));
    std::vector<double2> tmp(E);
    CK(cudaMemcpyAsync(tmp.data(), S->buf[S->cur], sizeof(double2) * E, cudaMemcpyDeviceToHost,
                       S->g->stream));
    CK(cudaStreamSynchronize(S->g->stream));
    for (int64_t e = 0; e < E; ++e) {
        if (h_prec) h_prec[e] = tmp[e].x;
        if (h_mean) h_mean[e] = tmp[e].y;
    }
    return GABP_OK;
}

int gabp_state_write(gabp_state_t *S, const double *h_prec, const double *h_mean) {
    if (!S || !h_prec || !h_mean) return fail(GABP_EINVAL, "NULL argument");
    const int64_t E = S->g->g.E;
    if (E == 0) return GABP_OK;
    CK(cudaSetDevice(S->g->device));
    std::vector<double2> tmp(E);
    for (int64_t e = 0; e < E; ++e) tmp[e] = make_double2(h_prec[e], h_mean[e]);
    CK(cudaMemcpyAsync(S->buf[S->cur], tmp.data(), sizeof(double2) * E, cudaMemcpyHostToDevice,
                       S->g->stream));
    CK(cudaStreamSynchronize(S->g->stream));
    return GABP_OK;
}

int gabp_state_counters(const gabp_state_t *S, int64_t *iteration, int64_t *messages_sent) {
    if (!S) return fail(GABP_EINVAL, "NULL state");
    if (iteration) *iteration = S->iteration;
    if (messages_sent) *messages_sent = S->messages_sent;
    return GABP_OK;
}

static int absmax_bits(const gabp_graph *G, const double2 *a, unsigned long long *bits) {
    unsigned long long *d = nullptr;
    CK(cudaMallocAsync(&d, sizeof(unsigned long long), G->stream));
    CK(gabp::launch_absmax(G->g.E, a, d, G->stream));
    CK(cudaMemcpyAsync(bits, d, sizeof(unsigned long long), cudaMemcpyDeviceToHost, G->stream));
    CK(cudaFreeAsync(d, G->stream));
    CK(cudaStreamSynchronize(G->stream));
    return GABP_OK;
}

// some message not finite, or the biggest |message| above blowup (solver.py:333-338)
static int state_blown(const gabp_graph *G, const double2 *m, double blowup, int32_t *blown) {
    unsigned long long bits = 0;
    int rc = absmax_bits(G, m, &bits);
    if (rc) return rc;
    const unsigned long long inf_bits = 0x7ff0000000000000ull;
    *blown = bits >= inf_bits || __builtin_bit_cast(double, bits) > blowup;
    return GABP_OK;
}


// ---- serial schedule (solver.py:176-217) ------------------------------------------------
// Dependency levels of a task sequence (the order): task t on node i goes one level above
// the last task on i or on any neighbour of i; tasks of one level touch disjoint messages
// (rowpar.cu: serial_level_kernel), so levels run in parallel and give the in-place
// sequential result exactly.  Built on the host from a copy of the CSR, cached per order.
static int serial_levels(gabp_graph *G, const int64_t *order, int64_t norder) {
    const int64_t n = G->g.n;
    const bool asc = order == nullptr;
    if (asc) norder = n;
    if (G->serial_valid && G->serial_ascending == asc &&
        (asc || ((int64_t)G->serial_order.size() == norder &&
                 memcmp(G->serial_order.data(), order, sizeof(int64_t) * norder) == 0)))
        return GABP_OK;
    for (int64_t t = 0; !asc && t < norder; ++t)
        if (order[t] < 0 || order[t] >= n)
            return fail(GABP_EINVAL, "serial order entry %lld out of range [0, %lld)",
                        (long long)order[t], (long long)n);
    if ((int64_t)G->h_rp.size() != n + 1) {
        // fetched into locals and kept only when every step succeeded: the cache key is
        // the size of h_rp, so a failed fetch must not leave a half-filled CSR behind
        std::vector<uint32_t> rp(n + 1), col(G->g.E);
        cudaError_t e = cudaMemcpyAsync(rp.data(), G->g.row_ptr, sizeof(uint32_t) * (n + 1),
                                        cudaMemcpyDeviceToHost, G->stream);
        if (e == cudaSuccess && G->g.E) {
            // the column field only (4 B per edge through PCIe, not the record), staged in
            // the library's stream-ordered pool
            uint32_t *dcol = nullptr;
            e = cudaMallocAsync(&dcol, sizeof(uint32_t) * G->g.E, G->stream);
            if (e == cudaSuccess) e = gabp::launch_edge_col(G->g.E, G->g.er, dcol, G->stream);
            if (e == cudaSuccess)
                e = cudaMemcpyAsync(col.data(), dcol, sizeof(uint32_t) * G->g.E,
                                    cudaMemcpyDeviceToHost, G->stream);
            if (dcol) cudaFreeAsync(dcol, G->stream);
        }
        if (e == cudaSuccess) e = cudaStreamSynchronize(G->stream);
        CK(e);
        G->h_rp.swap(rp);
        G->h_col.swap(col);
    }
    std::vector<uint32_t> last(n, 0u), lev(norder);
    uint32_t nlev = 0;
    for (int64_t t = 0; t < norder; ++t) {
        const int64_t i = asc ? t : order[t];
        uint32_t L = last[i];
        for (uint32_t e = G->h_rp[i]; e < G->h_rp[i + 1]; ++e) {
            const uint32_t k = G->h_col[e];
            L = last[k] > L ? last[k] : L;
        }
        lev[t] = L + 1;
        last[i] = L + 1;
        nlev = L + 1 > nlev ? L + 1 : nlev;
    }
    G->serial_lvl.assign((size_t)nlev + 1, 0);
    for (int64_t t = 0; t < norder; ++t) G->serial_lvl[lev[t]]++;
    for (uint32_t l = 1; l <= nlev; ++l) G->serial_lvl[l] += G->serial_lvl[l - 1];
    std::vector<int64_t> fill(G->serial_lvl.begin(), G->serial_lvl.end() - 1);
    std::vector<uint2> tasks(norder > 0 ? norder : 1);
    for (int64_t t = 0; t < norder; ++t) {
        const int64_t i = asc ? t : order[t];
        tasks[fill[lev[t] - 1]++] = make_uint2((uint32_t)i, (uint32_t)t);
    }
    if (G->d_serial) cudaFree(G->d_serial);
    G->d_serial = nullptr;
    if (G->serial_exec) cudaGraphExecDestroy(G->serial_exec);
    G->serial_exec = nullptr;
    CK(cudaMalloc(&G->d_serial, sizeof(uint2) * tasks.size()));
    CK(cudaMemcpy(G->d_serial, tasks.data(), sizeof(uint2) * tasks.size(),
                  cudaMemcpyHostToDevice));
    if (G->d_serial_lvl) cudaFree(G->d_serial_lvl);
    G->d_serial_lvl = nullptr;
    CK(cudaMalloc(&G->d_serial_lvl, sizeof(int64_t) * G->serial_lvl.size()));
    CK(cudaMemcpy(G->d_serial_lvl, G->serial_lvl.data(), sizeof(int64_t) * G->serial_lvl.size(),
                  cudaMemcpyHostToDevice));
    G->serial_maxw = 0;
    for (uint32_t l = 0; l < nlev; ++l) {
        const int64_t w = G->serial_lvl[l + 1] - G->serial_lvl[l];
        G->serial_maxw = w > G->serial_maxw ? w : G->serial_maxw;
    }
    G->serial_ascending = asc;
    if (asc)
        G->serial_order.clear();
    else
        G->serial_order.assign(order, order + norder);
    G->serial_valid = true;
    return GABP_OK;
}

int gabp_sweep_serial(const gabp_graph_t *Gc, gabp_state_t *S, const int64_t *order,
                      int64_t norder, double blowup, double *max_change, int32_t *out_of_range,
                      int64_t *singular_edge, int32_t *num_levels) {
    gabp_graph *G = const_cast<gabp_graph *>(Gc);
    if (!G || !S || S->g != Gc) return fail(GABP_EINVAL, "state does not belong to graph");
    if (order && norder < 0) return fail(GABP_EINVAL, "negative order length");
    if (G->g.row_lo != 0 || G->g.row_hi != G->g.n)
        return fail(GABP_EINVAL, "serial schedule needs the whole graph");
    CK(cudaSetDevice(G->device));
    int rc = ensure_workspace(G, 1);
    if (rc) return rc;
    rc = serial_levels(G, order, norder);
    if (rc) return rc;
    if (singular_edge) *singular_edge = -1;
    if (max_change) *max_change = 0.0;
    if (out_of_range) *out_of_range = 0;
    if (num_levels) *num_levels = (int32_t)(G->serial_lvl.size() - 1);
    // in place on a copy (solver.py:177-178 works on lists made from the state): a sweep
    // that meets a singular exclusion sum leaves the state as it was, like the reference
    double2 *msg = S->buf[S->cur ^ 1];
    Ctrl c = gabp::fresh_ctrl();
    c.serial_msg = msg;
    *G->h_ctrl = c;
    CK(cudaMemcpyAsync(G->ctrl, G->h_ctrl, sizeof(Ctrl), cudaMemcpyHostToDevice, G->stream));
    if (G->g.E)
        CK(cudaMemcpyAsync(msg, S->buf[S->cur], sizeof(double2) * G->g.E,
                           cudaMemcpyDeviceToDevice, G->stream));
    if (G->g.max_degree > gabp::kRowParMaxDegree && !G->serial_strip) {
        // tasks longer than the shared-memory strip: one global strip per warp
        G->serial_strip_stride = (G->g.max_degree + 7) & ~7ll;
        const int64_t warps = gabp::serial_strip_warps();
        CK(cudaMalloc(&G->serial_strip, sizeof(double2) * G->serial_strip_stride *
                                            (warps > 0 ? warps : 1)));
        if (G->serial_exec) {  // captured without the strip
            cudaGraphExecDestroy(G->serial_exec);
            G->serial_exec = nullptr;
        }
    }
    const double lim = blowup < DBL_MAX ? blowup : DBL_MAX;
    const int nlev = (int)G->serial_lvl.size() - 1;
    if (nlev <= 512 && !getenv("GABP_SERIAL_LEVEL_LAUNCHES")) {
        // few, wide levels: one cooperative launch, a grid barrier between levels
        SweepArgs a = make_args(G);
        CK(gabp::launch_serial_sweep(a, G->d_serial, G->d_serial_lvl, nlev, G->serial_maxw, lim,
                                     G->stream));
    } else {
        // many levels: the level launches as one CUDA graph (host launches cost ~7 us each),
        // captured once per order, workspace and blow-up limit
        if (G->serial_exec && (G->serial_gen != G->ws_gen || G->serial_lim != lim)) {
            cudaGraphExecDestroy(G->serial_exec);
            G->serial_exec = nullptr;
        }
        if (!G->serial_exec && G->serial_lvl.size() > 1) {
            SweepArgs a = make_args(G);
            cudaGraph_t graph;
            CK(cudaStreamBeginCapture(G->stream, cudaStreamCaptureModeThreadLocal));
            for (size_t l = 0; l + 1 < G->serial_lvl.size(); ++l) {
                cudaError_t e = gabp::launch_serial_level(a, G->d_serial + G->serial_lvl[l],
                                                          G->serial_lvl[l + 1] - G->serial_lvl[l],
                                                          lim, G->stream);
                if (e != cudaSuccess) {
                    cudaStreamEndCapture(G->stream, &graph);
                    if (graph) cudaGraphDestroy(graph);
                    return fail(GABP_ECUDA, "serial level capture: %s", cudaGetErrorString(e));
                }
            }
            CK(cudaStreamEndCapture(G->stream, &graph));
            cudaError_t e = cudaGraphInstantiate(&G->serial_exec, graph, 0);
            cudaGraphDestroy(graph);
            CK(e);
            G->serial_gen = G->ws_gen;
            G->serial_lim = lim;
        }
        if (G->serial_exec) CK(cudaGraphLaunch(G->serial_exec, G->stream));
    }
    CK(cudaMemcpyAsync(G->h_ctrl, G->ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, G->stream));
    CK(cudaStreamSynchronize(G->stream));
    const Ctrl &h = *G->h_ctrl;
    if (h.singular_min[1] != gabp::kNoIndex) {
        const int64_t e = (int64_t)(h.singular_min[1] & 0xffffffffull);
        if (singular_edge) *singular_edge = e;
        return fail(GABP_ESINGULAR, "P_excl = 0 on edge %lld", (long long)e);
    }
    S->cur ^= 1;
    S->iteration += 1;
    S->messages_sent += G->g.E;
    if (out_of_range) {  // on the final state, as the solve loop's test reads it
        int32_t blown = 0;
        rc = state_blown(G, S->buf[S->cur], blowup, &blown);
        if (rc) return rc;
        *out_of_range = blown;
    }
    if (max_change) {
        double v;
        unsigned long long bits = h.change_bits[1];
        memcpy(&v, &bits, sizeof(v));
        *max_change = v;
    }
    return GABP_OK;
}

int gabp_sweep(const gabp_graph_t *Gc, gabp_state_t *S, int32_t schedule, double *max_change,
               int64_t *singular_index, int32_t *singular_is_node) {
    gabp_graph *G = const_cast<gabp_graph *>(Gc);
    if (!G || !S || S->g != Gc) return fail(GABP_EINVAL, "state does not belong to graph");
    if (schedule != GABP_SCHED_PARALLEL && schedule != GABP_SCHED_BROADCAST)
        return fail(GABP_EINVAL, "schedule must be parallel (0) or broadcast (2)");
    CK(cudaSetDevice(G->device));
    int rc = ensure_workspace(G, 1);
    if (rc) return rc;
    if (singular_index) *singular_index = -1;
    if (singular_is_node) *singular_is_node = 0;
    if (max_change) *max_change = 0.0;
    Ctrl c = gabp::fresh_ctrl();
    *G->h_ctrl = c;
    CK(cudaMemcpyAsync(G->ctrl, G->h_ctrl, sizeof(Ctrl), cudaMemcpyHostToDevice, G->stream));
    SweepArgs a = make_args(G);
    a.msg[0] = S->buf[S->cur];
    a.msg[1] = S->buf[S->cur ^ 1];
    if (G->g.E > 0)
        CK(gabp::launch_sweep(a, schedule, gabp::kModeSingle, gabp::kGatherMessage, G->stream));
    CK(cudaMemcpyAsync(G->h_ctrl, G->ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, G->stream));
    CK(cudaStreamSynchronize(G->stream));
    const Ctrl &h = *G->h_ctrl;
    const int slot = 1;
    if (h.agg_singular[slot] != gabp::kNoIndex) {
        if (singular_index) *singular_index = (int64_t)h.agg_singular[slot];
        if (singular_is_node) *singular_is_node = 1;
        return fail(GABP_ESINGULAR, "aggregate precision P~(%lld) = 0",
                    (long long)h.agg_singular[slot]);
    }
    if (h.singular_min[slot] != gabp::kNoIndex) {
        if (singular_index) *singular_index = (int64_t)h.singular_min[slot];
        return fail(GABP_ESINGULAR, "P_excl = 0 on edge %lld", (long long)h.singular_min[slot]);
    }
    if (max_change) {  // NaN when a new message is NaN (np.max propagates it)
        double v;
        unsigned long long bits = h.change_bits[slot];
        memcpy(&v, &bits, sizeof(v));
        *max_change = (h.msg_nonfinite[slot] & 2) ? NAN : v;
    }
    S->cur ^= 1;
    S->iteration += 1;
    S->messages_sent += (schedule == GABP_SCHED_BROADCAST) ? G->g.n : G->g.E;
    return GABP_OK;
}

// ---- whole-state checks and point reads -----------------------------------------------

int gabp_state_blown(const gabp_state_t *S, double blowup, int32_t *blown) {
    if (!S || !blown) return fail(GABP_EINVAL, "NULL argument");
    CK(cudaSetDevice(S->g->device));
    return state_blown(S->g, S->buf[S->cur], blowup, blown);
}

int gabp_state_gather(const gabp_state_t *S, const int64_t *h_edges, int64_t count,
                      double *h_prec, double *h_mean) {
    if (!S || count < 0 || (count > 0 && !h_edges)) return fail(GABP_EINVAL, "bad arguments");
    const gabp_graph *G = S->g;
    for (int64_t k = 0; k < count; ++k)
        if (h_edges[k] < 0 || h_edges[k] >= G->g.E)
            return fail(GABP_EINVAL, "edge id %lld out of range [0, %lld)",
                        (long long)h_edges[k], (long long)G->g.E);
    if (count == 0) return GABP_OK;
    CK(cudaSetDevice(G->device));
    int64_t *d_idx = nullptr;
    double2 *d_out = nullptr;
    CK(cudaMallocAsync(&d_idx, sizeof(int64_t) * count, G->stream));
    CK(cudaMallocAsync(&d_out, sizeof(double2) * count, G->stream));
    std::vector<double2> out(count);
    cudaError_t e = cudaMemcpyAsync(d_idx, h_edges, sizeof(int64_t) * count,
                                    cudaMemcpyHostToDevice, G->stream);
    if (e == cudaSuccess) e = gabp::launch_gather(count, d_idx, S->buf[S->cur], d_out, G->stream);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(out.data(), d_out, sizeof(double2) * count, cudaMemcpyDeviceToHost,
                            G->stream);
    cudaFreeAsync(d_idx, G->stream);
    cudaFreeAsync(d_out, G->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(G->stream);
    CK(e);
    for (int64_t k = 0; k < count; ++k) {
        if (h_prec) h_prec[k] = out[k].x;
        if (h_mean) h_mean[k] = out[k].y;
    }
    return GABP_OK;
}

int gabp_infer_marginals(const gabp_graph_t *G, const gabp_state_t *S, double *h_means,
                         double *h_precs) {
    if (!G || !S || S->g != G) return fail(GABP_EINVAL, "state does not belong to graph");
    CK(cudaSetDevice(G->device));
    const int64_t n = G->g.n;
    double *d = nullptr;
    CK(cudaMallocAsync(&d, sizeof(double) * 2 * n, G->stream));
    CK(gabp::launch_marginals(n, G->g.row_ptr, G->g.er, G->g.diag, G->g.prior_num,
                              S->buf[S->cur], d, d + n, G->stream));
    if (h_means)
        CK(cudaMemcpyAsync(h_means, d, sizeof(double) * n, cudaMemcpyDeviceToHost, G->stream));
    if (h_precs)
        CK(cudaMemcpyAsync(h_precs, d + n, sizeof(double) * n, cudaMemcpyDeviceToHost,
                           G->stream));
    CK(cudaFreeAsync(d, G->stream));
    CK(cudaStreamSynchronize(G->stream));
    return GABP_OK;
}

// ---- solve --------------------------------------------------------------------------------

// Marginals of the last solve in row order: the slice path keeps them in position order,
// in the node state records {P_i, x_i}.
static int rows_order(gabp_graph *G, int64_t slot, int64_t r0, int64_t nr, const double **xm,
                      const double **pm) {
    if (!G->slice_order) return GABP_OK;
    const double *rec = reinterpret_cast<const double *>(G->rec[slot]);
    constexpr int kRecStride = (int)(sizeof(gabp::NodeState) / sizeof(double));
    CK(gabp::slice_to_rows(G->g, r0, nr, rec + offsetof(gabp::NodeState, x) / sizeof(double),
                           kRecStride, G->xs, G->stream));
    CK(gabp::slice_to_rows(G->g, r0, nr, rec, kRecStride, G->ps, G->stream));
    *xm = G->xs;
    *pm = G->ps;
    return GABP_OK;
}

// Copies a finished solve's outputs to the host; a rank's graph returns its owned rows.
static int copy_results(gabp_graph *G, const gabp_options_t *opt, double ms, double *h_means,
                        double *h_precs, double *h_change_hist, double *h_res_hist,
                        gabp_report_t *rep) {
    const Ctrl &c = *G->h_ctrl;
    cudaStream_t st = G->stream;
    const int64_t slot = c.final_slot;
    const int64_t r0 = G->dist ? G->g.row_lo : 0;
    const int64_t nr = G->dist ? G->g.row_hi - G->g.row_lo : G->g.n;
    const double *xm = G->x[slot], *pm = G->p[slot];
    int rc = rows_order(G, slot, r0, nr, &xm, &pm);
    if (rc) return rc;
    if (h_means)
        CK(cudaMemcpyAsync(h_means, xm + r0, sizeof(double) * nr, cudaMemcpyDeviceToHost, st));
    if (h_precs)
        CK(cudaMemcpyAsync(h_precs, pm + r0, sizeof(double) * nr, cudaMemcpyDeviceToHost, st));
    if (h_change_hist && c.n_hist > 0)
        CK(cudaMemcpyAsync(h_change_hist, G->change_hist, sizeof(double) * c.n_hist,
                           cudaMemcpyDeviceToHost, st));
    if (h_res_hist && c.n_hist > 0)
        CK(cudaMemcpyAsync(h_res_hist, G->res_hist, sizeof(double) * c.n_hist,
                           cudaMemcpyDeviceToHost, st));
    if (!G->dist && opt->h_means_history && G->xhist && c.n_hist > 0) {
        const int64_t r = c.n_hist < G->xhist_rows ? c.n_hist : G->xhist_rows;
        CK(cudaMemcpyAsync(opt->h_means_history, G->xhist, sizeof(double) * r * G->g.n,
                           cudaMemcpyDeviceToHost, st));
    }
    double rsq_last = NAN;
    if (c.n_hist > 0)
        CK(cudaMemcpyAsync(&rsq_last, G->rsq_hist + (c.n_hist - 1), sizeof(double),
                           cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    fill_report(G, opt, ms, rsq_last, rep);
    if (rep && G->dist) {
        rep->messages_sent = c.iterations * G->dist->n_global;
        rep->final_rel_residual = (c.n_hist >= 1 && G->dist->bnorm > 0.0)
                                      ? sqrt(rsq_last) / G->dist->bnorm : NAN;
    }
    return GABP_OK;
}

int gabp_solve(gabp_graph_t *G, const gabp_options_t *opt, double *h_means, double *h_precs,
               double *h_change_hist, double *h_res_hist, gabp_report_t *rep) {
    if (!G) return fail(GABP_EINVAL, "NULL graph");
    double ms = 0.0;
    int rc = run_solve(G, opt, &ms);
    if (rc) return rc;
    return copy_results(G, opt, ms, h_means, h_precs, h_change_hist, h_res_hist, rep);
}

// ---- multi-rank -----------------------------------------------------------------------

int gabp_nccl_unique_id(void *out128) {
    if (!out128) return fail(GABP_EINVAL, "NULL argument");
    int rc = load_nccl();
    if (rc) return rc;
    ncclUniqueId id;
    NK(g_nccl.getUniqueId(&id));
    memcpy(out128, &id, sizeof(id));
    return GABP_OK;
}

int gabp_dist_attach(gabp_graph_t *G, const void *nccl_id, int32_t rank, int32_t world,
                     int64_t n_global, double bnorm_global, int32_t npeers,
                     const int32_t *peers, const int64_t *send_counts, const int64_t *send_idx,
                     const int64_t *recv_counts, const int64_t *recv_idx) {
    if (!G || world < 1 || rank < 0 || rank >= world || npeers < 0)
        return fail(GABP_EINVAL, "bad multi-rank arguments");
    if (G->dist) return fail(GABP_EINVAL, "graph already attached");
    CK(cudaSetDevice(G->device));
    DistState *D = new DistState();
    D->rank = rank;
    D->world = world;
    D->n_global = n_global;
    D->bnorm = bnorm_global;
    D->local = (nccl_id == nullptr);
    // per-peer blocks start at even node offsets: 3*off doubles stays 16-byte aligned for
    // the {P, P mu~} pairs of the halo buffers
    int64_t ns = 0, nr = 0;
    for (int q = 0; q < npeers; ++q) {
        D->peers.push_back(peers[q]);
        D->soff.push_back(ns);
        D->roff.push_back(nr);
        D->scount.push_back(send_counts[q]);
        D->rcount.push_back(recv_counts[q]);
        ns += (send_counts[q] + 1) & ~1ll;
        nr += (recv_counts[q] + 1) & ~1ll;
    }
    G->dist = D;  // released with the graph from here on
    std::vector<uint32_t> si(ns > 0 ? ns : 1, 0u), ri(nr > 0 ? nr : 1, 0u);
    int64_t ks = 0, kr = 0;
    for (int q = 0; q < npeers; ++q) {
        for (int64_t k = 0; k < send_counts[q]; ++k) si[D->soff[q] + k] = (uint32_t)send_idx[ks++];
        for (int64_t k = 0; k < recv_counts[q]; ++k) ri[D->roff[q] + k] = (uint32_t)recv_idx[kr++];
    }
    CK(cudaMalloc(&D->d_sidx, sizeof(uint32_t) * si.size()));
    CK(cudaMalloc(&D->d_ridx, sizeof(uint32_t) * ri.size()));
    CK(cudaMalloc(&D->d_sbuf, sizeof(double) * 4 * si.size()));
    CK(cudaMalloc(&D->d_rbuf, sizeof(double) * 4 * ri.size()));
    CK(cudaMalloc(&D->d_stats, sizeof(double) * 8));
    CK(cudaMemcpy(D->d_sidx, si.data(), sizeof(uint32_t) * si.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(D->d_ridx, ri.data(), sizeof(uint32_t) * ri.size(), cudaMemcpyHostToDevice));
    if (D->local) return GABP_OK;  // agreed over the partitions by gabp_dist_solve_local
    int caps = dist_local_caps(G);
    const int64_t sig = dia_signature(G);
    bool dia = sig != 0;
    if (world > 1) {
        int rc = load_nccl();
        if (rc) return rc;
        ncclUniqueId id;
        memcpy(&id, nccl_id, sizeof(id));
        NK(g_nccl.commInitRank(&D->comm, world, id, rank));
        // one small all-reduce (min) of the capability bits: every rank then runs the same
        // kernel family and issues the same NCCL call sequence each sweep
        int32_t *d_caps = nullptr;
        CK(cudaMalloc(&d_caps, sizeof(int32_t) * 2));
        const int32_t hc[2] = {caps & 1, (caps >> 1) & 1};
        CK(cudaMemcpy(d_caps, hc, sizeof(hc), cudaMemcpyHostToDevice));
        NK(g_nccl.allReduce(d_caps, d_caps, 2, ncclInt32, ncclMin, D->comm, G->stream));
        int32_t ag[2] = {0, 0};
        CK(cudaMemcpyAsync(ag, d_caps, sizeof(ag), cudaMemcpyDeviceToHost, G->stream));
        CK(cudaStreamSynchronize(G->stream));
        cudaFree(d_caps);
        caps = (ag[0] ? 1 : 0) | (ag[1] ? 2 : 0);
        // the diagonal layout only if every rank has the same one: min and max of the
        // signatures agree (max as the min of the negated)
        int64_t *d_sig = nullptr;
        CK(cudaMalloc(&d_sig, sizeof(int64_t) * 2));
        const int64_t hs[2] = {sig, -sig};
        CK(cudaMemcpy(d_sig, hs, sizeof(hs), cudaMemcpyHostToDevice));
        NK(g_nccl.allReduce(d_sig, d_sig, 2, ncclInt64, ncclMin, D->comm, G->stream));
        int64_t as[2] = {0, 0};
        CK(cudaMemcpyAsync(as, d_sig, sizeof(as), cudaMemcpyDeviceToHost, G->stream));
        CK(cudaStreamSynchronize(G->stream));
        cudaFree(d_sig);
        dia = as[0] != 0 && as[0] == -as[1];
    }
    return dist_agree(G, caps, dia);
}

// In-process partitions on the diagonal layout: the NCCL loop of dia_launch_nccl with the
// statistics reduced on the host and the halo moved by device copies.
int dia_move_local(int nparts, gabp_graph_t **parts) {
    for (int p = 0; p < nparts; ++p) CK(cudaStreamSynchronize(parts[p]->stream));
    for (int p = 0; p < nparts; ++p) {
        DistState *D = parts[p]->dist;
        for (size_t q = 0; q < D->peers.size(); ++q) {
            const int src = D->peers[q];
            DistState *S = parts[src]->dist;
            size_t qs = 0;
            while (qs < S->peers.size() && S->peers[qs] != p) ++qs;
            if (qs == S->peers.size() || S->scount[qs] != D->rcount[q] ||
                S->dsend[qs].nd != D->drecv[q].nd)
                return fail(GABP_EINVAL, "halo lists of ranks %d and %d disagree", p, src);
            CK(cudaMemcpyAsync(D->d_drbuf + D->dia_w * D->roff[q],
                               S->d_dsbuf + S->dia_w * S->soff[qs],
                               sizeof(double) * D->dia_w * D->rcount[q],
                               cudaMemcpyDeviceToDevice, parts[p]->stream));
        }
    }
    return GABP_OK;
}

int dia_solve_local(int nparts, gabp_graph_t **parts, std::vector<SweepArgs> &args,
                    int64_t total, double *device_ms) {
    for (int p = 0; p < nparts; ++p) {
        CK(gabp::launch_dia_init(args[p], parts[p]->stream));
        int rc = dia_pack_all(parts[p], args[p], 0, 0, parts[p]->stream);
        if (rc) return rc;
    }
    int rc = dia_move_local(nparts, parts);
    if (rc) return rc;
    for (int p = 0; p < nparts; ++p) {
        rc = dia_unpack_all(parts[p], args[p], 0, 0, parts[p]->stream);
        if (rc) return rc;
    }
    gabp_graph *G0 = parts[0];
    for (int64_t s = 0; s < total; ++s) {
        for (int p = 0; p < nparts; ++p) CK(gabp::launch_dia_sweep(args[p], parts[p]->stream));
        double red[6] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY, -INFINITY, 0.0};
        for (int p = 0; p < nparts; ++p) {
            double st6[6];
            CK(cudaMemcpyAsync(st6, parts[p]->dist->d_stats, sizeof(st6),
                               cudaMemcpyDeviceToHost, parts[p]->stream));
            CK(cudaStreamSynchronize(parts[p]->stream));
            for (int k = 0; k < 5; ++k) red[k] = fmax(red[k], st6[k]);
            red[5] += st6[5];
        }
        for (int p = 0; p < nparts; ++p) {
            CK(cudaMemcpyAsync(parts[p]->dist->d_stats, red, sizeof(red), cudaMemcpyHostToDevice,
                               parts[p]->stream));
            CK(gabp::launch_dia_finish(args[p], parts[p]->stream));
            rc = dia_pack_all(parts[p], args[p], -1, 1, parts[p]->stream);
            if (rc) return rc;
        }
        rc = dia_move_local(nparts, parts);
        if (rc) return rc;
        for (int p = 0; p < nparts; ++p) {
            rc = dia_unpack_all(parts[p], args[p], -1, 1, parts[p]->stream);
            if (rc) return rc;
        }
        for (int p = 0; p < nparts; ++p) CK(cudaStreamSynchronize(parts[p]->stream));
        int32_t done = 0;
        CK(cudaMemcpy(&done, &G0->ctrl->done, sizeof(done), cudaMemcpyDeviceToHost));
        if (done) break;
    }
    double ms = 0.0;
    for (int p = 0; p < nparts; ++p) {
        int rc2 = finish_loop(parts[p], p == 0 ? &ms : nullptr);
        if (rc2 && p == 0) return rc2;
    }
    if (device_ms) *device_ms = ms;
    return GABP_OK;
}

// One GPU, several row blocks in this process: the multi-rank loop with the cross-rank
// reduction done on the host and the halo moved with device-to-device copies.  Same
// kernels as the NCCL path; used to test the partitioned solve on a single device.
int gabp_dist_solve_local(int32_t nparts, gabp_graph_t **parts, const gabp_options_t *opt,
                          double *device_ms) {
    if (nparts < 1 || !parts) return fail(GABP_EINVAL, "no partitions");
    for (int p = 0; p < nparts; ++p)
        if (!parts[p] || !parts[p]->dist || !parts[p]->dist->local || parts[p]->dist->rank != p)
            return fail(GABP_EINVAL, "partition %d is not attached in local mode as rank %d", p,
                        p);
    if (opt && opt->schedule != GABP_SCHED_BROADCAST)
        return fail(GABP_EINVAL, "the multi-rank solve runs the broadcast schedule");
    std::vector<SweepArgs> args(nparts);
    if (parts[0]->dist->use_slices < 0) {  // first solve: agree on the protocol (AND of caps)
        int caps = 3;
        const int64_t sig0 = dia_signature(parts[0]);
        bool dia = sig0 != 0;
        for (int p = 0; p < nparts; ++p) {
            caps &= dist_local_caps(parts[p]);
            dia = dia && dia_signature(parts[p]) == sig0;
        }
        for (int p = 0; p < nparts; ++p) {
            int rc = dist_agree(parts[p], caps, dia);
            if (rc) return rc;
        }
    }
    for (int p = 0; p < nparts; ++p) {
        int rc = solve_setup(parts[p], opt);
        if (rc) return rc;
        args[p] = make_dist_args(parts[p]);
        parts[p]->slice_order = !parts[p]->dist->use_dia &&
                                dist_gather(parts[p]) == gabp::kGatherSlice;
    }
    gabp_graph *G0 = parts[0];
    CK(cudaEventRecord(G0->ev[2], G0->stream));
    const int64_t total = opt->max_iter + 2;
    if (parts[0]->dist->use_dia) return dia_solve_local(nparts, parts, args, total, device_ms);
    for (int64_t s = 0; s < total; ++s) {
        for (int p = 0; p < nparts; ++p) {
            if (const int64_t nbs = split_slices(parts[p])) {  // the NCCL path's split sweep
                parts[p]->dist->split_launches++;
                SweepArgs b = args[p], in = args[p];
                b.sl_hi = nbs;
                int64_t gb = 0;
                CK(gabp::launch_slice_boundary(b, &gb, parts[p]->stream));
                in.sl_lo = nbs;
                in.part_base = gb;
                CK(gabp::launch_slice_part(in, kReserveSms, parts[p]->stream));
            } else {
                CK(gabp::launch_sweep(args[p], GABP_SCHED_BROADCAST, gabp::kModeSolve,
                                      dist_gather(parts[p]), parts[p]->stream));
            }
        }
        double red[6] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY, -INFINITY, 0.0};
        for (int p = 0; p < nparts; ++p) {
            double st6[6];
            CK(cudaMemcpyAsync(st6, parts[p]->dist->d_stats, sizeof(st6),
                               cudaMemcpyDeviceToHost, parts[p]->stream));
            CK(cudaStreamSynchronize(parts[p]->stream));
            for (int k = 0; k < 5; ++k) red[k] = fmax(red[k], st6[k]);
            red[5] += st6[5];
        }
        for (int p = 0; p < nparts; ++p) {
            CK(cudaMemcpyAsync(parts[p]->dist->d_stats, red, sizeof(red), cudaMemcpyHostToDevice,
                               parts[p]->stream));
            CK(gabp::launch_finish(args[p], parts[p]->stream));
            DistState *D = parts[p]->dist;
            for (size_t q = 0; q < D->peers.size(); ++q)
                CK(gabp::launch_halo_pack(args[p], D->d_sidx + D->soff[q], D->scount[q],
                                          D->d_sbuf + 4 * D->soff[q], parts[p]->stream, 0));
            CK(cudaStreamSynchronize(parts[p]->stream));
        }
        for (int p = 0; p < nparts; ++p) {  // move each peer's block for p into p's recv
            DistState *D = parts[p]->dist;
            for (size_t q = 0; q < D->peers.size(); ++q) {
                const int src = D->peers[q];
                DistState *S = parts[src]->dist;
                size_t qs = 0;
                while (qs < S->peers.size() && S->peers[qs] != p) ++qs;
                if (qs == S->peers.size() || S->scount[qs] != D->rcount[q])
                    return fail(GABP_EINVAL, "halo lists of ranks %d and %d disagree", p, src);
                CK(cudaMemcpyAsync(D->d_rbuf + 4 * D->roff[q], S->d_sbuf + 4 * S->soff[qs],
                                   sizeof(double) * 4 * D->rcount[q], cudaMemcpyDeviceToDevice,
                                   parts[p]->stream));
            }
            for (size_t q = 0; q < D->peers.size(); ++q)
                CK(gabp::launch_halo_unpack(args[p], D->d_ridx + D->roff[q], D->rcount[q],
                                            D->d_rbuf + 4 * D->roff[q], parts[p]->stream, 0));
        }
        for (int p = 0; p < nparts; ++p) CK(cudaStreamSynchronize(parts[p]->stream));
        int32_t done = 0;
        CK(cudaMemcpy(&done, &G0->ctrl->done, sizeof(done), cudaMemcpyDeviceToHost));
        if (done) break;
    }
    double ms = 0.0;
    for (int p = 0; p < nparts; ++p) {
        int rc = finish_loop(parts[p], p == 0 ? &ms : nullptr);
        if (rc && p == 0) return rc;
    }
    if (device_ms) *device_ms = ms;
    return GABP_OK;
}

// Outputs of the last solve of a partition (owned rows only).
int gabp_dist_results(gabp_graph_t *G, const gabp_options_t *opt, double *h_means,
                      double *h_precs, double *h_change_hist, double *h_res_hist,
                      gabp_report_t *rep) {
    if (!G || !G->dist) return fail(GABP_EINVAL, "not a partition");
    return copy_results(G, opt, 0.0, h_means, h_precs, h_change_hist, h_res_hist, rep);
}

int gabp_solve_device(gabp_graph_t *G, const gabp_options_t *opt, double *d_means,
                      double *d_precs, gabp_report_t *rep) {
    if (!G) return fail(GABP_EINVAL, "NULL graph");
    double ms = 0.0;
    int rc = run_solve(G, opt, &ms);
    if (rc) return rc;
    const Ctrl &c = *G->h_ctrl;
    cudaStream_t st = G->stream;
    const int64_t slot = c.final_slot;
    const double *xm = G->x[slot], *pm = G->p[slot];
    rc = rows_order(G, slot, 0, G->g.n, &xm, &pm);
    if (rc) return rc;
    if (d_means)
        CK(cudaMemcpyAsync(d_means, xm, sizeof(double) * G->g.n, cudaMemcpyDeviceToDevice, st));
    if (d_precs)
        CK(cudaMemcpyAsync(d_precs, pm, sizeof(double) * G->g.n, cudaMemcpyDeviceToDevice, st));
    double rsq_last = NAN;
    if (c.n_hist > 0)
        CK(cudaMemcpyAsync(&rsq_last, G->rsq_hist + (c.n_hist - 1), sizeof(double),
                           cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    fill_report(G, opt, ms, rsq_last, rep);
    return GABP_OK;
}

int gabp_solve_system(int64_t n, int64_t npairs, const double *h_diag, const double *h_rhs,
                      const int64_t *h_pair_i, const int64_t *h_pair_j,
                      const double *h_pair_v, int32_t device, const gabp_options_t *opt,
                      double *h_means, double *h_precs, double *h_change_hist,
                      double *h_res_hist, gabp_report_t *rep) {
    int rc = check_options(opt);
    if (rc) return rc;
    gabp_graph_t *G = nullptr;
    const double t0 = host_ms();
    rc = gabp_graph_create(n, npairs, h_diag, h_rhs, h_pair_i, h_pair_j, h_pair_v, device, &G);
    if (rc) return rc;
    const double t1 = host_ms();
    double ms = 0.0;
    rc = run_solve(G, opt, &ms);
    const double t2 = host_ms();
    if (!rc) rc = copy_results(G, opt, ms, h_means, h_precs, h_change_hist, h_res_hist, rep);
    const double t3 = host_ms();
    gabp_graph_destroy(G);
    if (host_timing())
        fprintf(stderr, "[gabp] solve_system: create %.2f ms, solve %.2f ms (device %.2f), "
                        "results %.2f ms, destroy %.2f ms\n",
                t1 - t0, t2 - t1, ms, t3 - t2, host_ms() - t3);
    return rc;
}

int gabp_residual_norm_per_eq(const gabp_graph_t *G, const double *h_x, double *out) {
    if (!G || !h_x || !out) return fail(GABP_EINVAL, "NULL argument");
    CK(cudaSetDevice(G->device));
    const int64_t n = G->g.n;
    const int64_t nparts = (n + 4095) / 4096;
    double *d = nullptr;
    CK(cudaMallocAsync(&d, sizeof(double) * (n + nparts + 1), G->stream));
    CK(cudaMemcpyAsync(d, h_x, sizeof(double) * n, cudaMemcpyHostToDevice, G->stream));
    CK(gabp::launch_residual_sq(n, G->g.row_ptr, G->g.er, G->g.diag, G->g.rhs, d, d + n, nparts,
                                d + n + nparts, G->stream));
    double ss = 0.0;
    CK(cudaMemcpyAsync(&ss, d + n + nparts, sizeof(double), cudaMemcpyDeviceToHost, G->stream));
    CK(cudaFreeAsync(d, G->stream));
    CK(cudaStreamSynchronize(G->stream));
    *out = sqrt(ss) / (double)n;
    return GABP_OK;
}

int gabp_small_plan(int64_t n, const uint32_t *row_ptr, int64_t *bounds, int64_t *cap_edges,
                    int64_t *cap_rows) {
    if (n < 1 || !row_ptr || !bounds) return 0;
    gabp::SmallPart p = {};
    if (!gabp::small_candidate(n, (int64_t)row_ptr[n]) || !gabp::small_plan(n, row_ptr, &p))
        return 0;
    for (int c = 0; c <= p.C; ++c) bounds[c] = (int64_t)p.nb[c];
    int64_t ce = 0, cr = 0;
    gabp::small_capacity(p.cfg, &ce, &cr);
    if (cap_edges) *cap_edges = ce;
    if (cap_rows) *cap_rows = cr;
    return p.C;
}

int gabp_bench_sweeps(gabp_graph_t *G, int32_t schedule, int32_t gather_mode, int64_t sweeps,
                      double *ms_per_sweep) {
    if (!G || sweeps < 1 || !ms_per_sweep) return fail(GABP_EINVAL, "bad argument");
    if (schedule != GABP_SCHED_PARALLEL && schedule != GABP_SCHED_BROADCAST)
        return fail(GABP_EINVAL, "bad schedule");
    CK(cudaSetDevice(G->device));
    int rc = ensure_workspace(G, 1);
    if (rc) return rc;
    Ctrl c = gabp::fresh_ctrl();
    c.next_sweep = 1;
    c.epsilon = 0.0;        // never "converged": every launch does the full sweep
    c.blowup = INFINITY;
    c.rel_tol = 0.0;
    c.bnorm = G->g.rhs_norm;
    c.max_iter = INT64_MAX / 4;
    c.n = G->g.n;
    *G->h_ctrl = c;
    cudaStream_t st = G->stream;
    // histories are only written when a decision is taken (t <= max_iter): size them
    rc = ensure_workspace(G, sweeps + 5);
    if (rc) return rc;
    CK(cudaMemcpyAsync(G->ctrl, G->h_ctrl, sizeof(Ctrl), cudaMemcpyHostToDevice, st));
    CK(cudaMemsetAsync(G->msg[0], 0, sizeof(double2) * msg_slots(G->g), st));
    SweepArgs a = make_args(G);
    gabp_options_t o{};
    o.schedule = schedule;
    o.gather_mode = gather_mode;
    o.epsilon = 1.0;
    o.max_iter = 1;
    o.blowup = 2.0;
    rc = check_options(&o);
    if (rc) return rc;
    if (schedule == GABP_SCHED_BROADCAST && gather_mode == GABP_GATHER_AUTO && G->g.dia_D > 0) {
        CK(gabp::launch_dia_init(a, st));
        for (int k = 0; k < 3; ++k) CK(gabp::launch_dia_sweep(a, st));
        CK(cudaEventRecord(G->ev[2], st));
        for (int64_t k = 0; k < sweeps; ++k) CK(gabp::launch_dia_sweep(a, st));
        CK(cudaEventRecord(G->ev[3], st));
        CK(cudaMemcpyAsync(G->h_ctrl, G->ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        float dms = 0.f;
        CK(cudaEventElapsedTime(&dms, G->ev[2], G->ev[3]));
        if (G->h_ctrl->done)
            return fail(GABP_EINVAL, "bench sweeps stopped early (diverged at sweep %lld)",
                        (long long)G->h_ctrl->iterations);
        *ms_per_sweep = dms / (double)sweeps;
        return GABP_OK;
    }
    if (schedule == GABP_SCHED_PARALLEL && gather_mode == GABP_GATHER_AUTO && G->g.dia_D > 0 &&
        !getenv("GABP_NO_DIA_PAR")) {
        for (int k = 0; k < 3; ++k) CK(gabp::launch_dia_par_sweep(a, st));
        CK(cudaEventRecord(G->ev[2], st));
        for (int64_t k = 0; k < sweeps; ++k) CK(gabp::launch_dia_par_sweep(a, st));
        CK(cudaEventRecord(G->ev[3], st));
        CK(cudaMemcpyAsync(G->h_ctrl, G->ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        float dms = 0.f;
        CK(cudaEventElapsedTime(&dms, G->ev[2], G->ev[3]));
        if (G->h_ctrl->done)
            return fail(GABP_EINVAL, "bench sweeps stopped early (diverged at sweep %lld)",
                        (long long)G->h_ctrl->iterations);
        *ms_per_sweep = dms / (double)sweeps;
        return GABP_OK;
    }
    rc = check_slice(G, &o);
    if (rc) return rc;
    const int gather = pick_gather(G, &o);
    if (gather == gabp::kGatherSliceParallel && !G->g.stwin) {
        rc = gabp::build_stwin(G->g, st, g_err, sizeof(g_err));
        if (rc) return rc;
        G->ws_gen++;
    }
    a.stwin = G->g.stwin;
    if (gather == gabp::kGatherRowParallel && G->g.bins == 0 && !G->dist) {
        rc = gabp::build_bins(G->g, st, g_err, sizeof(g_err));
        if (rc) return rc;
        G->ws_gen++;
        a = make_args(G);
    }
    // launches 1-3 stream less than a full sweep (zero initial messages, slice.cu launch
    // kinds): run them untimed, so the figure is the steady-state sweep
    for (int k = 0; k < 3; ++k) CK(gabp::launch_sweep(a, schedule, gabp::kModeSolve, gather, st));
    CK(cudaEventRecord(G->ev[2], st));
    for (int64_t k = 0; k < sweeps; ++k)
        CK(gabp::launch_sweep(a, schedule, gabp::kModeSolve, gather, st));
    CK(cudaEventRecord(G->ev[3], st));
    CK(cudaMemcpyAsync(G->h_ctrl, G->ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, G->ev[2], G->ev[3]));
    if (G->h_ctrl->done)
        return fail(GABP_EINVAL, "bench sweeps stopped early (diverged at sweep %lld)",
                    (long long)G->h_ctrl->iterations);
    *ms_per_sweep = ms / (double)sweeps;
    return GABP_OK;
}

// Debug hook (GABP_TIMELINE builds): clock64 timeline of CTA 0.
int gabp_debug_timeline(long long *out, int32_t n) {
    return gabp::read_timeline(out, n) == 0 ? GABP_OK : fail(GABP_EINVAL, "not a timeline build");
}

}  // extern "C"
