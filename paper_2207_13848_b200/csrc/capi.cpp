// C-ABI layer: device context, residency, validation, orchestration and the
// single NCCL all-reduce.  See include/spnnz_gpu/capi.h for the contract and
// the reference functions each entry point replaces.
//
// Built with -ffp-contract=off: the host-side estimator tail evaluates the
// reference's double expressions (predict.hpp:86-123, :163-188) in the same
// order, so device CR, host CR and the reference CR are the same IEEE value.
#include "spnnz_gpu/capi.h"

#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "kernels.h"

using namespace spnnz_gpu;

namespace {

thread_local std::string g_err;

int set_err(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CU(call)                                                                         \
    do {                                                                                 \
        cudaError_t e_ = (call);                                                         \
        if (e_ != cudaSuccess)                                                           \
            return set_err(e_ == cudaErrorMemoryAllocation ? SPNNZ_ENOMEM : SPNNZ_ECUDA, \
                           "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__,    \
                           __LINE__);                                                    \
    } while (0)

#define RC(call)                   \
    do {                           \
        int r_ = (call);           \
        if (r_ != SPNNZ_OK) return r_; \
    } while (0)

// ------------------------------------------------------------ NCCL (dlopen)
struct Nccl {
    bool loaded = false;
    std::string why;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

Nccl& nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        // The process's NCCL when one is loaded (e.g. torch's), else
        // SPNNZ_NCCL_LIB (the Python layer points it at the pip-installed
        // NCCL torch itself uses), else the loader's libnccl.so.2.  Local
        // binding: loading an older system libnccl.so.2 first would make a
        // later `import torch` bind to it and fail on newer NCCL symbols.
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h)
            if (const char* p = getenv("SPNNZ_NCCL_LIB"))
                if (*p) h = dlopen(p, RTLD_NOW | RTLD_LOCAL);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_LOCAL);
        if (!h) {
            n.why = dlerror();
            return;
        }
        n.GetUniqueId = reinterpret_cast<decltype(n.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
        n.CommInitRank = reinterpret_cast<decltype(n.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
        n.CommDestroy = reinterpret_cast<decltype(n.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
        n.AllReduce = reinterpret_cast<decltype(n.AllReduce)>(dlsym(h, "ncclAllReduce"));
        n.GroupStart = reinterpret_cast<decltype(n.GroupStart)>(dlsym(h, "ncclGroupStart"));
        n.GroupEnd = reinterpret_cast<decltype(n.GroupEnd)>(dlsym(h, "ncclGroupEnd"));
        n.GetErrorString =
            reinterpret_cast<decltype(n.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
        n.loaded = n.GetUniqueId && n.CommInitRank && n.CommDestroy && n.AllReduce &&
                   n.GroupStart && n.GroupEnd && n.GetErrorString;
        if (!n.loaded) n.why = "libnccl lacks required symbols";
    });
    return n;
}

#define NC(call)                                                                          \
    do {                                                                                  \
        ncclResult_t r_ = (call);                                                         \
        if (r_ != ncclSuccess)                                                            \
            return set_err(SPNNZ_ENCCL, "NCCL %s: %s", #call, nccl().GetErrorString(r_)); \
    } while (0)

// ---------------------------------------------------------- device buffer
// Guard bands (SPNNZ_GUARD=1 when a buffer is allocated): every allocation
// gets kGuardBytes of a known pattern after its last element, and
// spnnz_gpu_check_guards() reports any buffer whose band changed -- an
// out-of-bounds write past a library buffer.  (compute-sanitizer is closed on
// the GPU pool this was built on; this is the check that runs instead.)
constexpr size_t kGuardBytes = 256;
constexpr unsigned char kGuardByte = 0xA5;

struct GuardEntry {
    const void* base;
    size_t bytes;  // payload; the band follows
};
std::mutex g_guard_mu;
std::vector<GuardEntry> g_guards;
int64_t g_guard_released_broken = 0, g_guard_released = 0;

bool band_intact(const GuardEntry& g) {
    unsigned char band[kGuardBytes];
    if (cudaMemcpy(band, static_cast<const unsigned char*>(g.base) + g.bytes, kGuardBytes,
                   cudaMemcpyDeviceToHost) != cudaSuccess)
        return false;
    for (unsigned char b : band)
        if (b != kGuardByte) return false;
    return true;
}

bool guard_on() {
    const char* e = getenv("SPNNZ_GUARD");
    return e && atoi(e) > 0;
}

// Owns one device allocation; freed with the context (the destructor runs
// after spnnz_gpu_destroy has selected the context's device).
template <typename T>
struct DBuf {
    T* p = nullptr;
    int64_t n = 0;
    DBuf() = default;
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    ~DBuf() { release(); }
    int ensure(int64_t want) {
        if (want <= n && p) return SPNNZ_OK;
        release();
        const size_t bytes = sizeof(T) * static_cast<size_t>(std::max<int64_t>(want, 1));
        const bool guard = guard_on();
        cudaError_t e = cudaMalloc(&p, bytes + (guard ? kGuardBytes : 0));
        if (e != cudaSuccess) {
            p = nullptr;
            return set_err(SPNNZ_ENOMEM, "cudaMalloc(%zu): %s", bytes, cudaGetErrorString(e));
        }
        if (guard) {
            cudaMemset(reinterpret_cast<unsigned char*>(p) + bytes, kGuardByte, kGuardBytes);
            std::lock_guard<std::mutex> lk(g_guard_mu);
            g_guards.push_back(GuardEntry{p, bytes});
        }
        n = want;
        return SPNNZ_OK;
    }
    void release() {
        if (p) {
            {
                std::lock_guard<std::mutex> lk(g_guard_mu);
                for (size_t i = 0; i < g_guards.size(); ++i)
                    if (g_guards[i].base == p) {
                        ++g_guard_released;  // a buffer's band is checked before it is freed
                        if (!band_intact(g_guards[i])) ++g_guard_released_broken;
                        g_guards[i] = g_guards.back();
                        g_guards.pop_back();
                        break;
                    }
            }
            cudaFree(p);
        }
        p = nullptr;
        n = 0;
    }
};

}  // namespace

struct spnnz_gpu_ctx {
    int device = 0, rank = 0, world = 1, num_sms = 148;
    cudaStream_t stream = nullptr;
    // host-residency loads of C = A*A upload B.col in chunks on a copy stream
    // so the next FLOP pass can start on the tiles whose entries have landed
    cudaStream_t cstream = nullptr, fstream = nullptr;
    cudaStream_t hstream = nullptr;   // heavy batches beside the FLOP pass (heavy_beside)
    cudaEvent_t ev_hdone = nullptr;
    cudaEvent_t ev_gate = nullptr;    // the FLOP pass's end, for heavy runs gated behind it
    int heavy_beside = -1;            // A/B knob SPNNZ_HEAVY_BESIDE (-1: the policy in run_symbolic)
    static constexpr int kChunks = 8;
    cudaEvent_t ev_rpt = nullptr, ev_chunk[kChunks] = {}, ev_fdone = nullptr;
    int64_t chunk_tile_end[kChunks] = {};
    int n_chunks = 0;
    bool pending_upload = false;
    static constexpr int kSide = 4;
    cudaStream_t side[kSide] = {};        // symbolic tiers, concurrent with the heavy rows
    cudaEvent_t fork = nullptr, join[kSide] = {};
    cudaEvent_t ev_bin = nullptr, ev_flop = nullptr;  // early binning (run_symbolic)
    // device-residency inputs are read after the caller's work queued on
    // in_stream (default: the legacy default stream, where torch and most
    // callers queue); c->stream itself is non-blocking
    cudaStream_t in_stream = nullptr;
    cudaEvent_t ev_in = nullptr;
    ncclComm_t comm = nullptr;

    // matrices
    bool loaded = false;
    bool same_b = false;
    bool b_intervals = false;  // interval heavy path requested (SPNNZ_HEAVY_INTERVALS=1)
    bool b_sorted = false;     // ... and B's rows checked non-decreasing at load
    bool rows_mode = false;    // banded A: the FLOP pass's row-per-thread tiles (checked at load)
    int64_t mp_part = kMpPart;       // its products per pass (test knob SPNNZ_MP_PART, read at load)
    int64_t mp_max = kMpMaxDefault;  // multipass tier limit (knob SPNNZ_MP_MAX read at load; 0 = heavy path instead)
    int tiers_beside = -1;     // the symbolic tiers run beside the FLOP pass (A/B knob SPNNZ_TIERS_BESIDE; -1: policy)
    int32_t a_rows = 0, a_cols = 0, b_rows = 0, b_cols = 0;
    int32_t row_lo = 0, row_hi = 0;
    int64_t b_nnz = 0;
    DBuf<int64_t> b_rpt;
    DBuf<int32_t> b_col;
    DBuf<int64_t> a_rpt;  // shard rpt (only when A != B)
    DBuf<int32_t> a_col;
    DevCsr a;             // this rank's A shard view

    // profile
    DBuf<int64_t> flop;
    bool profile_valid = false;
    // own: computed by this context's FLOP pass over the loaded matrices;
    // else installed by the caller (set_profile) and used as the reference
    // uses its FlopProfile argument (tsize, f*, F, the per-row views)
    bool profile_own = false;
    DBuf<int64_t> flop_true;  // true FLOP of every local row under a caller profile (exact pass)
    uint64_t epoch = 0;          // bumped by every load (matrices changed)
    uint64_t profile_gen = 0;    // bumped whenever the resident profile changes

    // Heavy-row sizes (count, entries, products, boundary cells) a sampled
    // pass needs on the host to size its buffers.  Known in advance -- no
    // mid-call wait for the binning -- when no row can be heavy (the resident
    // own profile's max <= kBin5Max) or the same draw ran before on the same
    // matrices (cached below); checked against the device's counts after the
    // call, rerun eagerly on a mismatch.
    struct HeavySizes {
        int64_t count = 0, ents = 0, products = 0, cells = 0;
        bool operator==(const HeavySizes& o) const {
            return count == o.count && ents == o.ents && products == o.products && cells == o.cells;
        }
    };
    bool hc_valid = false;
    uint64_t hc_epoch = 0, hc_seed = 0;
    int64_t hc_n = 0;
    HeavySizes hc;
    HeavySizes observed;  // filled by run_symbolic from the device counts (valid after the call's sync)
    bool observed_set = false;

    // CUDA graph of a whole sync-free predictor call, replayed while its key
    // (matrices, profile, draw, outputs) is unchanged
    struct GraphKey {
        int kind = -1;  // 0 run_prediction, 1 on the resident profile
        uint64_t epoch = 0, profile_gen = 0, seed = 0;
        int64_t n = 0;
        const void *rows = nullptr, *ceil = nullptr, *real = nullptr;
        bool fused = false, profiling = false;
        bool operator==(const GraphKey& o) const {
            return kind == o.kind && epoch == o.epoch && profile_gen == o.profile_gen && seed == o.seed &&
                   n == o.n && rows == o.rows && ceil == o.ceil && real == o.real && fused == o.fused &&
                   profiling == o.profiling;
        }
    };
    cudaGraphExec_t gexec = nullptr;
    GraphKey gkey;
    // compute_flop's own graph: keyed by the matrices, the output and its
    // residency (the pass has no data-dependent host decision)
    cudaGraphExec_t fgexec = nullptr;
    uint64_t fg_epoch = 0;
    const void* fg_out = nullptr;
    int fg_res = -1;
    int64_t fg_launches = 0;
    int64_t g_launches = 0;
    HeavySizes g_known;
    bool dbg_t = false;              // SPNNZ_DEBUG_TIMELINE: per-stream end times to stderr
    cudaEvent_t dbg_ev[8] = {};       // [0] start [1] FLOP end [2..5] tier streams [6] heavy end [7] join
    bool used_small = false;  // the last pipeline took the fused small path (run_small)
    bool g_small = false;     // ... and so does the captured graph
    long long* h_init = nullptr;  // pinned: initial totals of a profile-mode call (read by its graph)
    bool capturing = false;
    int64_t profile_total = 0, profile_max = 0;

    // scratch
    DBuf<int32_t> tile_x;
    DBuf<unsigned long long> flop_sched;  // k_flop_smem tile tickets (zeroed once, kept zero)
    DBuf<uint16_t> deg;  // uint16 row lengths of B (rebuilt every FLOP pass)
    DBuf<unsigned> deg_escapes;  // 1 when some B row has >= 65535 entries (row-block kernels)
    uint64_t esc_epoch = ~0ull;   // the load whose B deg_escapes was last zeroed for
    DBuf<long long> tile_carry, tile_total, tile_max;
    DBuf<long long> totals;
    DBuf<long long> totals_table;  // world x kTotals: the all-reduce's all-gather table
    long long* h_totals = nullptr;  // pinned mirror
    int32_t* h_counts = nullptr;    // pinned mirror of bin counts
    DBuf<int32_t> counts;
    DBuf<int32_t> lists;
    int64_t list_cap = 0;
    DBuf<int64_t> heavy_unit_off, heavy_eoff, heavy_foff, heavy_epre, heavy_eb0, heavy_flops;
    DBuf<long long> heavy_rc, heavy_cur;
    DBuf<int32_t> heavy_pbuf, heavy_utab, heavy_slot_item;
    DBuf<int64_t> heavy_boff;                  // interval path (sorted B)
    DBuf<int32_t> heavy_bnd, heavy_unit_item, heavy_unit_e0;
    DBuf<int4> heavy_tasks;  // HeavyTask = 32 bytes = 2 x int4
    long long* h_meta = nullptr;    // pinned mirror of heavy_meta
    DBuf<uint32_t> pool;
    int64_t pool_slots = 0, pool_words = 0;
    DBuf<long long> heavy_meta;
    DBuf<long long> sorted_cnt;
    DBuf<int64_t> item_flop;  // FLOP of this rank's sampled rows (balanced multi-GPU pass)
    DBuf<int64_t> item_units; // their chunk offsets (flat item-FLOP decomposition)
    DBuf<int64_t> item_window;  // [lo, hi) of the sampled rows this rank counts
    DBuf<int32_t> redo;       // fused predict: rows left to an IEEE division
    DBuf<unsigned long long> nredo;
    DBuf<int32_t> samples;
    DBuf<int32_t> rows_in;
    DBuf<int64_t> out64;
    DBuf<double> outf;
    DBuf<int32_t> bad;

    // instrumentation
    bool profiling = false;
    bool fused = false;  // SPNNZ_FUSED_PREDICT=1: the fused single-pass predictor
    int ev_order = 0;
    cudaEvent_t ev[6] = {};
    double last_ms[5] = {};
    const char* flop_kernel = "";  // the last FLOP pass's kernel (instrumentation)
    int64_t last_launches = 0;
};

namespace {

int ensure_dev(spnnz_gpu_ctx* c) {
    CU(cudaSetDevice(c->device));
    return SPNNZ_OK;
}

// The main stream waits for a chunked upload still in flight (every entry
// point but the prediction pipeline, which overlaps its FLOP pass with it).
int settle_upload(spnnz_gpu_ctx* c) {
    if (!c->pending_upload) return SPNNZ_OK;
    CU(cudaStreamWaitEvent(c->stream, c->ev_rpt, 0));
    for (int k = 0; k < c->n_chunks; ++k) CU(cudaStreamWaitEvent(c->stream, c->ev_chunk[k], 0));
    c->pending_upload = false;
    return SPNNZ_OK;
}

// The context stream waits for the caller's queued work before it reads a
// device-residency input (e.g. a tensor an asynchronous kernel just wrote).
int order_after_caller(spnnz_gpu_ctx* c) {
    CU(cudaEventRecord(c->ev_in, c->in_stream));
    CU(cudaStreamWaitEvent(c->stream, c->ev_in, 0));
    return SPNNZ_OK;
}

int check_ctx(spnnz_gpu_ctx* c, bool need_loaded = true, bool settle = true) {
    if (!c) return set_err(SPNNZ_EINVAL, "null context");
    RC(ensure_dev(c));
    if (need_loaded && !c->loaded) return set_err(SPNNZ_ESTATE, "no matrices loaded");
    if (settle) RC(settle_upload(c));
    return SPNNZ_OK;
}

int dims_ok(spnnz_gpu_ctx* c, const char* who) {
    if (c->a_cols != c->b_rows)
        return set_err(SPNNZ_EINVAL, "%s: A.cols %d != B.rows %d", who, c->a_cols, c->b_rows);
    return SPNNZ_OK;
}

int local_rows(spnnz_gpu_ctx* c) { return c->row_hi - c->row_lo; }

// Copy a caller buffer to the device (or pass device pointers through).
template <typename T>
int stage_in(spnnz_gpu_ctx* c, const T* src, int64_t n, int residency, DBuf<T>& buf,
             const T** dev) {
    if (residency == SPNNZ_DEVICE || n == 0) {
        *dev = src;
        return SPNNZ_OK;
    }
    RC(buf.ensure(n));
    CU(cudaMemcpyAsync(buf.p, src, sizeof(T) * n, cudaMemcpyHostToDevice, c->stream));
    *dev = buf.p;
    return SPNNZ_OK;
}

int sym_scratch(spnnz_gpu_ctx* c, int64_t items, SymScratch* s) {
    if (items > c->list_cap) {
        RC(c->lists.ensure(items * kNumBins));
        RC(c->heavy_unit_off.ensure(items + 1));
        RC(c->heavy_eoff.ensure(items + 1));
        RC(c->heavy_foff.ensure(items + 1));
        c->list_cap = items;
    }
    RC(c->counts.ensure(16));
    RC(c->heavy_meta.ensure(kHeavyMeta));
    s->lists = c->lists.p;
    s->capacity = c->list_cap;
    s->counts = c->counts.p;
    s->heavy_unit_off = c->heavy_unit_off.p;
    s->heavy_eoff = c->heavy_eoff.p;
    s->heavy_foff = c->heavy_foff.p;
    s->heavy_epre = c->heavy_epre.p;
    s->heavy_eb0 = c->heavy_eb0.p;
    s->heavy_meta = c->heavy_meta.p;
    s->pool = c->pool.p;
    return SPNNZ_OK;
}

// The interval heavy path needs B's rows sorted and at most kMaxIntervals
// column intervals (B.cols <= 2^27).
bool interval_path(const spnnz_gpu_ctx* c) {
    return c->b_intervals && c->b_sorted && interval_geometry(c->b_cols).count <= kMaxIntervals;
}

// Buffers of one heavy batch (see heavy.cu); the merge-bitmap pool is zeroed
// when (re)allocated and returned to zero by the heavy path after each use.
int heavy_buffers(spnnz_gpu_ctx* c, int64_t count, int64_t ents, int64_t products,
                  int64_t cells, SymScratch* s) {
    const HeavyGeometry geo = heavy_geometry(c->b_cols);
    RC(c->heavy_epre.ensure(ents));
    RC(c->heavy_eb0.ensure(ents));
    s->heavy_epre = c->heavy_epre.p;
    s->heavy_eb0 = c->heavy_eb0.p;
    // unit -> (item, first entry) map, written by k_heavy_entries
    const int64_t units = products / kHeavyUnitProducts + count;
    RC(c->heavy_unit_item.ensure(units));
    RC(c->heavy_unit_e0.ensure(units));
    s->heavy_unit_item = c->heavy_unit_item.p;
    s->heavy_unit_e0 = c->heavy_unit_e0.p;
    if (interval_path(c)) {
        const int64_t tasks = count * int64_t(interval_geometry(c->b_cols).count);
        RC(c->heavy_boff.ensure(count + 1));
        RC(c->heavy_bnd.ensure(std::max<int64_t>(cells, 1)));
        RC(c->heavy_tasks.ensure(2 * std::max<int64_t>(tasks, 1)));
        s->heavy_boff = c->heavy_boff.p;
        s->heavy_bnd = c->heavy_bnd.p;
        s->heavy_bnd_cap = cells;
        s->heavy_tasks = c->heavy_tasks.p;
        s->heavy_task_cap = tasks;
        return SPNNZ_OK;
    }
    s->heavy_boff = nullptr;
    if (geo.ranges > 1) {
        RC(c->heavy_rc.ensure(count * geo.ranges));
        RC(c->heavy_cur.ensure(count * geo.ranges));
        RC(c->heavy_pbuf.ensure(products));
        if (geo.unit_sorted)
            RC(c->heavy_utab.ensure((products / kHeavyUnitProducts + count) * (geo.ranges + 1)));
    }
    const int64_t tasks = heavy_task_bound(count, products, geo.ranges);
    RC(c->heavy_tasks.ensure(2 * tasks));
    const int64_t words = int64_t(geo.wwords);
    const int64_t slots = heavy_slot_bound(count, products);
    if (c->pool_words != words || slots > c->pool_slots) {
        c->pool.release();
        RC(c->pool.ensure(slots * words));
        CU(cudaMemsetAsync(c->pool.p, 0, sizeof(uint32_t) * slots * words, c->stream));
        c->pool_slots = slots;
        c->pool_words = words;
    }
    s->heavy_rc = c->heavy_rc.p;
    s->heavy_cur = c->heavy_cur.p;
    s->heavy_pbuf = c->heavy_pbuf.p;
    s->heavy_utab = c->heavy_utab.p;
    s->heavy_tasks = c->heavy_tasks.p;
    s->heavy_task_cap = tasks;
    s->pool = c->pool.p;
    RC(c->heavy_slot_item.ensure(std::max<int64_t>(slots, 1)));
    s->heavy_slot_item = c->heavy_slot_item.p;

    return SPNNZ_OK;
}

// Symbolic pass over items (sampled rows or all local rows).  Adds the
// total into totals[slot] (device); per-item results to out (device, nullable).
// early (bin_stream set): the binning runs on bin_stream while the FLOP pass
// (already queued on c->stream, ending in c->ev_flop) is still running, so
// the host learns the heavy count without waiting for it; the tiers wait for
// the FLOP pass and the heavy batches queue behind it on c->stream -- no
// host round trip between the FLOP pass and the symbolic work.
// The heavy rows are the long pole of the call when their products exceed
// ~0.43x the FLOP pass's A entries (the heavy chain runs at ~100 G products/s,
// the pass at ~240 G entries/s); the products come from the sizes known in
// advance, else from the previous call on the same matrices.
bool heavy_long_pole(const spnnz_gpu_ctx* c, const spnnz_gpu_ctx::HeavySizes* known) {
    int64_t hp = -1;
    if (known) hp = known->products;
    else if (c->hc_valid && c->hc_epoch == c->epoch) hp = c->hc.products;
    return hp >= 0 && hp * 7 > int64_t(3) * std::max<int64_t>(c->a.nnz, 1);
}

int run_symbolic(spnnz_gpu_ctx* c, const int32_t* d_rows, int64_t n_items, int64_t* d_out,
                 int slot, bool sampled_flop, int64_t* launches, const int64_t* item_flop = nullptr,
                 const DevCsr* a_view = nullptr, const int64_t* window = nullptr,
                 cudaStream_t bin_stream = nullptr, const int64_t* tsize = nullptr,
                 long long tsize_cap = 0, const spnnz_gpu_ctx::HeavySizes* known = nullptr) {
    const bool early = bin_stream != nullptr;
    cudaStream_t bs = early ? bin_stream : c->stream;
    SymScratch s;
    RC(sym_scratch(c, n_items, &s));
    SymArgs g;
    g.a = a_view ? *a_view : c->a;
    g.brpt = c->b_rpt.p;
    g.bcol = c->b_col.p;
    g.bcols = c->b_cols;
    g.row_lo = a_view ? 0 : c->row_lo;
    g.flop = c->flop.p;
    g.item_flop = item_flop;
    g.rows = d_rows;
    g.n_items = n_items;
    g.out = d_out;
    g.totals = c->totals.p;
    g.total_slot = slot;
    g.sampled_flop = sampled_flop;
    g.window = window;
    g.tsize = tsize;
    g.tsize_cap = tsize_cap;
    g.mp_max = c->mp_max;
    g.mp_part = c->mp_part;
    CU(cudaMemsetAsync(c->counts.p, 0, sizeof(int32_t) * 16, bs));
    CU(cudaMemsetAsync(c->heavy_meta.p, 0, sizeof(long long) * kHeavyMeta, bs));
    if (n_items == 0) return SPNNZ_OK;
    CU(launch_sym_bin(g, s, bs));
    // The host learns the heavy rows' number (bin counts) while the tier
    // kernels run on side streams; the heavy batches then run on the main
    // stream concurrently with the tiers, joined at the end.
    CU(cudaEventRecord(c->fork, bs));
    CU(cudaMemcpyAsync(c->h_counts, c->counts.p, sizeof(int32_t) * 16, cudaMemcpyDeviceToHost, bs));
    CU(cudaMemcpyAsync(c->h_meta, c->heavy_meta.p, sizeof(long long) * kHeavyMeta, cudaMemcpyDeviceToHost, bs));
    if (early) CU(cudaEventRecord(c->ev_bin, bs));
    // Early mode (the FLOP pass queued before): which symbolic work runs
    // beside the pass.  When the heavy rows are the long pole (their products
    // above ~0.43 x the pass's A entries: the heavy chain runs at ~100 G
    // products/s, the pass at ~240 G entries/s) the heavy batches start right
    // after the binning and the tiers wait for the pass (config 2: step 430 ->
    // 404 us); otherwise the tiers start beside the pass and the heavy chain
    // follows it (config 5: 2819 -> 2793 us; heavy beside there: 2885).  The
    // heavy products come from the sizes known in advance (repeated draws),
    // else from the previous call on the same matrices.
    const bool heavy_long = heavy_long_pole(c, tsize ? nullptr : known);
    const bool tiers_beside = c->tiers_beside >= 0 ? c->tiers_beside > 0 : !heavy_long;
    const bool heavy_beside_pol = c->heavy_beside >= 0 ? c->heavy_beside > 0 : heavy_long;
    for (int i = 0; i < spnnz_gpu_ctx::kSide; ++i) {
        CU(cudaStreamWaitEvent(c->side[i], c->fork, 0));
        if (early && !tiers_beside) CU(cudaStreamWaitEvent(c->side[i], c->ev_flop, 0));
    }
    CU(launch_sym_tiers(g, s, c->num_sms, c->side));
    for (int i = 0; i < spnnz_gpu_ctx::kSide; ++i) CU(cudaEventRecord(c->join[i], c->side[i]));
    if (c->dbg_t) for (int i = 0; i < spnnz_gpu_ctx::kSide; ++i) CU(cudaEventRecord(c->dbg_ev[2 + i], c->side[i]));
    *launches += g.mp_max > kBin5Max ? 7 : 6;
    c->observed_set = true;  // the counts land in h_counts / h_meta by the call's end
    if (known && !tsize) {
        // sizes known in advance: no wait for the binning
        if (early) CU(cudaStreamWaitEvent(c->stream, c->fork, 0));  // heavy batches: after the bin
    } else if (early) {
        CU(cudaEventSynchronize(c->ev_bin));             // bin + the two small copies only
        CU(cudaStreamWaitEvent(c->stream, c->fork, 0));  // heavy batches: after the bin
    } else {
        CU(cudaStreamSynchronize(c->stream));  // bin + the two small copies
    }
    if (tsize && c->h_meta[kMetaCapacity] > 0) {  // symbolic.hpp:37-40
        for (int i = 0; i < spnnz_gpu_ctx::kSide; ++i) CU(cudaStreamWaitEvent(c->stream, c->join[i], 0));
        return set_err(SPNNZ_EINVAL, "HashAccumulator: tsize %lld exceeds capacity %lld",
                       static_cast<long long>(c->h_meta[kMetaCapacity]), tsize_cap);
    }
    const bool iv_path = interval_path(c);
    const int64_t heavy = known && !tsize ? known->count : c->h_counts[kHeavyBin];
    if (heavy > 0) {
        // One batch when the heavy rows fit the batch budgets (always for
        // sampled passes); exact passes over every row split the heavy list
        // greedily.  Budgets: products (bucket paths' product buffer) and
        // boundary-table cells (interval path).
        int64_t kBudget = int64_t(1) << 28;  // products per batch (1 GB buffer)
        if (const char* env = getenv("SPNNZ_HEAVY_BATCH_PRODUCTS"))  // test knob
            if (atoll(env) > 0) kBudget = atoll(env);
        const int64_t kCellBudget = kBudget;
        const bool iv = iv_path;
        struct Batch {
            int64_t first, count, ents, products, cells;
        };
        std::vector<Batch> batches{{0, heavy, c->h_meta[1], c->h_meta[2], iv ? c->h_meta[5] : 0}};
        if (known && !tsize) batches[0] = Batch{0, heavy, known->ents, known->products, known->cells};
        if (batches[0].products > kBudget || batches[0].cells > kCellBudget) {
            RC(c->heavy_flops.ensure(3 * heavy));
            CU(launch_heavy_flops(g, s, heavy, c->heavy_flops.p, c->stream));
            std::vector<int64_t> h(static_cast<size_t>(3 * heavy));
            CU(cudaMemcpyAsync(h.data(), c->heavy_flops.p, 8 * h.size(), cudaMemcpyDeviceToHost, c->stream));
            CU(cudaStreamSynchronize(c->stream));
            batches.clear();
            Batch b{0, 0, 0, 0, 0};
            for (int64_t i = 0; i < heavy; ++i) {
                const int64_t f = h[i], L = h[heavy + i], cl = iv ? h[2 * heavy + i] : 0;
                if (b.count > 0 && (b.products + f > kBudget || b.cells + cl > kCellBudget)) {
                    batches.push_back(b);
                    b = Batch{i, 0, 0, 0, 0};
                }
                ++b.count;
                b.ents += L + 1;
                b.products += f;
                b.cells += cl;
            }
            batches.push_back(b);
        }
        // beside: the heavy batches start on their own stream right after the
        // binning (early mode), concurrently with the FLOP pass
        const bool hb = early && heavy_beside_pol;
        cudaStream_t hs = hb ? c->hstream : c->stream;
        if (hb) CU(cudaStreamWaitEvent(hs, c->fork, 0));
        for (const Batch& b : batches) {
            RC(heavy_buffers(c, b.count, b.ents, b.products, b.cells, &s));
            CU(launch_sym_heavy(g, s, iv, b.first, b.count, c->num_sms, hs, launches,
                                c->pending_upload ? nullptr : c->fstream, c->ev_bin, c->ev_flop,
                                hb && c->heavy_beside == 2 ? c->ev_gate : nullptr));
        }
        if (hb) {
            CU(cudaEventRecord(c->ev_hdone, hs));
            CU(cudaStreamWaitEvent(c->stream, c->ev_hdone, 0));
        }
        if (c->dbg_t) CU(cudaEventRecord(c->dbg_ev[6], hs));
    }
    for (int i = 0; i < spnnz_gpu_ctx::kSide; ++i) CU(cudaStreamWaitEvent(c->stream, c->join[i], 0));
    return SPNNZ_OK;
}

// Degree tables of >= 8 M rows (16 MB) are gathered without L1 allocation.
bool flop_gather_nol1(const spnnz_gpu_ctx* c) {
    bool v = !c->rows_mode && c->b_rows >= (int32_t(1) << 23);
    if (const char* e = getenv("SPNNZ_FLOP_NOL1")) v = atoi(e) > 0;  // A/B knob
    return v;
}

// FLOP pass of the local rows into `out` (default: the resident profile).
int flop_pass_impl(spnnz_gpu_ctx* c, int64_t* launches, cudaStream_t stream, const PredOut& pred,
                   DBuf<int64_t>* out);
int flop_pass(spnnz_gpu_ctx* c, int64_t* launches, cudaStream_t stream = nullptr,
              const PredOut& pred = PredOut(), DBuf<int64_t>* out = nullptr) {
    const int rc = flop_pass_impl(c, launches, stream, pred, out);
    c->flop_kernel = last_flop_kernel();
    return rc;
}

int flop_pass_impl(spnnz_gpu_ctx* c, int64_t* launches, cudaStream_t stream, const PredOut& pred,
                   DBuf<int64_t>* out) {
    if (!stream) stream = c->stream;
    if (!out) out = &c->flop;
    const DevCsr& a = c->a;
    const int64_t tiles = flop_tiles(a);
    RC(out->ensure(std::max<int64_t>(a.rows, 1)));
    RC(c->tile_x.ensure(tiles + 1));
    RC(c->tile_carry.ensure(tiles + 1));
    RC(c->tile_total.ensure(tiles + 1));
    RC(c->tile_max.ensure(tiles + 1));
    RC(c->deg.ensure(int64_t(c->b_rows) + 8));  // + padding: shared-memory copies read 16-byte words
    FlopScratch s{c->tile_x.p, c->tile_carry.p, c->tile_total.p, c->tile_max.p};
    if (!c->flop_sched.p) {
        RC(c->flop_sched.ensure(2));
        CU(cudaMemsetAsync(c->flop_sched.p, 0, 2 * sizeof(unsigned long long), stream));
    }
    FlopMode mode;
    mode.sched = c->flop_sched.p;
    mode.b_rows = c->b_rows;
    mode.rows_mode = c->rows_mode;
    mode.num_sms = c->num_sms;
    if (const char* e = getenv("SPNNZ_FLOP_SMEM")) mode.no_smem = atoi(e) == 0;  // A/B knob
    mode.gather_nol1 = flop_gather_nol1(c);
    if (const char* e = getenv("SPNNZ_RB_PERSIST")) mode.rb_persistent = atoi(e) > 0;  // A/B knob
    // row mode: L2-prefetch the columns one wave (8 blocks x SMs) ahead
    mode.prefetch_ahead = c->rows_mode ? 8 * c->num_sms : 0;
    if (const char* e = getenv("SPNNZ_FLOP_PREFETCH")) mode.prefetch_ahead = atoi(e);  // A/B knob
    if (c->pending_upload && stream == c->stream) {
        // B.col still landing: degrees and the partition need only B.rpt; the
        // tiles of each chunk run on fstream as soon as the chunk is in; the
        // fixup and everything after wait for all of it
        CU(cudaStreamWaitEvent(c->stream, c->ev_rpt, 0));
        int64_t nk = 0;
        CU(launch_degree(c->b_rpt.p, c->b_rows, c->deg.p, c->num_sms, stream, &a, &s, &nk));
        CU(cudaEventRecord(c->ev_fdone, stream));
        CU(cudaStreamWaitEvent(c->fstream, c->ev_fdone, 0));
        int64_t t_prev = 0;
        const int64_t first_tile = a.base / kFlopTile;
        for (int k = 0; k < c->n_chunks; ++k) {
            int64_t t_end = c->chunk_tile_end[k] >= a.base + a.nnz
                                ? tiles
                                : c->chunk_tile_end[k] / kFlopTile - first_tile;
            t_end = std::max<int64_t>(std::min<int64_t>(t_end, tiles), t_prev);
            if (k + 1 == c->n_chunks) t_end = tiles;
            CU(cudaStreamWaitEvent(c->fstream, c->ev_chunk[k], 0));
            if (t_end > t_prev)
                CU(launch_flop_tiles(a, c->deg.p, c->b_rpt.p, s, out->p, t_prev, t_end, c->fstream, pred,
                                     mode));
            t_prev = t_end;
        }
        CU(cudaEventRecord(c->ev_fdone, c->fstream));
        CU(cudaStreamWaitEvent(c->stream, c->ev_fdone, 0));
        RC(settle_upload(c));
        CU(launch_flop_fixup(a, s, out->p, c->totals.p, stream, pred));
        *launches += a.rows ? nk + 1 + c->n_chunks : 0;
        return SPNNZ_OK;
    }
    // row blocks (one warp per 32 rows, no partition / fixup) when B is small
    // enough for their shared degree table (config 4: 65.5 us, the tile groups
    // 78.8) or A is banded (config 3: 121 us, row-mode tiles 135)
    bool rb = (!mode.no_smem && flop_rb_smem_fits(c->b_rows)) || c->rows_mode;
    if (const char* e = getenv("SPNNZ_FLOP_RB")) rb = atoi(e) > 0;  // A/B knob
    if (rb) {
        int64_t nk = 0;
        RC(c->deg_escapes.ensure(1));
        if (c->esc_epoch != c->epoch) {  // k_degree only ever raises the flag for the same B
            CU(cudaMemsetAsync(c->deg_escapes.p, 0, sizeof(unsigned), stream));
            c->esc_epoch = c->epoch;
        }
        CU(launch_degree(c->b_rpt.p, c->b_rows, c->deg.p, c->num_sms, stream, nullptr, nullptr, &nk,
                         c->deg_escapes.p));
        CU(launch_flop_rows(a, c->deg.p, c->b_rpt.p, out->p, c->totals.p, stream, pred, mode, c->deg_escapes.p));
        *launches += a.rows ? nk + 1 : 0;
        return SPNNZ_OK;
    }
    int64_t nk = 0;
    CU(launch_degree(c->b_rpt.p, c->b_rows, c->deg.p, c->num_sms, stream, &a, &s, &nk));
    CU(launch_flop(a, c->deg.p, c->b_rpt.p, s, out->p, c->totals.p, stream, pred, mode));
    *launches += a.rows ? nk + 2 : 0;
    return SPNNZ_OK;
}

// Sum of totals[first, first + count) (default: F, f*, z*, Z) and, with_max,
// the max of totals[kMax] across ranks -- ONE NCCL all-reduce: a SUM over a
// world x kTotals table in which each rank fills its own row (an all-gather
// of 8 x world int64), then the sums and the max are taken on the device.
int allreduce_totals(spnnz_gpu_ctx* c, int first = 0, int count = 4, bool with_max = true) {
    if (!c->comm) return SPNNZ_OK;
    RC(c->totals_table.ensure(int64_t(c->world) * kTotals));
    CU(launch_totals_spread(c->totals.p, c->totals_table.p, c->rank, c->world, c->stream));
    NC(nccl().AllReduce(c->totals_table.p, c->totals_table.p, size_t(c->world) * kTotals, ncclInt64, ncclSum,
                        c->comm, c->stream));
    CU(launch_totals_finish(c->totals.p, c->totals_table.p, c->world, first, count, with_max, c->stream));
    return SPNNZ_OK;
}

int read_totals(spnnz_gpu_ctx* c) {
    CU(cudaMemcpyAsync(c->h_totals, c->totals.p, sizeof(long long) * kTotals,
                       cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    return SPNNZ_OK;
}

int sample_count(int32_t num_rows, double fraction, int64_t cap, int64_t* n, double* p) {
    if (num_rows < 1) return set_err(SPNNZ_EINVAL, "make_sample_plan: M must be >= 1");
    if (cap < 0) cap = INT64_MAX;
    // predict.hpp:39-45
    int64_t k = static_cast<int64_t>(std::ceil(fraction * num_rows));
    k = std::min(k, cap);
    k = std::max<int64_t>(k, 1);
    *n = k;
    *p = static_cast<double>(k) / static_cast<double>(num_rows);
    return SPNNZ_OK;
}

void fill_report(spnnz_report* r, const long long* t, int64_t n, double p, uint64_t seed) {
    r->total_flop = t[kF];
    r->max_flop_row = t[kMax];
    r->sample_num = n;
    r->p = p;
    r->seed = seed;
    r->sampled_flop = t[kFStar];
    r->sampled_nnz = t[kZStar];
    r->sampled_cr = spnnz_sampled_cr(t[kFStar], t[kZStar]);
    r->z1_star = static_cast<double>(t[kZStar]) / p;  // predict.hpp:98 (p > 0 by construction)
    spnnz_predict_proposed(t[kFStar], t[kZStar], t[kF], &r->z2_star, &r->predicted_cr);
}

void ev_record(spnnz_gpu_ctx* c, int i) {
    // (inside a graph capture the timing events become external event-record
    // nodes, so a replayed graph still reports its phases)
    if (c->profiling)
        cudaEventRecordWithFlags(c->ev[i], c->stream, c->capturing ? cudaEventRecordExternal : cudaEventRecordDefault);
}

// last_ms: [0] FLOP pass (fused: + predict) [1] sampler (+ sampled-row FLOP)
// [2] symbolic [3] all-reduce(s) [4] predict pass (fused: 0)
void ev_collect(spnnz_gpu_ctx* c) {
    if (!c->profiling) return;
    cudaEventSynchronize(c->ev[5]);
    float m[5] = {0, 0, 0, 0, 0};
    for (int i = 0; i < 5; ++i) cudaEventElapsedTime(&m[i], c->ev[i], c->ev[i + 1]);
    if (c->ev_order == 0) {
        for (int i = 0; i < 5; ++i) c->last_ms[i] = m[i];
    } else {
        c->last_ms[0] = m[3];
        c->last_ms[1] = m[0];
        c->last_ms[2] = m[1];
        c->last_ms[3] = m[2] + m[4];
        c->last_ms[4] = 0.0;
    }
}

// The sampled rows this rank counts, and their FLOP.  Multi-GPU with C = A*A:
// every rank holds all of A (it is the replicated B), so the sampled rows are
// split by position in the sample list -- a random order, hence an even share
// of the heavy rows per rank -- instead of by row ownership (R-MAT's hub rows
// all sit in rank 0's shard); their FLOP comes straight from A and B.rpt.
// Otherwise the whole list, with the resident profile (or, fused, the same
// direct FLOP restricted to the shard).
struct SampleShare {
    const int32_t* rows = nullptr;
    int64_t n = 0;
    const int64_t* item_flop = nullptr;
    const int64_t* window = nullptr;  // device [lo, hi) of the items this rank counts
    DevCsr full;
    bool use_full = false;
};

int sample_share(spnnz_gpu_ctx* c, const int32_t* d_rows, int64_t n, bool need_flop,
                 SampleShare* sh, int64_t* launches, cudaStream_t stream = nullptr) {
    if (!stream) stream = c->stream;
    sh->rows = d_rows;
    sh->n = n;
    const bool split = c->world > 1 && c->same_b;
    if (split) {
        // every rank holds all of A (it is the replicated B): each derives the
        // FLOP of the whole list and counts a contiguous FLOP-balanced window
        sh->full.rows = c->b_rows;
        sh->full.cols = c->b_cols;
        sh->full.rpt = c->b_rpt.p;
        sh->full.col = c->b_col.p;
        sh->full.base = 0;
        sh->full.nnz = c->b_nnz;
        sh->use_full = true;
        need_flop = true;
    }
    if (need_flop) {
        RC(c->item_flop.ensure(std::max<int64_t>(sh->n, 1)));
        RC(c->item_units.ensure(sh->n + 1));
        CU(launch_item_flop(sh->use_full ? sh->full : c->a, c->b_rpt.p, sh->use_full ? 0 : c->row_lo,
                            sh->rows, sh->n, c->item_flop.p, c->item_units.p, c->num_sms, stream));
        *launches += 3;
        sh->item_flop = c->item_flop.p;
    }
    if (split && sh->n > 0) {
        RC(c->item_window.ensure(2));
        CU(launch_flop_window(c->item_flop.p, sh->n, c->rank, c->world, c->item_window.p, stream));
        ++*launches;
        sh->window = c->item_window.p;
    }
    return SPNNZ_OK;
}

// Small problems: the whole sampled symbolic pass as one kernel
// (launch_sym_small) when no row can leave bin 2 -- the resident profile is
// this context's own for the loaded matrices (a repeated call: the same
// matrices give the same max) and its max FLOP is at most kBin2Max -- on one
// rank.  A/B knob SPNNZ_SYM_SMALL=0.
bool small_path(const spnnz_gpu_ctx* c) {
    const char* e = getenv("SPNNZ_SYM_SMALL");
    if (e && atoi(e) == 0) return false;
    return c->world == 1 && c->profile_valid && c->profile_own && c->profile_max <= kBin3Max;
}

int run_small(spnnz_gpu_ctx* c, const int32_t* d_rows, int64_t n, bool draw, uint64_t seed, cudaStream_t stream,
              int64_t* launches) {
    SymArgs g;
    g.a = c->a;
    g.brpt = c->b_rpt.p;
    g.bcol = c->b_col.p;
    g.bcols = c->b_cols;
    g.row_lo = c->row_lo;
    g.flop = c->flop.p;
    g.rows = d_rows;
    g.n_items = n;
    g.out = nullptr;
    g.totals = c->totals.p;
    g.total_slot = kZStar;
    g.sampled_flop = true;
    // items above bin 2 (a block each) on a side stream beside the warps'
    const bool two = c->profile_max > kBin2Max;
    cudaStream_t sb = two ? c->side[1] : nullptr;
    if (two) {
        CU(cudaEventRecord(c->fork, stream));
        CU(cudaStreamWaitEvent(sb, c->fork, 0));
    }
    CU(launch_sym_small(g, seed, c->a_rows, draw, c->samples.p, c->num_sms, stream, sb));
    *launches += two ? 2 : 1;
    if (two) {
        CU(cudaEventRecord(c->join[1], sb));
        CU(cudaStreamWaitEvent(stream, c->join[1], 0));
    }
    // no heavy rows by construction: the call's observed heavy sizes are zero
    c->h_counts[kHeavyBin] = 0;
    c->observed_set = true;
    c->used_small = true;
    return SPNNZ_OK;
}

// Pipeline body shared by run_prediction and run_prediction_with_plan:
// FLOP pass -> sampler -> sampled symbolic -> one all-reduce -> predict pass.
// Default schedule (inputs resident): the sampler, the sampled rows' FLOP
// (and on multi-GPU their FLOP-balanced window) and the binning run on a side
// stream underneath the FLOP pass; the host reads the heavy count meanwhile
// and queues the symbolic tiers and heavy batches behind the pass (see
// run_symbolic's early mode).  While B is still landing from the host
// (chunked upload) the FLOP pass goes first and the rest follows it.
// With c->fused (SPNNZ_FUSED_PREDICT=1) the sampled rows' FLOP
// is derived directly so the symbolic pass and CR come first, and one FLOP
// pass writes every row's flop together with its prediction (two
// all-reduces on multi-GPU).  Measured slower on B200 at config 5 (the
// per-row division and scattered 8-byte stores land in the gather-bound FLOP
// kernel: 2.12 ms vs 1.85 + 0.07 ms), so it is not the default.
int pipeline(spnnz_gpu_ctx* c, const int32_t* d_rows, int64_t n, bool draw, uint64_t seed,
             int64_t* d_ceil, double* d_real, const spnnz_gpu_ctx::HeavySizes* known = nullptr) {
    int64_t launches = 0;
    const char* fenv = getenv("SPNNZ_FUSED_PREDICT");
    c->fused = fenv && atoi(fenv) > 0;
    CU(cudaMemsetAsync(c->totals.p, 0, sizeof(long long) * kTotals, c->stream));
    SampleShare sh;
    if (!c->fused) {
        ev_record(c, 0);
        // the sampler and the rank's sampled-row FLOP / window need only A,
        // B.rpt and the seed: they run on a side stream under the FLOP pass
        // (latency-bound small kernels, off the critical path)
        // (not while B is still landing from the host: the sampled rows read it)
        const bool beside = !c->pending_upload;
        cudaStream_t ss = beside ? c->side[0] : c->stream;
        if (beside) {
            // the FLOP pass is queued first (the GPU starts it while the host
            // queues the side-stream work), the side stream forks before it
            CU(cudaEventRecord(c->fork, c->stream));
            CU(cudaStreamWaitEvent(ss, c->fork, 0));
        }
        const bool small = small_path(c);
        c->dbg_t = !c->capturing && getenv("SPNNZ_DEBUG_TIMELINE") != nullptr;
        if (c->dbg_t) {
            for (auto& e : c->dbg_ev)
                if (!e) cudaEventCreate(&e);
            CU(cudaEventRecord(c->dbg_ev[0], c->stream));
        }
        RC(flop_pass(c, &launches));
        if (c->dbg_t) CU(cudaEventRecord(c->dbg_ev[1], c->stream));
        if (beside) {
            CU(cudaEventRecord(c->ev_flop, c->stream));
            CU(cudaEventRecord(c->ev_gate, c->stream));
        }
        if (small) {
            // draw + FLOP + count in one kernel beside the FLOP pass; with
            // rows above bin 2, two kernels after the pass (they read this
            // call's profile to pick each item's kernel)
            if (beside && c->profile_max > kBin2Max) CU(cudaStreamWaitEvent(ss, c->ev_flop, 0));
            RC(run_small(c, d_rows, n, draw, seed, ss, &launches));
            // phases: the FLOP pass ends at ev 1; ev 2 -> 3 is the symbolic
            // kernels' remainder after it (the join)
            ev_record(c, 1);
            ev_record(c, 2);
            if (beside) {
                CU(cudaEventRecord(c->join[0], ss));
                CU(cudaStreamWaitEvent(c->stream, c->join[0], 0));
            }
        } else {
        if (draw) {
            CU(launch_sample(seed, c->a_rows, n, c->samples.p, ss));
            ++launches;
        }
        // The sampled rows' FLOP: on one rank the binning reads the resident
        // profile after the pass (the pass's grid leaves no room beside it
        // anyway: deriving it directly only added three
        // kernels after the pass); multi-GPU splits the list by FLOP, which
        // sample_share derives directly from A and B.rpt
        // ... except when the heavy rows are the long pole (run_symbolic's
        // policy): their chain then starts beside the pass (config 2: 435 ->
        // 402 us with the direct FLOP; configs 3 / 4: 148 -> 144, 139 -> 130 us
        // from the profile)
        const char* ie = getenv("SPNNZ_ITEM_FLOP");  // A/B knob: 1 / 0 = always / never directly on one rank
        bool direct = c->world > 1 || heavy_long_pole(c, known);
        if (ie) direct = c->world > 1 || atoi(ie) > 0;
        direct = direct && beside;
        RC(sample_share(c, d_rows, n, direct, &sh, &launches, ss));
        if (beside && !sh.item_flop) CU(cudaStreamWaitEvent(ss, c->ev_flop, 0));
        ev_record(c, 1);
        ev_record(c, 2);
        RC(run_symbolic(c, sh.rows, sh.n, nullptr, kZStar, true, &launches, sh.item_flop,
                        sh.use_full ? &sh.full : nullptr, sh.window, beside ? ss : nullptr, nullptr, 0,
                        known));
        }
        if (c->dbg_t) {
            CU(cudaEventRecord(c->dbg_ev[7], c->stream));
            CU(cudaEventSynchronize(c->dbg_ev[7]));
            float t[8] = {};
            for (int i = 1; i < 8; ++i) cudaEventElapsedTime(&t[i], c->dbg_ev[0], c->dbg_ev[i]);
            fprintf(stderr, "timeline us: flop %.1f tiers %.1f %.1f %.1f %.1f heavy %.1f join %.1f\n", 1e3 * t[1],
                    1e3 * t[2], 1e3 * t[3], 1e3 * t[4], 1e3 * t[5], 1e3 * t[6], 1e3 * t[7]);
            heavy_debug_print(c->dbg_ev[0]);
            c->dbg_t = false;
        }
        ev_record(c, 3);
        RC(allreduce_totals(c));
        ev_record(c, 4);
        if (d_ceil || d_real) {
            CU(launch_predict(c->flop.p, local_rows(c), c->totals.p, 0.0, d_ceil, d_real, c->num_sms,
                              c->stream));
            ++launches;
        }
        ev_record(c, 5);
        c->ev_order = 0;
    } else {
        RC(settle_upload(c));  // the symbolic pass reads B first here
        ev_record(c, 0);
        if (draw) {
            CU(launch_sample(seed, c->a_rows, n, c->samples.p, c->stream));
            ++launches;
        }
        RC(sample_share(c, d_rows, n, true, &sh, &launches));
        ev_record(c, 1);
        RC(run_symbolic(c, sh.rows, sh.n, nullptr, kZStar, true, &launches, sh.item_flop,
                        sh.use_full ? &sh.full : nullptr, sh.window, nullptr, nullptr, 0, known));
        ev_record(c, 2);
        RC(allreduce_totals(c, kFStar, 2, false));  // f*, z*: CR is known everywhere
        ev_record(c, 3);
        PredOut pred;
        pred.totals = c->totals.p;
        pred.ceil = d_ceil;
        pred.real = d_real;
        if (pred.on()) {
            pred.redo_cap = std::min<int64_t>(std::max(local_rows(c), 1), int64_t(1) << 16);
            RC(c->redo.ensure(pred.redo_cap));
            RC(c->nredo.ensure(1));
            CU(cudaMemsetAsync(c->nredo.p, 0, sizeof(unsigned long long), c->stream));
            pred.redo = c->redo.p;
            pred.nredo = c->nredo.p;
        }
        RC(flop_pass(c, &launches, c->stream, pred));
        if (pred.on()) {
            CU(launch_predict_redo(c->flop.p, local_rows(c), pred, c->num_sms, c->stream));
            ++launches;
        }
        ev_record(c, 4);
        RC(allreduce_totals(c, kF, 1, true));  // F, max
        ev_record(c, 5);
        c->ev_order = 1;
    }
    c->profile_valid = true;
    c->profile_own = true;
    c->last_launches = launches;
    return SPNNZ_OK;
}

// run_prediction_with_plan (predict.hpp:202-216) on the RESIDENT profile --
// the reference takes the profile as an argument and runs no FLOP pass:
// sampled symbolic (tsize = the profile's flop), f* from the profile,
// F = profile.total_flop, one all-reduce of {f*, z*}, the per-row views of
// the profile's flop.
int pipeline_profile(spnnz_gpu_ctx* c, const int32_t* d_rows, int64_t n, int64_t* d_ceil,
                     double* d_real, const spnnz_gpu_ctx::HeavySizes* known = nullptr, bool draw = false,
                     uint64_t seed = 0) {
    int64_t launches = 0;
    RC(settle_upload(c));
    const bool small = small_path(c);
    if (draw && !small) {  // the plan drawn on the device into d_rows (= c->samples)
        CU(launch_sample(seed, c->a_rows, n, c->samples.p, c->stream));
        ++launches;
    }
    // (a graph of this call re-reads h_init: it holds this profile's values
    // until the profile changes, which also drops the graph)
    for (int i = 0; i < kTotals; ++i) c->h_init[i] = 0;
    c->h_init[kF] = c->profile_total;
    c->h_init[kMax] = c->profile_max;
    CU(cudaMemcpyAsync(c->totals.p, c->h_init, sizeof(long long) * kTotals, cudaMemcpyHostToDevice,
                       c->stream));
    const int64_t* item_flop = nullptr;
    if (!c->profile_own && n > 0) {
        // bin by each sampled row's true FLOP; the profile is the table size
        RC(c->item_flop.ensure(n));
        RC(c->item_units.ensure(n + 1));
        CU(launch_item_flop(c->a, c->b_rpt.p, c->row_lo, d_rows, n, c->item_flop.p, c->item_units.p,
                            c->num_sms, c->stream));
        launches += 3;
        item_flop = c->item_flop.p;
    }
    ev_record(c, 0);
    ev_record(c, 1);
    ev_record(c, 2);
    if (small)
        RC(run_small(c, d_rows, n, draw, seed, c->stream, &launches));
    else
        RC(run_symbolic(c, d_rows, n, nullptr, kZStar, true, &launches, item_flop, nullptr, nullptr,
                        nullptr, c->profile_own ? nullptr : c->flop.p, c->profile_max, known));
    ev_record(c, 3);
    RC(allreduce_totals(c, kFStar, 2, false));  // f*, z*; F and max are the profile's
    ev_record(c, 4);
    if (d_ceil || d_real) {
        CU(launch_predict(c->flop.p, local_rows(c), c->totals.p, 0.0, d_ceil, d_real, c->num_sms,
                          c->stream));
        ++launches;
    }
    ev_record(c, 5);
    c->ev_order = 0;
    c->last_launches = launches;
    return SPNNZ_OK;
}

}  // namespace

extern "C" {

int spnnz_gpu_abi_version(void) { return SPNNZ_GPU_ABI_VERSION; }

const char* spnnz_gpu_last_error(void) { return g_err.c_str(); }

int spnnz_gpu_nccl_unique_id(void* id128) {
    Nccl& n = nccl();
    if (!n.loaded) return set_err(SPNNZ_ENCCL, "NCCL unavailable: %s", n.why.c_str());
    ncclUniqueId id;
    NC(n.GetUniqueId(&id));
    std::memcpy(id128, &id, sizeof id);
    return SPNNZ_OK;
}

int spnnz_gpu_create(int device, int rank, int world, const void* nccl_id, spnnz_gpu_ctx** out) {
    if (!out) return set_err(SPNNZ_EINVAL, "null out");
    *out = nullptr;
    if (world < 1 || rank < 0 || rank >= world)
        return set_err(SPNNZ_EINVAL, "bad rank %d / world %d", rank, world);
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0)
        return set_err(SPNNZ_ECUDA, "no CUDA device: %s", cudaGetErrorString(e));
    if (device < 0 || device >= ndev) return set_err(SPNNZ_EINVAL, "bad device %d", device);
    CU(cudaSetDevice(device));
    cudaDeviceProp prop;
    CU(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
        return set_err(SPNNZ_ECUDA, "device %d is sm_%d%d; this build targets sm_100a", device,
                       prop.major, prop.minor);
    auto* c = new spnnz_gpu_ctx;
    c->device = device;
    c->rank = rank;
    c->world = world;
    c->num_sms = prop.multiProcessorCount;
    // stream priorities (A/B knob SPNNZ_STREAM_PRIO): 1 = main stream (FLOP,
    // heavy rows) above the symbolic side streams, 2 = the reverse
    int prio_main = 0, prio_side = 0;
    if (const char* pe = getenv("SPNNZ_STREAM_PRIO")) {
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        if (atoi(pe) == 1) prio_main = hi, prio_side = lo;
        if (atoi(pe) == 2) prio_main = lo, prio_side = hi;
    }
    e = cudaStreamCreateWithPriority(&c->stream, cudaStreamNonBlocking, prio_main);
    if (e == cudaSuccess) e = cudaMallocHost(&c->h_totals, sizeof(long long) * kTotals);
    if (e == cudaSuccess) e = cudaMallocHost(&c->h_counts, sizeof(int32_t) * 16);
    if (e == cudaSuccess) e = cudaMallocHost(&c->h_meta, sizeof(long long) * kHeavyMeta);
    if (e == cudaSuccess) e = cudaMallocHost(&c->h_init, sizeof(long long) * kTotals);
    for (int i = 0; i < 6 && e == cudaSuccess; ++i) e = cudaEventCreate(&c->ev[i]);
    for (int i = 0; i < spnnz_gpu_ctx::kSide && e == cudaSuccess; ++i)
        e = cudaStreamCreateWithPriority(&c->side[i], cudaStreamNonBlocking, prio_side);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->cstream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->fstream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->hstream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_hdone, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_gate, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_rpt, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_fdone, cudaEventDisableTiming);
    for (int i = 0; i < spnnz_gpu_ctx::kChunks && e == cudaSuccess; ++i)
        e = cudaEventCreateWithFlags(&c->ev_chunk[i], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->fork, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_bin, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_flop, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_in, cudaEventDisableTiming);
    for (int i = 0; i < spnnz_gpu_ctx::kSide && e == cudaSuccess; ++i)
        e = cudaEventCreateWithFlags(&c->join[i], cudaEventDisableTiming);
    int rc = SPNNZ_OK;
    if (e != cudaSuccess) rc = set_err(SPNNZ_ECUDA, "create: %s", cudaGetErrorString(e));
    if (rc == SPNNZ_OK) rc = c->totals.ensure(kTotals);
    // Without an id a shard is detached: no communicator, totals stay
    // rank-local and the caller combines them (sharding checks on one GPU).
    // A one-rank communicator is allowed (it exercises the NCCL path).
    if (rc == SPNNZ_OK && nccl_id) {
        Nccl& n = nccl();
        if (!n.loaded) {
            rc = set_err(SPNNZ_ENCCL, "NCCL unavailable: %s", n.why.c_str());
        } else {
            ncclUniqueId id;
            std::memcpy(&id, nccl_id, sizeof id);
            ncclResult_t r = n.CommInitRank(&c->comm, world, id, rank);
            if (r != ncclSuccess)
                rc = set_err(SPNNZ_ENCCL, "ncclCommInitRank: %s", n.GetErrorString(r));
        }
    }
    if (rc != SPNNZ_OK) {
        spnnz_gpu_destroy(c);
        return rc;
    }
    *out = c;
    return SPNNZ_OK;
}

int spnnz_gpu_destroy(spnnz_gpu_ctx* c) {
    if (!c) return SPNNZ_OK;
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    if (c->cstream) cudaStreamSynchronize(c->cstream);
    if (c->fstream) cudaStreamSynchronize(c->fstream);
    if (c->hstream) cudaStreamSynchronize(c->hstream);
    if (c->comm) nccl().CommDestroy(c->comm);
    // device buffers: the DBuf members free themselves in `delete c` below
    // (the device is already selected)
    if (c->h_totals) cudaFreeHost(c->h_totals);
    if (c->h_counts) cudaFreeHost(c->h_counts);
    if (c->h_meta) cudaFreeHost(c->h_meta);
    if (c->h_init) cudaFreeHost(c->h_init);
    if (c->gexec) cudaGraphExecDestroy(c->gexec);
    if (c->fgexec) cudaGraphExecDestroy(c->fgexec);
    for (auto& e : c->ev)
        if (e) cudaEventDestroy(e);
    for (int i = 0; i < spnnz_gpu_ctx::kSide; ++i) {
        if (c->side[i]) cudaStreamDestroy(c->side[i]);
        if (c->join[i]) cudaEventDestroy(c->join[i]);
    }
    if (c->fork) cudaEventDestroy(c->fork);
    if (c->ev_bin) cudaEventDestroy(c->ev_bin);
    if (c->ev_flop) cudaEventDestroy(c->ev_flop);
    if (c->ev_in) cudaEventDestroy(c->ev_in);
    for (auto ev : c->ev_chunk)
        if (ev) cudaEventDestroy(ev);
    if (c->ev_rpt) cudaEventDestroy(c->ev_rpt);
    if (c->ev_fdone) cudaEventDestroy(c->ev_fdone);
    if (c->cstream) cudaStreamDestroy(c->cstream);
    if (c->fstream) cudaStreamDestroy(c->fstream);
    if (c->hstream) cudaStreamDestroy(c->hstream);
    if (c->ev_hdone) cudaEventDestroy(c->ev_hdone);
    if (c->ev_gate) cudaEventDestroy(c->ev_gate);
    if (c->stream) cudaStreamDestroy(c->stream);
    delete c;
    return SPNNZ_OK;
}

int spnnz_gpu_synchronize(spnnz_gpu_ctx* c) {
    RC(check_ctx(c, false));
    CU(cudaStreamSynchronize(c->stream));
    return SPNNZ_OK;
}

void* spnnz_gpu_stream(spnnz_gpu_ctx* c) { return c ? c->stream : nullptr; }

int spnnz_gpu_set_input_stream(spnnz_gpu_ctx* c, void* stream) {
    if (!c) return set_err(SPNNZ_EINVAL, "null context");
    c->in_stream = static_cast<cudaStream_t>(stream);
    return SPNNZ_OK;
}

int spnnz_gpu_host_alloc(size_t bytes, void** out) {
    cudaError_t e = cudaMallocHost(out, std::max<size_t>(bytes, 1));
    if (e != cudaSuccess) return set_err(SPNNZ_ENOMEM, "cudaMallocHost: %s", cudaGetErrorString(e));
    return SPNNZ_OK;
}

int spnnz_gpu_host_free(void* p) {
    if (p) cudaFreeHost(p);
    return SPNNZ_OK;
}

int spnnz_gpu_partition_rows(const int64_t* rpt, int32_t rows, int world, int32_t* bounds) {
    if (!rpt || !bounds || world < 1 || rows < 0)
        return set_err(SPNNZ_EINVAL, "partition_rows: bad arguments");
    // balanced on nnz + rows: a row costs about what an entry does (its flop
    // written, its offsets read, its prediction written vs one column read and
    // one degree gather), and R-MAT's empty tail rows would otherwise pile
    // onto the last rank (5.1 M of 16.8 M rows at N = 8 by nnz alone)
    const int64_t work = rpt[rows] - rpt[0] + rows;
    bounds[0] = 0;
    for (int r = 1; r < world; ++r) {
        const int64_t target = work / world * r + work % world * r / world;
        int64_t lo = 0, hi = rows;  // first i with (rpt[i] - rpt[0]) + i >= target
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (rpt[mid] - rpt[0] + mid < target) lo = mid + 1; else hi = mid;
        }
        int32_t b = static_cast<int32_t>(lo);
        b = std::max(b, bounds[r - 1]);
        bounds[r] = std::min(b, rows);
    }
    bounds[world] = rows;
    return SPNNZ_OK;
}

int spnnz_gpu_load(spnnz_gpu_ctx* c, const spnnz_csr_view* a, const spnnz_csr_view* b,
                   int residency) {
    RC(check_ctx(c, false));
    if (!a || a->rows < 0 || a->cols < 0) return set_err(SPNNZ_EINVAL, "load: bad A");
    const bool same = (b == nullptr || b == a ||
                       (b->rpt == a->rpt && b->col == a->col && b->rows == a->rows &&
                        b->cols == a->cols));
    const spnnz_csr_view* bv = same ? a : b;
    if (bv->rows < 0 || bv->cols < 0) return set_err(SPNNZ_EINVAL, "load: bad B");
    if (!a->rpt || !bv->rpt) return set_err(SPNNZ_EINVAL, "load: null rpt");
    c->loaded = false;
    c->profile_valid = false;
    c->profile_own = false;
    ++c->epoch;
    ++c->profile_gen;
    c->hc_valid = false;
    c->same_b = same;
    c->a_rows = a->rows;
    c->a_cols = a->cols;
    c->b_rows = bv->rows;
    c->b_cols = bv->cols;

    // Shard bounds need A.rpt on the host.
    std::vector<int64_t> host_arpt;
    const int64_t* arpt_h = a->rpt;
    if (residency == SPNNZ_DEVICE) {
        RC(order_after_caller(c));
        host_arpt.resize(static_cast<size_t>(a->rows) + 1);
        CU(cudaMemcpy(host_arpt.data(), a->rpt, 8 * host_arpt.size(), cudaMemcpyDeviceToHost));
        arpt_h = host_arpt.data();
    }
    std::vector<int32_t> bounds(static_cast<size_t>(c->world) + 1);
    RC(spnnz_gpu_partition_rows(arpt_h, a->rows, c->world, bounds.data()));
    c->row_lo = bounds[c->rank];
    c->row_hi = bounds[c->rank + 1];
    const auto kind = residency == SPNNZ_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;

    // B replicated (it is also A's storage when C = A*A).
    int64_t b_nnz = 0;
    if (residency == SPNNZ_DEVICE) {
        CU(cudaMemcpy(&b_nnz, bv->rpt + bv->rows, 8, cudaMemcpyDeviceToHost));
    } else {
        b_nnz = bv->rpt[bv->rows];
    }
    c->b_nnz = b_nnz;
    RC(c->b_rpt.ensure(int64_t(bv->rows) + 1));
    RC(c->b_col.ensure(std::max<int64_t>(b_nnz, 1) + kColPad));
    const bool chunked = residency == SPNNZ_HOST && same && b_nnz >= (int64_t(1) << 24);
    c->n_chunks = 0;
    if (!chunked) {
        CU(cudaMemcpyAsync(c->b_rpt.p, bv->rpt, 8 * (size_t(bv->rows) + 1), kind, c->stream));
        if (b_nnz) CU(cudaMemcpyAsync(c->b_col.p, bv->col, 4 * size_t(b_nnz), kind, c->stream));
    } else {
        // copy stream: B.rpt, then B.col in kChunks pieces (cut at FLOP-tile
        // multiples), one event each; the main stream waits on them lazily
        CU(cudaEventRecord(c->ev_rpt, c->stream));  // after whatever the main stream holds
        CU(cudaStreamWaitEvent(c->cstream, c->ev_rpt, 0));
        CU(cudaMemcpyAsync(c->b_rpt.p, bv->rpt, 8 * (size_t(bv->rows) + 1), kind, c->cstream));
        CU(cudaEventRecord(c->ev_rpt, c->cstream));
        int64_t prev = 0;
        for (int k = 0; k < spnnz_gpu_ctx::kChunks; ++k) {
            int64_t end = b_nnz * (k + 1) / spnnz_gpu_ctx::kChunks;
            end = k + 1 == spnnz_gpu_ctx::kChunks ? b_nnz : (end / kFlopTile) * kFlopTile;
            if (end > prev)
                CU(cudaMemcpyAsync(c->b_col.p + prev, bv->col + prev, 4 * size_t(end - prev), kind,
                                   c->cstream));
            CU(cudaEventRecord(c->ev_chunk[k], c->cstream));
            c->chunk_tile_end[k] = end;  // absolute entry end; tiles resolved per shard below
            prev = end;
        }
        c->n_chunks = spnnz_gpu_ctx::kChunks;
        c->pending_upload = true;
    }

    DevCsr v;
    v.rows = c->row_hi - c->row_lo;
    v.cols = a->cols;
    const int64_t a_lo = arpt_h[c->row_lo], a_hi = arpt_h[c->row_hi];
    v.nnz = a_hi - a_lo;
    v.base = a_lo;
    if (same) {
        v.rpt = c->b_rpt.p + c->row_lo;
        v.col = c->b_col.p;
    } else {
        RC(c->a_rpt.ensure(int64_t(v.rows) + 1));
        RC(c->a_col.ensure(std::max<int64_t>(v.nnz, 1) + kColPad));
        CU(cudaMemcpyAsync(c->a_rpt.p, a->rpt + c->row_lo, 8 * (size_t(v.rows) + 1), kind,
                           c->stream));
        if (v.nnz)
            CU(cudaMemcpyAsync(c->a_col.p, a->col + a_lo, 4 * size_t(v.nnz), kind, c->stream));
        v.rpt = c->a_rpt.p;
        v.col = c->a_col.p - a_lo;  // indexed with absolute offsets
    }
    c->a = v;
    // Banded A (consecutive rows reach consecutive columns): sampled pairs of
    // consecutive rows of the shard; on the host for host views, else by a
    // small kernel (the device path synchronizes here anyway)
    {
        int st[3] = {0, 0, 0};
        const int32_t lo = c->row_lo, hi = c->row_hi;
        if (hi - lo >= 2) {
            if (residency == SPNNZ_HOST) {
                for (int i = 0; i < kLocalitySamples; ++i) {
                    const int32_t r = lo + static_cast<int32_t>((int64_t(hi - lo - 1) * i) / kLocalitySamples);
                    const int64_t p0 = a->rpt[r], p1 = a->rpt[r + 1], p2 = a->rpt[r + 2];
                    if (p1 > p0 && p2 > p1) {
                        ++st[0];
                        const int d = a->col[p1] - a->col[p0];
                        st[1] += d >= 0 && d <= 2;
                        st[2] += p1 - p0 <= 64;
                    }
                }
            } else {
                RC(c->bad.ensure(3));
                CU(launch_locality(a->rpt, a->col, lo, hi, kLocalitySamples, c->bad.p, c->stream));
                CU(cudaMemcpyAsync(st, c->bad.p, sizeof(st), cudaMemcpyDeviceToHost, c->stream));
                CU(cudaStreamSynchronize(c->stream));
            }
        }
        c->rows_mode = banded_rows(st[0], st[1], st[2]);
        c->tiers_beside = -1;
        if (const char* e = getenv("SPNNZ_TIERS_BESIDE")) c->tiers_beside = atoi(e) > 0;  // A/B knob
        c->mp_max = kMpMaxDefault;
        if (const char* e = getenv("SPNNZ_MP_MAX")) c->mp_max = atoll(e);  // A/B knob
        c->mp_part = kMpPart;
        if (const char* e = getenv("SPNNZ_MP_PART")) c->mp_part = std::max<long long>(1, atoll(e));  // test knob
        c->heavy_beside = -1;
        if (const char* e = getenv("SPNNZ_HEAVY_BESIDE")) c->heavy_beside = atoi(e);  // A/B knob (2: sort beside, runs after the pass)
        if (const char* e = getenv("SPNNZ_FLOP_ROWS")) c->rows_mode = atoi(e) > 0;  // A/B knob
    }
    // The interval heavy path (opt-in, SPNNZ_HEAVY_INTERVALS=1) needs B's rows
    // sorted -- the reference's CsrMatrix invariant, checked here once.
    const char* ivenv = getenv("SPNNZ_HEAVY_INTERVALS");
    c->b_intervals = ivenv && atoi(ivenv) > 0;
    c->b_sorted = false;
    if (c->b_intervals) {
        // B may still be landing on the copy stream (chunked upload)
        RC(settle_upload(c));
        RC(c->sorted_cnt.ensure(2));
        CU(launch_check_sorted(c->b_rpt.p, c->b_col.p, c->b_rows, b_nnz,
                               reinterpret_cast<unsigned long long*>(c->sorted_cnt.p), c->num_sms,
                               c->stream));
        long long cnt[2] = {0, 0};
        CU(cudaMemcpyAsync(cnt, c->sorted_cnt.p, sizeof(cnt), cudaMemcpyDeviceToHost, c->stream));
        CU(cudaStreamSynchronize(c->stream));
        c->b_sorted = cnt[0] == cnt[1];
    }
    c->loaded = true;
    return SPNNZ_OK;
}

int spnnz_gpu_shard(spnnz_gpu_ctx* c, int32_t* lo, int32_t* hi, int32_t* rows) {
    RC(check_ctx(c, true, false));  // host-side facts only
    if (lo) *lo = c->row_lo;
    if (hi) *hi = c->row_hi;
    if (rows) *rows = c->a_rows;
    return SPNNZ_OK;
}

int spnnz_gpu_compute_flop(spnnz_gpu_ctx* c, int64_t* flop_out, int residency, int64_t* total,
                           int64_t* max) {
    RC(check_ctx(c));
    RC(dims_ok(c, "compute_flop"));
    int64_t launches = 0;
    const int m = local_rows(c);
    const auto body = [&]() -> int {
        CU(cudaMemsetAsync(c->totals.p, 0, sizeof(long long) * kTotals, c->stream));
        RC(flop_pass(c, &launches));
        RC(allreduce_totals(c));
        if (flop_out && m) {
            CU(cudaMemcpyAsync(flop_out, c->flop.p, 8 * size_t(m),
                               residency == SPNNZ_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                               c->stream));
        }
        return SPNNZ_OK;
    };
    // a repeated pass on the same matrices and output replays one CUDA graph
    // (host-side launch cost of the memset, the kernels and the copy, ~35 ->
    // ~20 us per call on small matrices); no NCCL inside graphs
    const char* genv = getenv("SPNNZ_GRAPH");
    const bool graphable = !c->pending_upload && !c->comm && !(genv && atoi(genv) == 0);
    if (graphable && c->fgexec && c->fg_epoch == c->epoch && c->fg_out == flop_out && c->fg_res == residency) {
        CU(cudaGraphLaunch(c->fgexec, c->stream));
        launches = c->fg_launches;
    } else if (graphable && c->fg_epoch == c->epoch && c->fg_res == -2) {
        // second pass on these matrices: capture it
        cudaGraph_t graph = nullptr;
        bool ran = false;
        if (cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeRelaxed) == cudaSuccess) {
            c->capturing = true;
            const int rc = body();
            c->capturing = false;
            const cudaError_t ce = cudaStreamEndCapture(c->stream, &graph);
            if (rc == SPNNZ_OK && ce == cudaSuccess && graph) {
                // the previous matrices' executable graph is updated in place
                // when the topology allows (a new shape, same kernels), else
                // re-instantiated
                cudaError_t ie = cudaErrorUnknown;
                if (c->fgexec) {
                    cudaGraphExecUpdateResultInfo info;
                    ie = cudaGraphExecUpdate(c->fgexec, graph, &info);
                    if (ie != cudaSuccess) {
                        cudaGetLastError();
                        cudaGraphExecDestroy(c->fgexec);
                        c->fgexec = nullptr;
                    }
                }
                if (!c->fgexec) ie = cudaGraphInstantiate(&c->fgexec, graph, 0);
                if (ie == cudaSuccess) {
                    c->fg_out = flop_out;
                    c->fg_res = residency;
                    c->fg_launches = launches;
                    CU(cudaGraphLaunch(c->fgexec, c->stream));
                    ran = true;
                } else {
                    c->fgexec = nullptr;
                }
            }
            if (graph) cudaGraphDestroy(graph);
        }
        cudaGetLastError();
        if (!ran) {
            launches = 0;
            RC(body());
        }
    } else {
        RC(body());
        c->fg_epoch = c->epoch;
        c->fg_res = -2;  // seen once: the next call on these matrices is captured
    }
    RC(read_totals(c));
    c->profile_valid = true;
    c->profile_own = true;
    ++c->profile_gen;
    c->profile_total = c->h_totals[kF];
    c->profile_max = c->h_totals[kMax];
    if (total) *total = c->profile_total;
    if (max) *max = c->profile_max;
    c->last_launches = launches;
    return SPNNZ_OK;
}

int spnnz_gpu_set_profile(spnnz_gpu_ctx* c, const int64_t* flop_in, int64_t rows, int residency,
                          int64_t total, int64_t max) {
    RC(check_ctx(c, false));
    if (!c->loaded) {
        // profile-only mode (sampled_flop / predict_row_structure need no matrices)
        if (rows < 0 || rows > INT32_MAX) return set_err(SPNNZ_EINVAL, "bad profile length");
        c->a_rows = static_cast<int32_t>(rows);
        c->row_lo = 0;
        c->row_hi = static_cast<int32_t>(rows);
    }
    if (rows != local_rows(c))
        return set_err(SPNNZ_EINVAL, "symbolic: profile does not match A");
    RC(c->flop.ensure(std::max<int64_t>(rows, 1)));
    if (residency == SPNNZ_DEVICE) RC(order_after_caller(c));
    if (rows)
        CU(cudaMemcpyAsync(c->flop.p, flop_in, 8 * size_t(rows),
                           residency == SPNNZ_DEVICE ? cudaMemcpyDeviceToDevice
                                                     : cudaMemcpyHostToDevice,
                           c->stream));
    c->profile_valid = true;
    c->profile_own = false;
    ++c->profile_gen;
    c->profile_total = total;
    c->profile_max = max;
    return SPNNZ_OK;
}

namespace {
int check_rows(spnnz_gpu_ctx* c, const int32_t* rows, int64_t n, int residency, const char* who,
               const int32_t** d_rows) {
    if (n < 0) return set_err(SPNNZ_EINVAL, "%s: negative count", who);
    if (n > 0 && !rows) return set_err(SPNNZ_EINVAL, "%s: null rows", who);
    if (residency == SPNNZ_HOST) {
        for (int64_t i = 0; i < n; ++i)
            if (rows[i] < 0 || rows[i] >= c->a_rows)
                return set_err(SPNNZ_EINVAL, "%s: row %d out of range", who, rows[i]);
    } else if (n > 0) {
        RC(order_after_caller(c));
        RC(c->bad.ensure(1));
        CU(cudaMemsetAsync(c->bad.p, 0, 4, c->stream));
        CU(launch_check_rows(rows, n, c->a_rows, c->bad.p, c->stream));
        int32_t bad = 0;
        CU(cudaMemcpyAsync(&bad, c->bad.p, 4, cudaMemcpyDeviceToHost, c->stream));
        CU(cudaStreamSynchronize(c->stream));
        if (bad) return set_err(SPNNZ_EINVAL, "%s: %d rows out of range", who, bad);
    }
    return stage_in(c, rows, n, residency, c->rows_in, d_rows);
}
}  // namespace

int spnnz_gpu_sampled_flop(spnnz_gpu_ctx* c, const int32_t* rows, int64_t n, int residency,
                           int64_t* out) {
    RC(check_ctx(c, false));
    if (!c->profile_valid) return set_err(SPNNZ_ESTATE, "sampled_flop: no resident profile");
    const int32_t* d_rows = nullptr;
    RC(check_rows(c, rows, n, residency, "sampled_flop", &d_rows));
    CU(cudaMemsetAsync(c->totals.p, 0, sizeof(long long) * kTotals, c->stream));
    CU(launch_sampled_flop(c->flop.p, c->row_lo, local_rows(c), d_rows, n, c->totals.p, c->stream));
    RC(allreduce_totals(c));
    RC(read_totals(c));
    *out = c->h_totals[kFStar];
    return SPNNZ_OK;
}

int spnnz_gpu_make_sample_plan(spnnz_gpu_ctx* c, int32_t num_rows, uint64_t seed, double fraction,
                               int64_t cap, int32_t* rows, int residency, int64_t* n, double* p) {
    RC(sample_count(num_rows, fraction, cap, n, p));
    if (!rows) return SPNNZ_OK;
    RC(check_ctx(c, false));
    int32_t* dst = rows;
    if (residency == SPNNZ_HOST) {
        RC(c->samples.ensure(*n));
        dst = c->samples.p;
    }
    CU(launch_sample(seed, num_rows, *n, dst, c->stream));
    if (residency == SPNNZ_HOST)
        CU(cudaMemcpyAsync(rows, dst, 4 * size_t(*n), cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    return SPNNZ_OK;
}

int spnnz_gpu_sampled_symbolic(spnnz_gpu_ctx* c, const int32_t* rows, int64_t n, int residency,
                               int64_t* per_sample, int64_t* total) {
    RC(check_ctx(c));
    if (c->a_cols != c->b_rows) return set_err(SPNNZ_EINVAL, "symbolic: A.cols != B.rows");
    if (!c->profile_valid) return set_err(SPNNZ_ESTATE, "sampled_symbolic: no resident profile");
    const int32_t* d_rows = nullptr;
    RC(check_rows(c, rows, n, residency, "sampled_symbolic", &d_rows));
    int64_t* d_out = nullptr;
    if (per_sample) {
        if (residency == SPNNZ_DEVICE) {
            d_out = per_sample;
        } else {
            RC(c->out64.ensure(n));
            d_out = c->out64.p;
        }
    }
    int64_t launches = 0;
    CU(cudaMemsetAsync(c->totals.p, 0, sizeof(long long) * kTotals, c->stream));
    const int64_t* item_flop = nullptr;
    if (!c->profile_own && n > 0) {  // caller profile: bin by true FLOP, profile = tsize
        RC(c->item_flop.ensure(n));
        RC(c->item_units.ensure(n + 1));
        CU(launch_item_flop(c->a, c->b_rpt.p, c->row_lo, d_rows, n, c->item_flop.p, c->item_units.p,
                            c->num_sms, c->stream));
        launches += 3;
        item_flop = c->item_flop.p;
    }
    RC(run_symbolic(c, d_rows, n, d_out, kZStar, false, &launches, item_flop, nullptr, nullptr,
                    nullptr, c->profile_own ? nullptr : c->flop.p, c->profile_max));
    RC(allreduce_totals(c));
    if (per_sample && residency == SPNNZ_HOST && n)
        CU(cudaMemcpyAsync(per_sample, d_out, 8 * size_t(n), cudaMemcpyDeviceToHost, c->stream));
    RC(read_totals(c));
    *total = c->h_totals[kZStar];
    c->last_launches = launches;
    return SPNNZ_OK;
}

int spnnz_gpu_exact_symbolic(spnnz_gpu_ctx* c, int64_t* per_row, int residency, int64_t* total) {
    RC(check_ctx(c));
    if (c->a_cols != c->b_rows) return set_err(SPNNZ_EINVAL, "symbolic: A.cols != B.rows");
    if (!c->profile_valid) return set_err(SPNNZ_ESTATE, "exact_symbolic: no resident profile");
    const int m = local_rows(c);
    int64_t* d_out = nullptr;
    if (per_row) {
        if (residency == SPNNZ_DEVICE) {
            d_out = per_row;
        } else {
            RC(c->out64.ensure(m));
            d_out = c->out64.p;
        }
    }
    int64_t launches = 0;
    CU(cudaMemsetAsync(c->totals.p, 0, sizeof(long long) * kTotals, c->stream));
    const int64_t* item_flop = nullptr;
    if (!c->profile_own && m > 0) {  // caller profile: bin by true FLOP, profile = tsize
        RC(flop_pass(c, &launches, c->stream, PredOut(), &c->flop_true));
        item_flop = c->flop_true.p;
    }
    RC(run_symbolic(c, nullptr, m, d_out, kZ, false, &launches, item_flop, nullptr, nullptr,
                    nullptr, c->profile_own ? nullptr : c->flop.p, c->profile_max));
    RC(allreduce_totals(c));
    if (per_row && residency == SPNNZ_HOST && m)
        CU(cudaMemcpyAsync(per_row, d_out, 8 * size_t(m), cudaMemcpyDeviceToHost, c->stream));
    RC(read_totals(c));
    *total = c->h_totals[kZ];
    c->last_launches = launches;
    return SPNNZ_OK;
}

namespace {
int predict_view(spnnz_gpu_ctx* c, double cr, int64_t* out_ceil, double* out_real, int residency,
                 const char* who) {
    RC(check_ctx(c, false));
    if (!(cr > 0.0)) return set_err(SPNNZ_EINVAL, "%s: predicted_cr must be positive", who);
    if (!c->profile_valid) return set_err(SPNNZ_ESTATE, "%s: no resident profile", who);
    const int m = local_rows(c);
    if ((!out_ceil && !out_real) || m == 0) return SPNNZ_OK;
    int64_t* d_ceil = out_ceil;
    double* d_real = out_real;
    if (residency == SPNNZ_HOST) {
        if (out_ceil) {
            RC(c->out64.ensure(m));
            d_ceil = c->out64.p;
        } else {
            RC(c->outf.ensure(m));
            d_real = c->outf.p;
        }
    }
    CU(launch_predict(c->flop.p, m, nullptr, cr, d_ceil, d_real, c->num_sms, c->stream));
    if (residency == SPNNZ_HOST)
        CU(cudaMemcpyAsync(out_ceil ? static_cast<void*>(out_ceil) : static_cast<void*>(out_real),
                           out_ceil ? static_cast<void*>(d_ceil) : static_cast<void*>(d_real),
                           8 * size_t(m), cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    return SPNNZ_OK;
}
}  // namespace

int spnnz_gpu_predict_row_structure(spnnz_gpu_ctx* c, double cr, double* out, int residency) {
    return predict_view(c, cr, nullptr, out, residency, "predict_row_structure");
}

int spnnz_gpu_predict_row_structure_ceil(spnnz_gpu_ctx* c, double cr, int64_t* out,
                                         int residency) {
    return predict_view(c, cr, out, nullptr, residency, "predict_row_structure_ceil");
}

namespace {
// Heavy sizes the device reported for the call that just completed.
spnnz_gpu_ctx::HeavySizes observed_sizes(const spnnz_gpu_ctx* c) {
    spnnz_gpu_ctx::HeavySizes o;
    if (!c->observed_set) return o;
    o.count = c->h_counts[kHeavyBin];
    if (o.count > 0) {
        o.ents = c->h_meta[1];
        o.products = c->h_meta[2];
        o.cells = interval_path(c) ? c->h_meta[5] : 0;
    }
    return o;
}

int run_common(spnnz_gpu_ctx* c, const int32_t* d_rows, int64_t n, double p, bool draw,
               uint64_t seed, spnnz_report* rep, int64_t* row_ceil, double* row_real,
               int residency, bool with_profile = false, bool redo = false) {
    const int m = local_rows(c);
    int64_t* d_ceil = row_ceil;
    double* d_real = row_real;
    if (residency == SPNNZ_HOST) {
        if (row_ceil) {
            RC(c->out64.ensure(m));
            d_ceil = c->out64.p;
        }
        if (row_real) {
            RC(c->outf.ensure(m));
            d_real = c->outf.p;
        }
    }
    if (!m) d_ceil = nullptr, d_real = nullptr;
    const char* fenv = getenv("SPNNZ_FUSED_PREDICT");
    const bool fused = !with_profile && fenv && atoi(fenv) > 0;
    // heavy sizes known in advance?  (a) no row can be heavy: the resident
    // profile is this context's own for the loaded matrices and its max fits
    // bin 5 (for run_prediction the pass recomputes the same profile);
    // (b) the same draw ran before on the same matrices
    using HS = spnnz_gpu_ctx::HeavySizes;
    const HS zero{};
    const HS* known = nullptr;
    if (redo) {
    } else if (c->profile_valid && c->profile_own && c->profile_max <= kBin5Max) known = &zero;
    else if (draw && c->hc_valid && c->hc_epoch == c->epoch && c->hc_seed == seed && c->hc_n == n) known = &c->hc;
    if (known && (known->products > (int64_t(1) << 28) || known->cells > (int64_t(1) << 28))) known = nullptr;
    if (const char* e = getenv("SPNNZ_HEAVY_BATCH_PRODUCTS"))  // test knob: batch planning needs the sync
        if (atoll(e) > 0) known = nullptr;
    const HS known_v = known ? *known : HS{};

    // a whole sync-free call runs as one CUDA graph, captured on first use
    // and replayed while its key holds (no NCCL in graphs, no profiling events)
    spnnz_gpu_ctx::GraphKey key;
    key.kind = with_profile ? 1 : 0;
    key.epoch = c->epoch;
    key.profile_gen = with_profile ? c->profile_gen : 0;
    key.seed = draw ? seed : 0;
    key.n = n;
    key.rows = draw ? nullptr : d_rows;
    key.ceil = d_ceil;
    key.real = d_real;
    key.fused = fused;
    key.profiling = c->profiling;
    const char* genv = getenv("SPNNZ_GRAPH");
    const bool graphable = known && !c->pending_upload && !c->comm && !(genv && atoi(genv) == 0);
    c->observed_set = false;
    c->used_small = false;
    if (graphable && c->gexec && c->gkey == key && c->g_known == known_v) {
        if (c->g_small) c->h_counts[kHeavyBin] = 0;  // (no copy of the bin counts in that graph)
        CU(cudaGraphLaunch(c->gexec, c->stream));
        c->last_launches = c->g_launches;
        c->observed_set = n > 0;
        if (!with_profile) {
            c->profile_valid = true;
            c->profile_own = true;
        }
    } else {
        bool ran = false;
        if (graphable) {
            // capture on first use (buffers a first call must size are
            // allocated during the relaxed-mode capture) and launch; a capture
            // that fails for any reason falls back to the eager call below.
            // The executable graph is updated in place when the topology
            // allows (a new key with the same kernels), else re-instantiated.
            cudaGraph_t graph = nullptr;
            cudaError_t be = cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeRelaxed);
            int rc = SPNNZ_ECUDA;
            cudaError_t ce = be;
            if (be == cudaSuccess) {
                c->capturing = true;
                rc = with_profile ? pipeline_profile(c, d_rows, n, d_ceil, d_real, &known_v, draw, seed)
                                  : pipeline(c, d_rows, n, draw, seed, d_ceil, d_real, &known_v);
                c->capturing = false;
                ce = cudaStreamEndCapture(c->stream, &graph);
            }
            if (rc == SPNNZ_OK && ce == cudaSuccess && graph) {
                cudaError_t ie = cudaErrorUnknown;
                if (c->gexec) {
                    cudaGraphExecUpdateResultInfo info;
                    ie = cudaGraphExecUpdate(c->gexec, graph, &info);
                    if (ie != cudaSuccess) {
                        cudaGetLastError();
                        cudaGraphExecDestroy(c->gexec);
                        c->gexec = nullptr;
                    }
                }
                if (!c->gexec) ie = cudaGraphInstantiate(&c->gexec, graph, 0);
                cudaGraphDestroy(graph);
                if (ie == cudaSuccess) {
                    c->gkey = key;
                    c->g_known = known_v;
                    c->g_small = c->used_small;
                    c->g_launches = c->last_launches;
                    CU(cudaGraphLaunch(c->gexec, c->stream));
                    ran = true;
                } else {
                    if (getenv("SPNNZ_DEBUG_GRAPH"))
                        fprintf(stderr, "spnnz_gpu: graph instantiate failed: %s\n", cudaGetErrorString(ie));
                    cudaGetLastError();
                    c->gexec = nullptr;
                }
            } else {
                if (getenv("SPNNZ_DEBUG_GRAPH"))
                    fprintf(stderr, "spnnz_gpu: graph capture failed: rc %d, %s\n", rc, cudaGetErrorString(ce));
                if (graph) cudaGraphDestroy(graph);
                cudaGetLastError();
                if (c->gexec) {
                    cudaGraphExecDestroy(c->gexec);
                    c->gexec = nullptr;
                }
            }
        }
        if (!ran) {
            if (with_profile)
                RC(pipeline_profile(c, d_rows, n, d_ceil, d_real, known, draw, seed));
            else
                RC(pipeline(c, d_rows, n, draw, seed, d_ceil, d_real, known));
        }
    }
    if (residency == SPNNZ_HOST && m) {
        if (row_ceil)
            CU(cudaMemcpyAsync(row_ceil, d_ceil, 8 * size_t(m), cudaMemcpyDeviceToHost, c->stream));
        if (row_real)
            CU(cudaMemcpyAsync(row_real, d_real, 8 * size_t(m), cudaMemcpyDeviceToHost, c->stream));
    }
    RC(read_totals(c));
    const HS seen = observed_sizes(c);
    if (known && !(seen == known_v)) {
        // the advance sizes were wrong (not expected: the same draw on the same
        // matrices bins the same rows): drop them and redo the call eagerly
        c->hc_valid = false;
        if (c->gexec) {
            cudaGraphExecDestroy(c->gexec);
            c->gexec = nullptr;
        }
        if (const char* e = getenv("SPNNZ_STRICT_SIZES"))
            if (atoi(e) > 0) return set_err(SPNNZ_ECUDA, "heavy-row sizes known in advance were wrong");
        return run_common(c, d_rows, n, p, draw, seed, rep, row_ceil, row_real, residency, with_profile, true);
    }
    if (draw && !known) {
        c->hc_valid = true;
        c->hc_epoch = c->epoch;
        c->hc_seed = seed;
        c->hc_n = n;
        c->hc = seen;
    }
    ev_collect(c);
    if (!with_profile) {
        c->profile_total = c->h_totals[kF];
        c->profile_max = c->h_totals[kMax];
        ++c->profile_gen;
    }
    if (rep) fill_report(rep, c->h_totals, n, p, seed);
    return SPNNZ_OK;
}
}  // namespace

int spnnz_gpu_run_prediction(spnnz_gpu_ctx* c, uint64_t seed, double fraction, int64_t cap,
                             spnnz_report* rep, int64_t* row_ceil, double* row_real,
                             int32_t* sample_rows, int residency) {
    RC(check_ctx(c, true, false));  // the pipeline overlaps a pending upload
    RC(dims_ok(c, "compute_flop"));
    int64_t n = 0;
    double p = 0;
    RC(sample_count(c->a_rows, fraction, cap, &n, &p));
    RC(c->samples.ensure(n));
    RC(run_common(c, c->samples.p, n, p, true, seed, rep, row_ceil, row_real, residency));
    if (sample_rows)
        CU(cudaMemcpy(sample_rows, c->samples.p, 4 * size_t(n),
                      residency == SPNNZ_DEVICE ? cudaMemcpyDeviceToDevice
                                                : cudaMemcpyDeviceToHost));
    return SPNNZ_OK;
}

int spnnz_gpu_predict_sampled(spnnz_gpu_ctx* c, uint64_t seed, double fraction, int64_t cap,
                              spnnz_report* rep, int32_t* sample_rows) {
    RC(check_ctx(c));
    if (c->a_cols != c->b_rows) return set_err(SPNNZ_EINVAL, "symbolic: A.cols != B.rows");
    if (!c->profile_valid) return set_err(SPNNZ_ESTATE, "predict_sampled: no resident profile");
    int64_t n = 0;
    double p = 0;
    RC(sample_count(c->a_rows, fraction, cap, &n, &p));
    RC(c->samples.ensure(n));
    RC(run_common(c, c->samples.p, n, p, true, seed, rep, nullptr, nullptr, SPNNZ_HOST, true));
    if (sample_rows) CU(cudaMemcpy(sample_rows, c->samples.p, 4 * size_t(n), cudaMemcpyDeviceToHost));
    return SPNNZ_OK;
}

int spnnz_gpu_run_prediction_with_plan(spnnz_gpu_ctx* c, const int32_t* rows, int64_t n, double p,
                                       int rows_residency, spnnz_report* rep, int64_t* row_ceil,
                                       double* row_real, int out_residency) {
    RC(check_ctx(c));
    if (c->a_cols != c->b_rows) return set_err(SPNNZ_EINVAL, "symbolic: A.cols != B.rows");
    if (!c->profile_valid)
        return set_err(SPNNZ_ESTATE, "run_prediction_with_plan: no resident profile");
    const int32_t* d_rows = nullptr;
    RC(check_rows(c, rows, n, rows_residency, "sampled_symbolic", &d_rows));
    if (!(p > 0.0)) return set_err(SPNNZ_EINVAL, "predict_reference: p must be positive");
    return run_common(c, d_rows, n, p, false, 0, rep, row_ceil, row_real, out_residency, true);
}

// ------------------------------------------------------------ estimators
double spnnz_sampled_cr(int64_t f, int64_t z) {
    return (f > 0 && z > 0) ? static_cast<double>(f) / static_cast<double>(z) : 1.0;
}

int spnnz_predict_reference(int64_t z, double p, double* z1) {
    if (!(p > 0.0)) return set_err(SPNNZ_EINVAL, "predict_reference: p must be positive");
    *z1 = static_cast<double>(z) / p;
    return SPNNZ_OK;
}

int spnnz_predict_proposed(int64_t f, int64_t z, int64_t total_flop, double* z2, double* cr) {
    if (f <= 0 || z <= 0) {
        *cr = 1.0;
        *z2 = static_cast<double>(total_flop);
        return SPNNZ_OK;
    }
    *cr = static_cast<double>(f) / static_cast<double>(z);
    *z2 = static_cast<double>(total_flop) * static_cast<double>(z) / static_cast<double>(f);
    return SPNNZ_OK;
}

int spnnz_error_report(double z1, double z2, int64_t f_star, int64_t exact_nnz, int64_t total_flop,
                       double p, double* out4) {
    if (exact_nnz <= 0 || total_flop <= 0)
        return set_err(SPNNZ_EINVAL, "error_report: relative error undefined for Z = 0 or F = 0");
    if (!(p > 0.0)) return set_err(SPNNZ_EINVAL, "error_report: p must be positive");
    const double z = static_cast<double>(exact_nnz), f = static_cast<double>(total_flop);
    const double fs = static_cast<double>(f_star) / p;
    out4[0] = (z1 - z) / z;
    out4[1] = (fs - f) / f;
    out4[2] = (z2 - z) / z;
    out4[3] = f_star > 0 ? std::fabs(out4[2] - (out4[0] - out4[1]) / (1.0 + out4[1])) : 0.0;
    return SPNNZ_OK;
}

int spnnz_gpu_set_profiling(spnnz_gpu_ctx* c, int enabled) {
    if (!c) return set_err(SPNNZ_EINVAL, "null context");
    c->profiling = enabled != 0;
    return SPNNZ_OK;
}

int spnnz_gpu_probe_flop_floor(spnnz_gpu_ctx* c, int reps, double* stream_ms, double* gather_ms) {
    RC(check_ctx(c));
    if (reps < 1) return set_err(SPNNZ_EINVAL, "probe: reps must be >= 1");
    RC(c->deg.ensure(int64_t(c->b_rows) + 8));
    DBuf<long long> out;
    RC(out.ensure(std::max<int64_t>(std::max<int64_t>(c->a.nnz / 16, int64_t(c->num_sms) * 1024), 1)));
    CU(launch_degree(c->b_rpt.p, c->b_rows, c->deg.p, c->num_sms, c->stream));
    double* res[2] = {stream_ms, gather_ms};
    // the loads of the kernel the FLOP pass picks for this matrix: the row
    // streams' shape with its shared-memory table, else the tile kernel's
    const bool table = pattern_table_applies(c->a, c->b_rows, c->rows_mode);
    const bool nol1 = flop_gather_nol1(c);
    const auto probe = [&](bool gather) {
        return table ? launch_pattern_table(c->a, c->deg.p, c->b_rows, c->num_sms, gather, out.p, c->stream)
                     : launch_pattern(c->a, c->deg.p, gather, nol1, out.p, c->stream);
    };
    for (int g = 0; g < 2; ++g) {
        CU(probe(g == 1));  // warm-up
        CU(cudaEventRecord(c->ev[0], c->stream));
        for (int i = 0; i < reps; ++i) CU(probe(g == 1));
        CU(cudaEventRecord(c->ev[1], c->stream));
        CU(cudaEventSynchronize(c->ev[1]));
        float ms = 0;
        CU(cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]));
        if (res[g]) *res[g] = ms / reps;
    }
    return SPNNZ_OK;
}

int spnnz_gpu_check_guards(int64_t* checked, int64_t* broken) {
    CU(cudaDeviceSynchronize());
    std::lock_guard<std::mutex> lk(g_guard_mu);
    int64_t bad = g_guard_released_broken;
    for (const GuardEntry& g : g_guards) bad += band_intact(g) ? 0 : 1;
    if (checked) *checked = static_cast<int64_t>(g_guards.size()) + g_guard_released;
    if (broken) *broken = bad;
    return SPNNZ_OK;
}

const char* spnnz_gpu_last_flop_kernel(spnnz_gpu_ctx* c) { return c && c->flop_kernel ? c->flop_kernel : ""; }

int spnnz_gpu_last_timings(spnnz_gpu_ctx* c, double* ms5, int64_t* launches) {
    if (!c) return set_err(SPNNZ_EINVAL, "null context");
    if (ms5)
        for (int i = 0; i < 5; ++i) ms5[i] = c->last_ms[i];
    if (launches) *launches = c->last_launches;
    return SPNNZ_OK;
}

}  // extern "C"
