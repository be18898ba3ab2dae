// Host-side declarations of the predictor's kernel launchers (sm_100a).
// Every launcher enqueues on `stream` and returns cudaGetLastError().
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#ifdef __CUDACC__
#define SPNNZ_HD __host__ __device__
#else
#define SPNNZ_HD
#endif

namespace spnnz_gpu {

// Device view of a CSR row range.  `rpt` points at the first row's offset
// (rows + 1 entries, ABSOLUTE offsets into `col`); `col` is indexed with those
// absolute offsets.  For a shard of A that shares B's arrays (C = A*A), rpt is
// a view into B's rpt and col is B's col.
struct DevCsr {
    int32_t rows = 0;
    int32_t cols = 0;
    const int64_t* rpt = nullptr;
    const int32_t* col = nullptr;
    int64_t nnz = 0;   // rpt[rows] - rpt[0]
    int64_t base = 0;  // rpt[0] (absolute offset of the first entry), known on the host
};

// Slots of the per-call device totals array (long long[kTotals]).
enum TotalSlot : int {
    kF = 0,       // total FLOP of the (local) rows
    kFStar = 1,   // sampled FLOP f*
    kZStar = 2,   // sampled NNZ z*
    kZ = 3,       // exact NNZ Z (scoring)
    kMax = 4,     // max FLOP of a row
    kTotals = 8
};

// ---------------------------------------------------------------- FLOP
// Fixed tiles of kFlopTile nonzeros (aligned to absolute multiples of the
// tile size), one block each; a tile owns the rows that start inside it.
#ifndef SPNNZ_FLOP_BLOCK
#define SPNNZ_FLOP_BLOCK 128
#endif
constexpr int kFlopBlock = SPNNZ_FLOP_BLOCK;
#ifndef SPNNZ_FLOP_IPT
#define SPNNZ_FLOP_IPT 16
#endif
constexpr int kFlopIpt = SPNNZ_FLOP_IPT;
constexpr int kFlopTile = kFlopBlock * kFlopIpt;
static_assert((kFlopTile & (kFlopTile - 1)) == 0, "tile size is a power of two");

int64_t flop_tiles(const DevCsr& a);

struct FlopScratch {
    int32_t* tile_x = nullptr;       // tiles + 1: first owned row of each tile
    long long* tile_carry = nullptr; // tiles: sum of the leading slice (row owned earlier)
    long long* tile_total = nullptr; // tiles
    long long* tile_max = nullptr;   // tiles
};

// deg[k] = min(B.rpt[k+1] - B.rpt[k], 0xFFFF) as uint16; 0xFFFF escapes to
// B.rpt for the exact length.  Gathered under an L2 evict_last policy.
// Degree array of B and, when a and s are given, A's tile partition (fused
// into the same pass when A.rpt is a view of B.rpt); *launches counts kernels.
// escapes (nullable): set to 1 when some B row has >= 65535 entries.
cudaError_t launch_degree(const int64_t* brpt, int64_t k_rows, uint16_t* deg, int num_sms,
                          cudaStream_t stream, const DevCsr* a = nullptr, const FlopScratch* s = nullptr,
                          int64_t* launches = nullptr, unsigned* escapes = nullptr);
// Fused predict: with ceil/real set, the FLOP pass also writes
// min(flop, ceil(flop / cr)) (and flop / cr) for every row as its flop becomes
// final, cr derived on the device from totals[kFStar], totals[kZStar].
struct PredOut {
    const long long* totals = nullptr;
    int64_t* ceil = nullptr;
    double* real = nullptr;
    // rows whose quotient the reciprocal fast path could not certify
    // (ties): redone with an IEEE division by launch_predict_redo
    int32_t* redo = nullptr;
    unsigned long long* nredo = nullptr;
    int64_t redo_cap = 0;
    SPNNZ_HD bool on() const { return ceil || real; }
};
// Kernel choice of a FLOP pass.  B with few rows: its whole uint16 degree
// table sits in shared memory (persistent blocks of 8 tile groups, config 4's
// 65536 rows = 128 KB); banded A (rows_mode, checked on the host at load):
// tiles of short rows walk one row per thread over shared-staged columns.
struct FlopMode {
    int32_t b_rows = 0;
    bool rows_mode = false;
    bool no_smem = false;  // A/B knob: keep the degree table in global memory
    int prefetch_ahead = 0;  // k_flop: L2-prefetch the columns this many tiles ahead (0: off)
    // k_flop: degree gathers skip L1 allocation -- for degree tables far
    // larger than L1 with no locality to keep (config 5: -1.8 %; config 2's
    // 2 MB table gains from L1 hits: +80 % without them)
    bool gather_nol1 = false;
    unsigned long long* sched = nullptr;  // k_flop_smem's tile tickets: 2 zeroed words, left zeroed
    bool rb_persistent = true;  // k_flop_rb with L2 degrees: one wave of persistent blocks (A/B knob)
    int num_sms = 148;
};
bool flop_smem_fits(int32_t k_rows);
// Tail padding (entries) of the device A.col / B.col buffers: the row-stream
// FLOP kernel loads whole 256-entry chunks past a shard's last entry.
constexpr int64_t kColPad = 512;
// the FLOP kernel this host thread launched last (instrumentation)
const char* last_flop_kernel();
// Row-block FLOP pass (A with short rows): one warp per 32 rows over
// shared-staged columns, degree table in shared memory when B's rows fit
// (flop_rb_smem_fits); writes flop and adds F / max into totals directly (no
// partition, no fixup).  mode.sched: the smem kernel's tickets.
bool flop_rb_smem_fits(int32_t k_rows);
cudaError_t launch_flop_rows(const DevCsr& a, const uint16_t* bdeg, const int64_t* brpt, int64_t* flop,
                             long long* totals, cudaStream_t stream, const PredOut& pred, const FlopMode& mode,
                             const unsigned* escapes);
// Sampled banded-A check (n pairs of consecutive rows in [lo, hi)), rpt/col
// device arrays with absolute offsets: out3 = {pairs, advancing, short}.
cudaError_t launch_locality(const int64_t* rpt, const int32_t* col, int32_t lo, int32_t hi, int n, int* out3,
                            cudaStream_t stream);
constexpr int kLocalitySamples = 4096;
// Instrumentation: the FLOP pass's A.col stream (and, with gather, its degree
// gathers) without the row logic; out needs nnz / 16 entries.
cudaError_t launch_pattern(const DevCsr& a, const uint16_t* deg, bool gather, bool nol1, long long* out,
                           cudaStream_t stream);
// The same for the row-stream pass (degree table in shared memory): the
// shape of k_flop_rs (one 1024-thread block per SM); out needs num_sms * 1024.
bool pattern_table_applies(const DevCsr& a, int32_t k_rows, bool rows_mode);
cudaError_t launch_pattern_table(const DevCsr& a, const uint16_t* deg, int32_t k_rows, int num_sms, bool gather,
                                 long long* out, cudaStream_t stream);
// rows_mode when most sampled consecutive rows advance like a stencil's
inline bool banded_rows(int pairs, int advancing, int short_rows) {
    return pairs >= 64 && advancing * 4 >= pairs * 3 && short_rows * 20 >= pairs * 19;
}
// Redoes the rows listed by a fused FLOP pass (or every row when the list
// overflowed) with __ddiv_rn.
cudaError_t launch_predict_redo(const int64_t* flop, int64_t m, const PredOut& pred, int num_sms,
                                cudaStream_t stream);
cudaError_t launch_flop(const DevCsr& a, const uint16_t* bdeg, const int64_t* brpt,
                        const FlopScratch& s, int64_t* flop, long long* totals,
                        cudaStream_t stream, const PredOut& pred, const FlopMode& mode);
// The same in two steps: tiles [t_begin, t_end) (any order, any streams),
// then the fixup once every tile is done.
cudaError_t launch_flop_tiles(const DevCsr& a, const uint16_t* bdeg, const int64_t* brpt,
                              const FlopScratch& s, int64_t* flop, int64_t t_begin, int64_t t_end,
                              cudaStream_t stream, const PredOut& pred, const FlopMode& mode);
cudaError_t launch_flop_fixup(const DevCsr& a, const FlopScratch& s, int64_t* flop, long long* totals,
                              cudaStream_t stream, const PredOut& pred = PredOut());

// -------------------------------------------------------------- sampler
cudaError_t launch_sample(uint64_t seed, int32_t num_rows, int64_t n, int32_t* rows,
                          cudaStream_t stream);

// ------------------------------------------------------------- symbolic
// Items are either an explicit list of GLOBAL row ids (sampled mode) or all
// local rows (exact mode, rows == nullptr).  Items whose row is outside the
// shard [row_lo, row_lo + a.rows) get 0.  Rows are binned by FLOP:
constexpr int kNumBins = 8;
constexpr int64_t kBin1Max = 32;     // warp, __match_any_sync dedup
constexpr int64_t kBin2Max = 512;    // warp, 1024-slot smem hash per warp
#ifndef SPNNZ_BIN3_MAX
#define SPNNZ_BIN3_MAX 2048
#endif
#ifndef SPNNZ_BIN4_MAX
#define SPNNZ_BIN4_MAX 8192
#endif
#ifndef SPNNZ_BIN5_MAX
#define SPNNZ_BIN5_MAX 24576
#endif
constexpr int64_t kBin3Max = SPNNZ_BIN3_MAX;  // 256-thread block, 4096-slot smem hash
constexpr int64_t kBin4Max = SPNNZ_BIN4_MAX;  // 512-thread block, 16384-slot smem hash
constexpr int64_t kBin5Max = SPNNZ_BIN5_MAX;  // 1024-thread block, 49152-slot smem hash
constexpr int kHeavyBin = 6;         // heavier: units of kHeavyUnitProducts
// kBin5Max < FLOP <= SymArgs::mp_max: bin 5's block and table, the row's
// products walked in P = ceil(FLOP / kMpPart) passes, pass k inserting the
// keys whose mixed hash falls in part k (k_sym_multipass, symbolic.cu)
constexpr int kMpBin = 7;
constexpr int kForeignBin = 8;       // row owned by another rank
constexpr int kNoBin = 9;            // padding lane
#ifndef SPNNZ_MP_PART
#define SPNNZ_MP_PART 20000
#endif
constexpr int64_t kMpPart = SPNNZ_MP_PART;  // products per pass (mean): table load ~0.4
// Off by default (0: those rows take the heavy path): measured 3x slower at
// config 5 (SPNNZ_MP_MAX=98304: k_sym_multipass 922 us for 45 M products) --
// a filtered-out product saves no warp instructions while any lane of its
// warp matches, so a pass costs as much as bin 5's single pass.  Opt-in
// through the runtime knob SPNNZ_MP_MAX (read at load), kept under test.
#ifndef SPNNZ_MP_MAX
#define SPNNZ_MP_MAX 0
#endif
constexpr int64_t kMpMaxDefault = SPNNZ_MP_MAX;
// row tickets of the block tiers live in the spare bin counters (16 in all)
SPNNZ_HD constexpr int ticket_slot(int bin) { return bin == kMpBin ? 13 : 7 + bin; }
//        products, many blocks per row over a global bitmap of B.cols bits.
constexpr int64_t kHeavyUnitProducts = 4096;
// Sorted B (the interval path, heavy.cu): B's columns are cut into
// P = ceil(B.cols / 2^shift) intervals of 2^shift <= 2^kIvShift columns (one
// 64 KB shared bitmap each); a heavy row's task is a run of consecutive
// non-empty intervals with at most ~kIntervalTarget products.
constexpr int kIvShift = 19;
constexpr int kMaxIntervals = 256;  // B.cols <= 2^27; wider B takes the bucket path
constexpr int64_t kIntervalTarget = 32768;
struct Intervals {
    int shift;
    int32_t count;
};
SPNNZ_HD inline Intervals interval_geometry(int32_t bcols) {
    int lg = 5;
    while ((int64_t(1) << lg) < bcols) ++lg;  // 2^lg >= B.cols
    Intervals iv;
    iv.shift = lg < kIvShift ? lg : kIvShift;
    iv.count = static_cast<int32_t>((int64_t(bcols) + (int64_t(1) << iv.shift) - 1) >> iv.shift);
    if (iv.count < 1) iv.count = 1;
    return iv;
}

constexpr int kHeavyMeta = 16;

struct SymScratch {
    int32_t* lists = nullptr;        // kNumBins * capacity item ids
    int64_t capacity = 0;
    int32_t* counts = nullptr;       // kNumBins (+ spare) counters
    // heavy-row work decomposition (per batch of heavy items, see heavy.cu)
    int64_t* heavy_unit_off = nullptr;   // capacity + 1: product-unit prefix per item
    int64_t* heavy_eoff = nullptr;       // capacity + 1: entry-array offset per item
    int64_t* heavy_foff = nullptr;       // capacity + 1: product prefix per item
    int64_t* heavy_epre = nullptr;       // per entry: exclusive product prefix (L_i + 1 per item)
    int64_t* heavy_eb0 = nullptr;        // per entry: start of its B row
    long long* heavy_rc = nullptr;       // count * R: bucket counts, then bucket starts
    long long* heavy_cur = nullptr;      // count * R: placement cursors
    int32_t* heavy_pbuf = nullptr;       // products grouped by (item, range) or (unit, range)
    int32_t* heavy_utab = nullptr;       // units * (R + 1): range starts inside each sorted unit
    void* heavy_tasks = nullptr;         // HeavyTask[heavy_task_cap]
    int64_t heavy_task_cap = 0;
    uint32_t* pool = nullptr;            // merge bitmaps (W bits each), zero between calls
    int32_t* heavy_slot_item = nullptr;  // per merge slot: the batch item it belongs to
    long long* heavy_meta = nullptr;     // kHeavyMeta slots: [0] units [1] sum(len+1)
                                         // [2] sum(flop) of heavy rows [3] tasks [4] merge
                                         // slots used [5] sum((P-1) len) [6] sum(P) of heavy
                                         // rows (interval path) [7] interval-task cursor
                                         // [8] small tasks (stored from the list's end)
    // interval path (sorted B)
    int64_t* heavy_boff = nullptr;       // capacity + 1: boundary-table offset per item
    int32_t* heavy_bnd = nullptr;        // per item (P-1) x len: interval starts inside each B row
    int64_t heavy_bnd_cap = 0;
    int32_t* heavy_unit_item = nullptr;  // per unit: its item
    int32_t* heavy_unit_e0 = nullptr;    // per unit: the entry holding its first product
};

// Column-range geometry of the heavy path: ranges of 2^wshift bits (at most
// 2^20, a 128 KB shared bitmap), `ranges` of them cover B.cols.
struct HeavyGeometry {
    int wshift = 20;
    int ranges = 1;
    int32_t wwords = 1 << 15;
    bool unit_sorted = false;  // 1 < ranges <= 256: units sorted in place (no count pass)
};
HeavyGeometry heavy_geometry(int32_t bcols);
int64_t heavy_task_bound(int64_t count, int64_t products, int ranges);
int64_t heavy_slot_bound(int64_t count, int64_t products);

struct SymArgs {
    DevCsr a;
    const int64_t* brpt = nullptr;
    const int32_t* bcol = nullptr;
    int32_t bcols = 0;          // N (columns of B)
    int32_t row_lo = 0;         // global id of local row 0
    const int64_t* flop = nullptr;  // local profile
    const int64_t* item_flop = nullptr;  // per item FLOP (balanced multi-GPU pass), else flop[row]
    const int32_t* rows = nullptr;  // global row ids, or nullptr = all local rows
    int64_t n_items = 0;
    int64_t* out = nullptr;         // per item NNZ (nullable)
    long long* totals = nullptr;
    int total_slot = kZStar;        // kZStar (sampled) or kZ (exact)
    bool sampled_flop = false;      // also accumulate f* into totals[kFStar]
    const int64_t* window = nullptr;  // device [lo, hi): the items this rank counts (nullable = all)
    // A caller-provided FlopProfile (set_profile): its flop_per_row is the
    // reference's table size `tsize` (symbolic.hpp:35-40) -- a row with
    // tsize 0 counts 0 and tsize > max_flop_row is the reference's
    // invalid_argument (reported through heavy_meta[kMetaCapacity]); f* sums
    // tsize.  Binning and buffer sizing always use the row's true FLOP
    // (item_flop), so a profile that disagrees with the matrices cannot
    // overrun a tier's table.  nullptr: the profile is this context's own.
    const int64_t* tsize = nullptr;
    long long tsize_cap = 0;
    int64_t mp_max = 0;  // rows of kBin5Max < FLOP <= mp_max take the multipass tier (0: none)
    int64_t mp_part = kMpPart;  // its products per pass (test knob SPNNZ_MP_PART: a large value forces redos)
};
constexpr int kMetaCapacity = 9;  // heavy_meta slot: largest tsize above the profile's capacity

// Small problems (every row's FLOP <= kBin3Max, one rank, the context's own
// profile in args.flop): draw (draw: rows_out[i] = make_sample_plan's row i),
// FLOP and distinct count of every item -- items of FLOP <= kBin2Max one warp
// each on `stream`, the rest (stream_b non-null: the profile's max is above
// bin 2) one block each on stream_b; adds z* (and f*) to totals.
cudaError_t launch_sym_small(const SymArgs& args, uint64_t seed, int32_t num_rows, bool draw, int32_t* rows_out,
                             int num_sms, cudaStream_t stream, cudaStream_t stream_b = nullptr);
// Classifies items into bins (writes out[] = 0 for empty / foreign rows).
cudaError_t launch_sym_bin(const SymArgs& args, const SymScratch& s, cudaStream_t stream);
// Runs the smem tiers (bins 1-5) over the binned lists; grids are persistent
// and read the counts on the device.  streams[0..3] run concurrently (the
// caller forks them from its stream and joins them afterwards).
cudaError_t launch_sym_tiers(const SymArgs& args, const SymScratch& s, int num_sms,
                             const cudaStream_t* streams);
// Heavy tier for entries [first, first + count) of the heavy list (the host
// learns the count after a sync and sizes the batch's buffers).
// sorted: B rows non-decreasing -> the interval path (no product buffer).
// aux (nullable): a second stream for the small-range tasks, forked and
// joined through the events ev_a, ev_b.
cudaError_t launch_sym_heavy(const SymArgs& args, const SymScratch& s, bool sorted, int64_t first,
                             int64_t count, int num_sms, cudaStream_t stream, int64_t* launches = nullptr,
                             cudaStream_t aux = nullptr, cudaEvent_t ev_a = nullptr, cudaEvent_t ev_b = nullptr,
                             cudaEvent_t run_gate = nullptr);
void heavy_debug_print(cudaEvent_t start);  // SPNNZ_DEBUG_TIMELINE
// Per heavy item in list order: out[i] = FLOP, out[count + i] = A-row length,
// out[2 count + i] = boundary-table cells (batch planning when the heavy rows'
// products exceed one batch's buffers).
cudaError_t launch_heavy_flops(const SymArgs& args, const SymScratch& s, int64_t count,
                               int64_t* out, cudaStream_t stream);

// The single all-reduce of the totals (sums and the max): spread this rank's
// totals into row `rank` of a world x kTotals table (zero elsewhere), SUM
// all-reduce the table, finish: totals[first..first+count) = column sums,
// totals[kMax] = column max (with_max).
cudaError_t launch_totals_spread(const long long* totals, long long* table, int rank, int world,
                                 cudaStream_t stream);
cudaError_t launch_totals_finish(long long* totals, const long long* table, int world, int first, int count,
                                 bool with_max, cudaStream_t stream);

// -------------------------------------------------------------- predict
// ceil view min(flop, ceil(flop / cr)) and/or real view flop / cr.  If
// totals != nullptr the CR is derived on the device from totals[kFStar],
// totals[kZStar] (predict.hpp:111-117); else cr is used as given.
cudaError_t launch_predict(const int64_t* flop, int64_t m, const long long* totals, double cr,
                           int64_t* ceil_out, double* real_out, int num_sms, cudaStream_t stream);

// sampled_flop over global rows (flop.hpp:64-74); atomics into totals[kFStar].
cudaError_t launch_sampled_flop(const int64_t* flop, int32_t row_lo, int32_t local_rows,
                                const int32_t* rows, int64_t n, long long* totals,
                                cudaStream_t stream);

// Validation: counts rows outside [0, num_rows) into *bad.
// FLOP of each listed row (global ids; 0 outside [row_lo, row_lo + a.rows)),
// straight from A and B.rpt.  units: scratch of n + 1 entries.
cudaError_t launch_item_flop(const DevCsr& a, const int64_t* brpt, int32_t row_lo,
                             const int32_t* rows, int64_t n, int64_t* out, int64_t* units, int num_sms,
                             cudaStream_t stream);
// FLOP-balanced share of a sample list: window[0..1] = [lo, hi) such that
// rank's items carry ~1/world of the list's total FLOP (item_flop[n]).
cudaError_t launch_flop_window(const int64_t* item_flop, int64_t n, int rank, int world, int64_t* window,
                               cudaStream_t stream);
// B rows non-decreasing? cnt[0] == cnt[1] afterwards (device counters).
cudaError_t launch_check_sorted(const int64_t* rpt, const int32_t* col, int32_t rows, int64_t nnz,
                                unsigned long long* cnt, int num_sms, cudaStream_t stream);
cudaError_t launch_check_rows(const int32_t* rows, int64_t n, int32_t num_rows, int32_t* bad,
                              cudaStream_t stream);

}  // namespace spnnz_gpu
