// Internal declarations shared by the host planner (plan.cpp), the kernels
// (kernels.cu) and the C ABI (abi.cu).  Not part of the public interface.
#pragma once

#include <cuda_runtime_api.h>

#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/biluk.h"

#ifdef __CUDACC__
#define BILUK_HD __host__ __device__
#else
#define BILUK_HD
#endif

namespace biluk {

// ---------------------------------------------------------------------------
// error plumbing
// ---------------------------------------------------------------------------
void set_error(const std::string &msg);
int fail(int code, const std::string &msg);

// ---------------------------------------------------------------------------
// tile geometry (shared by host planner and device kernels)
//
// A sweep processes block rows in level-major order (ascending row index
// inside a level), R rows per "tile"; one warp owns one tile at a time, one
// lane per block row (lanes >= R idle).  Row i of a sweep has a POSITION
// pos = tile * R + lane; the sweep's intermediate vector lives at positions,
// component-major (v[c * npos + pos]), so the 32 dependencies a warp reads
// are (near-)contiguous and a published tile is one coalesced store.
// A tile record is one contiguous, 128-byte aligned byte range:
//   rows  int32[R]                       (128 B; natural row index, -1 = padding)
//   ypos  int32[R]                       (128 B; U' sweep only: the row's L position)
//   cols  int32[S][R]                    (dependency POSITIONS; -1 = padding slot)
//   dinv  f64[bs*bs][R]                  (U' sweep only: D^-1 of the row)
//   vals  f64[S][bs*bs][R]               (block values, element e = c*bs + r)
// so that a whole tile is moved by ONE bulk async copy (cp.async.bulk) and
// every lane reads its own row's data lane-contiguously from shared memory.
// ---------------------------------------------------------------------------
BILUK_HD constexpr inline int rows_per_tile(int bs) {
    return bs <= 4 ? 32 : (bs <= 6 ? 16 : 8);
}
BILUK_HD constexpr inline int64_t align128(int64_t x) { return (x + 127) & ~int64_t(127); }
// doubles per position in the sweep vectors (power of two >= bs: vector loads/stores)
BILUK_HD constexpr inline int vec_stride(int bs) { return bs <= 1 ? 1 : (bs <= 2 ? 2 : (bs <= 4 ? 4 : 8)); }
// doubles per position of the parity-TAGGED sweep vectors y_t / x_t (both
// engines): a power of two >= bs + 1, the extra word carrying the values'
// displaced mantissa LSBs so that published values stay exact (device_util.cuh)
BILUK_HD constexpr inline int tag_stride(int bs) { return bs < 2 ? 2 : (bs < 4 ? 4 : (bs < 8 ? 8 : 16)); }
// header: rows int32[R] (natural block-row index, -1 = padding); U' tiles add
// ypos int32[R] (the row's position in the L sweep, where its y lives)
BILUK_HD constexpr inline int64_t rec_hdr_bytes(bool upper) { return upper ? 256 : 128; }
BILUK_HD constexpr inline int64_t rec_cols_bytes(int bs, int S) {
    return align128(int64_t(S) * rows_per_tile(bs) * 4);
}
BILUK_HD constexpr inline int64_t rec_dinv_off(int bs, int S) { return 256 + rec_cols_bytes(bs, S); }
BILUK_HD constexpr inline int64_t rec_vals_off(int bs, int S, bool upper) {
    return upper ? rec_dinv_off(bs, S) + int64_t(bs) * bs * rows_per_tile(bs) * 8 : 128 + rec_cols_bytes(bs, S);
}
BILUK_HD constexpr inline int64_t rec_bytes(int bs, int S, bool upper) {
    return align128(rec_vals_off(bs, S, upper) + int64_t(S) * bs * bs * rows_per_tile(bs) * 8);
}
// SpMV tiles (natural row order, no rows array): cols int32[S][R] | vals f64[S][bs*bs][R]
BILUK_HD constexpr inline int64_t ell_vals_off(int bs, int S) { return rec_cols_bytes(bs, S); }
BILUK_HD constexpr inline int64_t ell_bytes(int bs, int S) {
    return align128(ell_vals_off(bs, S) + int64_t(S) * bs * bs * rows_per_tile(bs) * 8);
}

struct TileMeta {      // 32 bytes
    uint32_t off128;   // record offset in 128-byte units
    int32_t nslot;     // S
    int32_t level;     // 1-based dependency level of the tile's rows (sweeps only)
    int32_t probe[2];  // probe[d-1]: one ancestor at level - d to wait on cheaply before the
                       // full poll: >= 0: position in this sweep's vector; <= -2: L position
                       // -(probe+2) of a y value (U' tiles of the first levels); -1: none
    int32_t pad[3];
};

// device status block (lives in the workspace)
struct DevStatus {
    int32_t status;          // sticky apply status (0 / BILUK_ETIMEOUT)
    int32_t fstatus;         // factorization status (0 / ESINGULAR / EZEROPIVOT)
    long long ferr_row;      // first failing block row (atomicMin)
    uint32_t epoch;          // apply epoch; parity tag of the sweep vectors
    uint32_t done_ctas;      // CTAs finished in the current sweep launch
    uint32_t prefix;         // every combined level <= prefix is complete (progress hint)
    uint32_t pad0;
};

// runtime knobs of the sweep (biluk_plan_tune)
struct SweepTune {
    int gap = 0;             // fine-grained polling starts once prefix >= level - gap (<= 0: no gate, no counters)
    int coarse_sleep_ns = 64;
    int fine_sleep_ns = 0;
    int warps = 4;           // warps per CTA actually launched (0 = the planned maximum)
    int poll_all = 1;        // 1: poll every component at once (one round trip, more traffic)
    int probe = 0;           // d = 1, 2: one lane waits on an ancestor d levels back before the full poll
    int probe_sleep_ns = 32;
    int trace_mode = 1;      // diagnostics layout of the per-tile trace
};

struct Sweep {                       // host copy of one sweep's tile layout
    int64_t ntiles = 0;
    std::vector<int32_t> tile_rows;  // ntiles * R
    std::vector<int32_t> pos;        // n: position of every block row in this sweep
    std::vector<TileMeta> meta;      // ntiles
    int64_t rec_total = 0;           // bytes of all records
    int32_t max_slots = 0;
    int64_t max_rec = 0;
};

// ---------------------------------------------------------------------------
// Partitioned sweep (the apply engine).
//
// The block rows are cut into P contiguous ranges ("parts"), one CTA each.
// Every L dependency of a row lies in its own part or an EARLIER part, every
// U' dependency in its own part or a LATER one, so the parts form a chain and
// the level chain mostly stays inside one SM: a dependency on the same part
// is read from a shared-memory ring of recent results, one on another part is
// fetched (parity-tag polled) from L2 by a prefetch warp ahead of use.
// A part's rows are processed in (global level, row) order, one thread per
// row, in RECORDS of <= nthreads rows of one level; a record is one
// contiguous byte range moved by one cp.async.bulk:
//   hdr   PRecHdr (32 B)
//   iarr  int32[nrows]          L: the row's U' position (where it stores y for
//                               the U' sweep); U': natural block row (x scatter);
//                               bit 31: publish the row to the tagged vector (some
//                               record fetches it)
//   desc  int16[S][nrows]       >= 0: vector-ring slot (slot `ring` is zero);
//                               < 0: fetched dependency -(d+1); padded to a word
//   gpos  int32[nglob]          deduplicated dependency positions in the
//                               sweep's own vector (parity-tag polled)
//   (align 16)
//   dinv  f64[bs*bs][nrows]     U' only
//   vals  f64[S][bs*bs][nrows]  element e = c*bs + r (column-major blocks)
//   (align 16)                  = `bytes`, streamed by one bulk copy
// and, in shared memory only, behind it:
//   input f64[nrows][pvs]       the rows' own inputs, a second bulk copy of
//                               the position-ordered b (L) or y (U') vector
//   deps  f64[bs][nglob]        fetched dependencies (exact), component-major
// ---------------------------------------------------------------------------
struct PRecHdr {        // 32 bytes
    int32_t nrows, S, nglob;
    int32_t flags;      // bit 0: U' record; bits 1..9: rows; bits 10..: dependency level (diagnostics)
    int32_t seq0;       // ring sequence number of the first row
    int32_t pos0;       // vector position of the first row (y_t for L, x_t for U')
    int32_t vals_off;   // byte offset of dinv (U') / vals inside the record
    int32_t in_off;     // byte offset of the input area (= record bytes); deps follow the inputs
};
struct PRecInfo {       // 64 bytes: one per record, read by the producer, the gather warp and the pack kernel
    uint64_t off;       // byte offset of the record (16-aligned)
    uint64_t idx_off;   // int32 offset of its index section in the compact index image (16-aligned)
    int64_t vmap_off;   // first entry of its value map (S * nrows P' slots, -1 = padding)
    uint32_t bytes;     // streamed record bytes (multiple of 16) = offset of the value area
    uint32_t idx_words; // int32 words of the index section (header .. gpos)
    int32_t nrows, S;
    uint32_t foot;      // shared-memory footprint: bytes + value area
    int32_t level;      // dependency level of its rows * 2 + upper (= PRecHdr::flags)
    int32_t nglob;      // fetched dependencies
    int32_t pos0;       // vector position of its first row (inputs: pos0 .. pos0 + nrows)
    int32_t pad[2];
};
// component planes of the partitioned sweep's vector ring (component-major:
// one plane of ring + 2 doubles per component; (ring + 2) * 8 is a multiple of 16)
BILUK_HD constexpr inline int ps_vec_stride(int bs) { return bs; }
// the rows' inputs (b in L-position order, y in U'-position order) are packed,
// bs doubles per position; a record's input area in shared memory holds its
// rows plus the 8 bytes of slack the bulk copy may start early by (it starts
// at the 16-byte boundary at or below the first row)
BILUK_HD constexpr inline int64_t ps_in_bytes(int bs, int nrows) { return (int64_t(nrows) * bs * 8 + 8 + 15) & ~int64_t(15); }
// fetched dependencies per record (a multiple of 32: one per poll lane and round)
BILUK_HD constexpr inline int ps_glob_cap(int) { return 1024; }   // fetched dependencies per record (the compute threads loop over them)
constexpr int PS_KSLOTS = 16;      // records in flight per CTA (mbarrier sets)

// an assignment of block rows to parts (any assignment is deadlock-free:
// every CTA walks its rows in global level order)
struct Partition {
    int P = 0;
    int kind = 0;                    // 0: contiguous row ranges, 1: structured-grid (y, z) columns
    int64_t grid[3] = {0, 0, 0};     // nx, ny, nz (kind 1)
    int split[2] = {0, 0};           // parts along y, z (kind 1)
    std::vector<int32_t> part_of;    // n
    std::vector<std::vector<int32_t>> rows;   // rows of each part, ascending
    std::vector<int32_t> base;       // P+1 first vector position of each part
};

struct PSweep {
    int32_t P = 0;                   // parts = CTAs
    int32_t partition = 0;           // Partition::kind
    int64_t grid[3] = {0, 0, 0};
    int32_t split[2] = {0, 0};
    int32_t nthreads = 128;          // rows per record at most = threads of a compute group
    int32_t ring = 1024;             // vector ring rows (power of two; slot `ring` is all zeros)
    int64_t data_ring = 0;           // shared-memory bytes of the record ring
    int64_t xval_ring = 0;           // shared-memory bytes of the fetched-value ring
    int64_t rec_cap = 0, glob_cap = 0;
    int groups = 3;                  // compute groups of the sweep kernel (2 or 3, see psweep.cu)
    int nprod = 2;                   // producer warps of the sweep kernel (1 or 2, see psweep.cu)
    int32_t nlrec_max = 0;           // most L records of one part
    std::vector<int32_t> part_rec;   // P+1 record ranges (a part's L records, then its U' records),
                                     // then P counts of L records
    std::vector<PRecInfo> rec;
    std::vector<int32_t> idx;        // compact index sections
    std::vector<int32_t> vmap;       // value maps
    std::vector<int32_t> posL, posU; // vector position of every block row in each sweep
    int64_t rec_total = 0, max_rec = 0, max_glob = 0, nglob_total = 0;
    double est_us = 0;               // planner's time estimate for the chosen P
};

// ---------------------------------------------------------------------------
// Grid sweep (engine 2; gsweep.cu): ILU(0) of a 7-point block
// stencil on an nx x ny x nz natural-order grid.  The parts are the (y, z)
// column blocks of the partitioned sweep (<= 128 columns each, one CTA per
// part).  Thread t of a part owns column t (columns ordered by d = y + z, so
// the columns holding a row of level s = x + d are a contiguous range) and
// walks its column's rows level by level: the x-1 (U': x+1) dependency is the
// thread's own previous result (a register), the y and z neighbours are the
// neighbouring threads' previous results (shared memory, double-buffered,
// one named barrier per level), or -- on a part face -- the rows other parts
// publish to the parity-tagged vectors (polled ahead by halo warps).  The
// factor blocks stream as one record per (part, level):
//   hdr  int32[4]  nrows, lo (first column), stride R (rows, even), 0
//   L:   f64[3][bs*bs][R]            blocks of the x-1, y-1, z-1 neighbours
//   U':  f64[bs*bs][R] D^-1, then f64[3][bs*bs][R]  (x+1, y+1, z+1)
// (zero blocks where a neighbour is outside the grid).
// ---------------------------------------------------------------------------
struct GPart {          // 32 bytes
    int32_t y0, y1, z0, z1;
    int32_t ncols;      // columns (<= 128), ordered by (y + z, y)
    int32_t nl, nu;     // L and U' records
    int32_t rec0;       // first record
};
struct GRec {           // 16 bytes
    int64_t off;        // byte offset of the record in the stream
    int32_t bytes;      // record bytes (multiple of 16)
    int32_t nrows;
};
struct GSweep {
    int32_t P = 0, py = 0, pz = 0;
    int64_t nx = 0, ny = 0, nz = 0;
    int32_t ne = 0;                  // halo entries of a part (max over parts and sweeps)
    int32_t slot_bytes = 0, kslots = 0;
    int64_t stream_bytes = 0;
    std::vector<GPart> part;
    std::vector<GRec> rec;
    std::vector<int32_t> rec_lo;     // first column of each record
    std::vector<int32_t> cols;       // P * 128: (y << 16) | z of each part's columns
};

struct Plan {
    int32_t bs = 0, k = 0;
    int64_t n = 0;
    int64_t nnzA = 0, nnzP = 0, nL = 0, nU = 0;
    // pattern of A and of the ILU(k) pattern P' (int32 indices)
    std::vector<int32_t> a_rp, a_ci;
    std::vector<int32_t> p_rp, p_ci, p_diag;
    std::vector<int32_t> a2p;        // A slot -> P' slot
    // block level sets
    std::vector<int32_t> lev_L, lev_U;
    int32_t nlev_L = 0, nlev_U = 0;
    std::vector<int32_t> forder;     // rows in L-level order (factorization)
    std::vector<int64_t> fptr;       // level pointers into forder (nlev_L + 1)
    int32_t max_row_len = 0;         // longest P' row (factor shared memory)
    Sweep sl, su;                    // L sweep, U' sweep
    PSweep ps;                       // partitioned sweep layout
    GSweep gs;                       // grid sweep layout
    int32_t engine = 1;              // 2: grid sweep, 1: partitioned sweep, 0: tiled level-order sweep
    std::vector<uint32_t> lvl_tiles; // tiles per combined level (L levels, then U' levels), 1-based
    SweepTune tune;
    unsigned long long *trace = nullptr;   // optional per-tile timing records (diagnostics)
    // launch configuration of the sweep kernel
    int32_t sweep_ctas = 0, sweep_warps = 0, sweep_stages = 0;
    int64_t stage_bytes = 0;
    int32_t num_sms = 0;
    // workspace layout (byte offsets)
    struct {
        uint64_t p_rp, p_ci, p_diag, a2p, forder, pvals, dinv, sl_rows, sl_meta, sl_rec, su_rows, su_meta,
            su_rec, pos_l, pos_u, y_t, x_t, lvl_tiles, lvl_cnt, status, ps_rec, ps_info, ps_part, ps_idx,
            ps_vmap, ps_posl, ps_bperm, ps_yu, gs_part, gs_rec, gs_lo, gs_cols, gs_stream, gs_y, total;
    } off{};
    // bound device pointers
    unsigned char *ws = nullptr;
    bool bound = false, factored = false;
    bool factor_only = false;        // created by biluk_plan_create_ex(BILUK_PLAN_FACTOR_ONLY): no sweep plan
};

// A block sparse operator for SpMV: sliced-ELL tiles of R consecutive block
// rows (natural order), tile record = cols int32[S][R] | vals f64[S][bs*bs][R].
struct Op {
    int32_t bs = 0;
    int64_t n = 0, ncols = 0, nnz = 0;
    std::vector<int32_t> rp, ci;
    int64_t ntiles = 0;
    std::vector<TileMeta> meta;
    int64_t rec_total = 0;
    int32_t num_sms = 148;
    struct {
        uint64_t rp, ci, meta, rec, total;
    } off{};
    unsigned char *ws = nullptr;
    bool bound = false, valued = false;
};

// positions of the sweep vectors y_t / x_t (each position holds one block row,
// vec_stride(bs) contiguous doubles)
inline int64_t plan_npos(const Plan &p) {
    const int64_t a = p.sl.ntiles * rows_per_tile(p.bs), b = p.su.ntiles * rows_per_tile(p.bs);
    const int64_t m = a > b ? a : b;
    return m > p.n ? m : p.n;
}
// doubles per position of the tagged sweep vectors y_t / x_t (either engine)
inline int plan_vs(const Plan &p) { return tag_stride(p.bs); }

// host planner (plan.cpp)
int symbolic_phase(int64_t n, const int32_t *rp, const int32_t *ci, int k, std::vector<int32_t> &out_rp,
                   std::vector<int32_t> &out_ci, int64_t *err_row);
void level_schedule(int64_t m, const int64_t *rp, const int64_t *ci, bool upper, int64_t *lev, int64_t *nlev);
int validate_bsr(int64_t n, int64_t ncols, const int64_t *rp, const int64_t *ci);
int plan_analyse(Plan &p, int32_t bs, int64_t n, const int64_t *rp, const int64_t *ci, int32_t k, int64_t *err_row);
int plan_tiles(Plan &p);
void plan_layout(Plan &p, int num_sms, size_t smem_per_sm);
// partitioned sweep planner (psweep_plan.cpp): parts = 0 chooses P by the cost model
int plan_psweep(Plan &p, int num_sms, size_t smem_per_block, int parts);
double psweep_estimate_us(const Plan &p, const Partition &pt);
bool detect_grid(const Plan &p, int64_t g[3]);
void partition_grid_columns(const Plan &p, int P, const int64_t g[3], Partition &pt);   // (y, z) column parts
// grid sweep planner (gsweep.cu): BILUK_OK, or BILUK_EUNSUPPORTED when the
// pattern is not a 7-point ILU(0) grid the engine handles
int plan_gsweep(Plan &p, int num_sms, size_t smem_per_block);
int op_analyse(Op &o, int32_t bs, int64_t n, int64_t ncols, const int64_t *rp, const int64_t *ci);

}  // namespace biluk

// the opaque handles of the C ABI
struct biluk_plan {
    biluk::Plan p;
    // optional CUDA events around the sweep launch (biluk_plan_set_timing)
    cudaEvent_t tev[2] = {nullptr, nullptr};
    // the last apply's completion and stream: an apply on another stream waits
    // for it, because every apply of a plan uses the plan's sweep workspace
    cudaEvent_t last_ev = nullptr;
    cudaStream_t last_stream = nullptr;
    ~biluk_plan() {
        for (cudaEvent_t e : tev)
            if (e) cudaEventDestroy(e);
        if (last_ev) cudaEventDestroy(last_ev);
    }
};
struct biluk_op {
    biluk::Op o;
};

namespace biluk {
// biluk_plan_apply with a device skip word (abi.cu; Krylov graphs)
int plan_apply(biluk_plan *plan, const double *dev_b, double *dev_x, cudaStream_t st, const int *skip);
// order the plan's next apply on `st` outside a stream capture
int plan_adopt_stream(biluk_plan *plan, cudaStream_t st);
// record that the plan's last apply was issued on `st` (after graph replays)
int plan_mark(biluk_plan *plan, cudaStream_t st);
}  // namespace biluk
