// Internal declarations shared by the host planner (plan.cpp), the kernels
// (kernels.cu) and the C ABI (abi.cu).  Not part of the public interface.
#pragma once

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
            su_rec, pos_l, pos_u, y_t, x_t, lvl_tiles, lvl_cnt, status, total;
    } off{};
    // bound device pointers
    unsigned char *ws = nullptr;
    bool bound = false, factored = false;
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
    return a > b ? a : b;
}

// host planner (plan.cpp)
int symbolic_phase(int64_t n, const int32_t *rp, const int32_t *ci, int k, std::vector<int32_t> &out_rp,
                   std::vector<int32_t> &out_ci, int64_t *err_row);
void level_schedule(int64_t m, const int64_t *rp, const int64_t *ci, bool upper, int64_t *lev, int64_t *nlev);
int validate_bsr(int64_t n, int64_t ncols, const int64_t *rp, const int64_t *ci);
int plan_analyse(Plan &p, int32_t bs, int64_t n, const int64_t *rp, const int64_t *ci, int32_t k, int64_t *err_row);
void plan_layout(Plan &p, int num_sms, size_t smem_per_sm);
int op_analyse(Op &o, int32_t bs, int64_t n, int64_t ncols, const int64_t *rp, const int64_t *ci);

}  // namespace biluk

// the opaque handles of the C ABI
struct biluk_plan {
    biluk::Plan p;
};
struct biluk_op {
    biluk::Op o;
};
