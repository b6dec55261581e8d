// Kernel launch interface used by the C ABI (abi.cu).
#pragma once

#include <cuda_runtime.h>

#include "biluk_internal.h"

namespace biluk {

struct SweepArgs {
    const TileMeta *meta_l;
    const TileMeta *meta_u;
    const unsigned char *rec_l;
    const unsigned char *rec_u;
    int64_t nl, nu;          // tiles of the L and U' sweeps
    const double *b;         // right-hand side (n*bs)
    double *y_t;             // parity-tagged intermediate y at L positions, component-major
    double *x_t;             // parity-tagged result x at U' positions, component-major
    int64_t npos;            // component stride of y_t / x_t (>= tiles * R of either sweep)
    double *out;             // untagged result (may be null)
    DevStatus *st;
    const int *skip_flag;    // when non-null and *skip_flag != 0 the launch is a no-op
    int stages;
    int stage_bytes;
    uint64_t timeout_ns;
    const uint32_t *lvl_tiles;   // tiles per combined level (1-based)
    uint32_t *lvl_cnt;           // tiles finished per combined level (reset by the last CTA)
    int nlev_l;                  // combined level of U' level l is nlev_l + l
    int nlev_total;
    int gap;
    int coarse_sleep_ns;
    int fine_sleep_ns;
    int poll_all;
    int probe;
    int probe_sleep_ns;
    unsigned long long *trace;   // optional: per tile {t_ready, t_released, t_done, t_deps | cycle splits}
    int trace_mode;              // 1: t_deps in the 4th word; 2: packed cycle splits after the poll
};

// partitioned sweep (psweep.cu)
struct PSweepArgs {
    const PRecInfo *rec;         // all records (a CTA's range: part_rec[c] .. part_rec[c+1])
    const unsigned char *recs;   // record bytes
    const int32_t *part_rec;     // P+1 record ranges, then P counts of L records
    const double *b;             // right-hand side (n*bs, natural order)
    double *y_t;                 // parity-tagged y at L positions (tag_stride(bs) doubles each)
    double *x_t;                 // parity-tagged x at U' positions
    double *out;                 // untagged x (natural order; may be null)
    DevStatus *st;
    const int *skip_flag;        // when non-null and *skip_flag != 0 the launch is a no-op
    uint64_t timeout_ns;
    int ring_mask;               // vector ring rows - 1 (slot ring_mask+1 holds zeros)
    uint32_t data_bytes;         // record ring bytes
    unsigned long long *trace;   // optional: 8 x u64 per record (globaltimer stamps), then diagnostics
    int64_t nrec_total;
    const double *b_perm;        // b in L-position order (pvs doubles per position; launch_permute_b)
    double *y_u;                 // y in U'-position order (written by the L sweep, read by U' records)
};
// grid sweep (gsweep.cu)
struct GSweepArgs {
    const GPart *parts;
    const GRec *recs;
    const int32_t *cols;         // P * 128: (y << 16) | z
    const unsigned char *stream; // record bytes
    const double *b;             // right-hand side (n*bs, natural order)
    double *y;                   // y (n*bs, natural order; written by L, read by U')
    double *out;                 // x (natural order; may be null)
    double *y_t;                 // parity-tagged rows (natural index, tag_stride(bs) doubles each)
    double *x_t;
    DevStatus *st;
    const int *skip_flag;
    uint64_t timeout_ns;
    int64_t nx, ny, nz;
    int slot_bytes, kslots;
    unsigned long long *trace;   // optional: 8 x u64 per record (globaltimer stamps, gsweep.cu), then clock64 stages
    int64_t nrec_total;
};
cudaError_t launch_gsweep(const Plan &p, const GSweepArgs &a, cudaStream_t s);
cudaError_t gsweep_occupancy(const Plan &p, int *blocks_per_sm);
cudaError_t launch_gpack(const Plan &p, cudaStream_t s);
size_t gsweep_smem_bytes(const Plan &p);
cudaError_t launch_ppack(const Plan &p, cudaStream_t s);
cudaError_t launch_permute_b(const Plan &p, const double *b, cudaStream_t s, const int *skip = nullptr);
cudaError_t launch_psweep(const Plan &p, const PSweepArgs &a, cudaStream_t s);
cudaError_t psweep_occupancy(const Plan &p, int *blocks_per_sm);
size_t psweep_smem_bytes(const Plan &p);

cudaError_t launch_materialize(const Plan &p, const double *avals, cudaStream_t s);
cudaError_t launch_factor(const Plan &p, cudaStream_t s);
cudaError_t launch_split(const Plan &p, cudaStream_t s);
cudaError_t launch_diag_invert(const Plan &p, cudaStream_t s);   // stages.cu: D^-1 of a loaded factored matrix
cudaError_t launch_pack(const Plan &p, cudaStream_t s);
cudaError_t launch_pack_ell(const Op &o, const double *avals, cudaStream_t s);
cudaError_t launch_sweep(const Plan &p, const SweepArgs &a, cudaStream_t s);
cudaError_t sweep_occupancy(const Plan &p, int *blocks_per_sm);
size_t sweep_smem_bytes(const Plan &p);
cudaError_t launch_spmv(const Op &o, const double *x, double *y, const int *skip, cudaStream_t s);

}  // namespace biluk
