/*
 * fa.h -- C ABI of libfa: B200-native parallel non-divergent (D8) flow
 * accumulation, after Barnes, "Parallel Non-divergent Flow Accumulation for
 * Trillion Cell Digital Elevation Models" (arXiv 1608.04431).
 *
 * Citations: "P:Lnn" is /root/reference/PAPER.md line nn; "Dn" is reading n
 * in DESIGN.md ("Readings of the paper").
 *
 * Conventions (all entry points)
 *  - Rasters are row-major, contiguous (pitch == cols).  Pointers may be
 *    CUDA device pointers on the context's device, or host pointers (pinned
 *    or pageable); the library detects which (cudaPointerGetAttributes) and
 *    stages host buffers through device memory inside the call.  The caller
 *    owns every buffer it passes; the library never frees them.
 *  - Every call enqueues on the context's stream and returns only after the
 *    work completed, so data-dependent errors (cycle, bad code, overflow)
 *    are reported.  Outputs are undefined unless FA_OK is returned.
 *  - No call aborts, throws or prints.  fa_last_error() gives a message.
 *  - Scratch memory is owned by the context: allocated lazily, grown on
 *    demand, freed by fa_destroy().  A context is bound to one device and is
 *    not thread-safe.
 *  - Direction codes (D1): 0 NoFlow, 1 N(0,-1), 2 NE(+1,-1), 3 E(+1,0),
 *    4 SE(+1,+1), 5 S(0,+1), 6 SW(-1,+1), 7 W(-1,0), 8 NW(-1,-1) as (dx,dy)
 *    with y = row index growing downward; 255 NoData.
 *  - NoData elevation: z == nodata or z non-finite.  NoData output marker:
 *    0xFFFFFFFF (u32), all-ones (u64), quiet NaN (f64) (D9).
 */
#ifndef FA_H
#define FA_H

#include <stdint.h>

#if defined(__GNUC__)
#define FA_API __attribute__((visibility("default")))
#else
#define FA_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct fa_ctx fa_ctx;

typedef enum {
  FA_OK = 0,
  FA_E_ARG = 1,      /* NULL/negative sizes, dem and dirs both or neither, bad wtype/atype, bad weight (D21),
                        alpha outside [0,1] (absorption), device/host buffer kind not accepted by the call */
  FA_E_DIRCODE = 2,  /* a direction byte not in {0..8, 255} (D1) */
  FA_E_CYCLE = 3,    /* some data cell never retires: the direction graph has a cycle */
  FA_E_OVERFLOW = 4, /* integer accumulation could exceed the output type (D10) */
  FA_E_NOMEM = 5,
  FA_E_CUDA = 6,
  FA_E_NCCL = 7,
  FA_E_STATE = 8     /* wrong device, ranks disagree, communicator missing */
} fa_status;

typedef enum { FA_W_NONE = 0, FA_W_U32 = 1, FA_W_F32 = 2 } fa_wtype; /* NONE => w = 1 */
typedef enum { FA_A_U32 = 0, FA_A_U64 = 1, FA_A_F64 = 2 } fa_atype;
/* valid (wtype, atype): (NONE|U32, U32|U64), (F32, F64), (NONE, F64) */

/* Create a context on `device`, enqueuing on `cuda_stream` (a cudaStream_t;
 * NULL = the legacy default stream).  tile_rows x tile_cols is the paper's
 * tile ("subdivided into rectangular tiles of equal dimension"); the
 * last tile row/column is ragged (D20).  <= 0 means the whole raster is one
 * tile.  The tiling never changes results; it sets the
 * granularity of the perimeter records (fa_perimeter_records) and of the
 * multi-GPU exchange. */
FA_API fa_status fa_create(fa_ctx** out, int device, void* cuda_stream, int64_t tile_rows,
                    int64_t tile_cols);
FA_API fa_status fa_destroy(fa_ctx* ctx);
FA_API const char* fa_last_error(const fa_ctx* ctx);

/* Context options (per context, default in brackets; read at each call).
 * None changes results: they select among equivalent schedules of the same
 * method, so every option value is covered by the same parity tests.
 *   FA_OPT_RETENTION  [FA_RETAIN] | FA_EVICT: the paper's memory retention
 *       strategies.  RETAIN keeps the block-local accumulation in
 *       the output and the finalize walks each entry's path adding its offset
 *       (P:L260); EVICT recomputes the block accumulation with w + x.
 *   FA_OPT_D8  [FA_D8_SPLIT] | FA_D8_FUSED: H1 as its own kernel, or fused
 *       into the pass-1 block kernel (DEM input only).
 *   FA_OPT_BLOCK_ROWS  [32] | 16 | 64: rows of the warp-resident blocks
 *       (32 wide).  Absorption always runs with 32.
 *   FA_OPT_WALK_CAP  [128], 0..2^20: steps of a perimeter-graph walk before
 *       it re-queues (0: level-synchronous peeling only).
 *   FA_OPT_FILL_TILE  [32] | 64: tile side of fa_fill.
 *   FA_OPT_VALUES  [FA_VALUES_L2] | FA_VALUES_SMEM: where the pass-1 /
 *       EVICT pass-2 block kernels keep the block's values while Alg. 1 runs:
 *       in the output raster (L2-resident, pushes as global atomics, many
 *       warps per SM) or in shared memory (no global round trip, fewer warps).
 *   FA_OPT_GRAPH  [FA_GRAPH_AUTO] | FA_GRAPH_HOST | FA_GRAPH_DEVICE: the
 *       perimeter-graph solver (H5) as kernels driven from the host (a
 *       device-to-host read per decision: frontier size, residual size, jump
 *       convergence, segments), or as one cooperative persistent kernel
 *       taking every decision on the device (no host round trip; slower on
 *       large graphs: fewer walks in flight).  AUTO: single-device calls with
 *       at most 2^24 block slots (~134 M cells) run without any host round
 *       trip before the final status read (the node count stays on the
 *       device, the device solver reads it); larger ones use the host-driven
 *       solver.
 *   FA_OPT_DIST_RECORDS  [FA_DIST_STRIPS] | FA_DIST_TILES: the record
 *       granularity of the multi-GPU exchange -- each rank's strip as one
 *       tile (the strip's block-exit graph cut only at its edges, records =
 *       the strip perimeter, the producer graph over N strips; needs equal
 *       strips, the last may be shorter, else the tiles are used) or the
 *       context's tiles (every tile's perimeter all-gathered).
 *       fa_accumulate_strips / fa_accumulate_absorb with nstrips > 1 follow
 *       the same option (strips of ceil(rows / nstrips) rows as tiles).
 * Unknown option or value out of range: FA_E_ARG, the option unchanged. */
typedef enum {
  FA_OPT_RETENTION = 1,
  FA_OPT_D8 = 2,
  FA_OPT_BLOCK_ROWS = 3,
  FA_OPT_WALK_CAP = 4,
  FA_OPT_FILL_TILE = 5,
  FA_OPT_VALUES = 6,
  FA_OPT_GRAPH = 7,
  FA_OPT_DIST_RECORDS = 8
} fa_option;
enum { FA_RETAIN = 0, FA_EVICT = 1 };
enum { FA_D8_SPLIT = 0, FA_D8_FUSED = 1 };
enum { FA_VALUES_L2 = 0, FA_VALUES_SMEM = 1 };
enum { FA_GRAPH_HOST = 0, FA_GRAPH_DEVICE = 1, FA_GRAPH_AUTO = 2 };
enum { FA_DIST_TILES = 0, FA_DIST_STRIPS = 1 };
FA_API fa_status fa_set_option(fa_ctx* ctx, int option, int64_t value);
FA_API fa_status fa_get_option(const fa_ctx* ctx, int option, int64_t* value);

/* H1: D8 flow directions of a DEM ("D8 ... a single one of its
 * neighbours"; BASELINE north_star: steepest strictly-downhill neighbour,
 * diagonal drop divided by sqrt2 (exact compare, D4), ties to the lowest
 * code (D2), outlet fallback to the lowest off-grid/NoData code (D3),
 * NoFlow (0) if none (D6), NoData -> 255).
 *   dem  : rows x cols float32, in.       dirs : rows x cols uint8, out. */
FA_API fa_status fa_flowdirs(fa_ctx* ctx, const float* dem, int64_t rows, int64_t cols, float nodata,
                      uint8_t* dirs);

/* Depression filling ("the depressions can be filled to the
 * level of their lowest outlets ... Priority-Flood"; D15): out = the
 * Priority-Flood+epsilon surface W of dem -- W = z at seeds (data cells on
 * the grid edge or 8-adjacent to NoData), W(p) = max(z(p), nextafterf(min
 * of the data neighbours' W, +inf)) elsewhere (unique; the input the D8 of
 * fa_flowdirs / fa_accumulate expects).  NoData (== nodata or non-finite)
 * is copied.  rows x cols f32, device or host buffers; out may not alias dem.
 * stats: ms_total, launches. */
FA_API fa_status fa_fill(fa_ctx* ctx, const float* dem, int64_t rows, int64_t cols, float nodata,
                         float* out);

/* H1-H6: flow accumulation A(p) = w(p) + sum_{n: target(n)=p} A(n)
 * (Eq. 1, alpha in {0,1}).  Exactly one of `dem` (then D8 is
 * computed, H1) or `dirs` is non-NULL.  `w` may be NULL (w = 1).  Flow into
 * NoData or off the grid is dropped (D8); NoFlow cells keep inflow plus
 * their own w (D7).  Integer results are exact; f64 results are within
 * 1e-9 relative of the exact sum (D13).  f32 weights must be finite and
 * >= 0 (D21); weights of NoData cells are ignored.
 *   acc : rows x cols of u32 / u64 / f64 according to atype, out. */
FA_API fa_status fa_accumulate(fa_ctx* ctx, int64_t rows, int64_t cols, const float* dem, float nodata,
                        const uint8_t* dirs, const void* w, fa_wtype wtype, void* acc,
                        fa_atype atype);

/* The row-strip pipeline of fa_accumulate_dist (H4-H7) on one device: the
 * raster is cut into `nstrips` strips of whole tile rows, each strip runs
 * phase A (pass 1 with halo rows, tile records), the records of all strips
 * are exchanged by device copies instead of NCCL, and each strip runs phase
 * B.  Same inputs, outputs and results as fa_accumulate; it exists so the
 * multi-GPU data path can be verified on one GPU. */
FA_API fa_status fa_accumulate_strips(fa_ctx* ctx, int nstrips, int64_t rows, int64_t cols,
                                      const float* dem, float nodata, const uint8_t* dirs,
                                      const void* w, fa_wtype wtype, void* acc, fa_atype atype);

/* Absorption (Eq. 1 with a per-cell alpha: "flow may
 * be absorbed during its downhill movement ... alpha is constrained such
 * that sum_p alpha(n,p) <= 1"; "most forms of absorption represent a simple
 * extension of the algorithm"):
 *   A(p) = w(p) + sum_{n : target(n) = p} alpha(n) A(n)
 * alpha: f32 rows x cols (same layout as the raster), the fraction of a
 * cell's accumulation passed to its D8 target; data cells need a finite
 * value in [0, 1] (else FA_E_ARG); NoData cells' alpha is ignored.  Output
 * f64 (NoData = quiet NaN); wtype FA_W_NONE (w = 1) or FA_W_F32.  Device or
 * host buffers.  32x32 blocks (the default); the block-exit graph is solved
 * with multiplicative edges (walks, peeling and affine chain contraction).
 * nstrips <= 1: one device, uncut; nstrips > 1: the row-strip pipeline of
 * the multi-GPU path on this device, with the tile links carrying their
 * alpha path factors (tile records, the producer graph G2 and the offsets
 * all weighted). */
FA_API fa_status fa_accumulate_absorb(fa_ctx* ctx, int nstrips, int64_t rows, int64_t cols,
                                      const float* dem, float nodata, const uint8_t* dirs,
                                      const void* w, fa_wtype wtype, const float* alpha,
                                      double* acc);

/* Out-of-core accumulation (the paper's EVICT strategy, P:L79-81,
 * P:L255): dem / dirs / w / acc are HOST buffers (pinned memory
 * gives full-speed copies; pageable works) and the raster may exceed device
 * memory.  Only strips of whole tile rows are resident: `strip_rows` raster
 * rows per strip (rounded up to the tile height; <= 0: sized from free
 * device memory, ~40 B per resident cell).  Phase A uploads each strip (z
 * with two halo rows per side, or dirs with one; w), runs D8 + pass 1 + the
 * tile records and drops the strip; the perimeter graph is solved once;
 * phase B uploads each strip again, recomputes pass 1, injects the offsets,
 * finalizes and downloads A.  Copies of neighbouring strips overlap the
 * compute (an upload and a download stream).  PCIe traffic per cell: 2x(z or dirs, w) in,
 * A out.  Same results and errors as fa_accumulate; device pointers are
 * rejected with FA_E_ARG. */
FA_API fa_status fa_accumulate_streamed(fa_ctx* ctx, int64_t rows, int64_t cols, const float* dem,
                                        float nodata, const uint8_t* dirs, const void* w,
                                        fa_wtype wtype, void* acc, fa_atype atype,
                                        int64_t strip_rows);

/* A batch of `count` independent rasters of one shape, each accumulated
 * exactly as fa_accumulate does it (same kernels, results and errors), from
 * HOST buffers (pinned for overlap): dem[i] or dirs[i] (pass NULL for the
 * array not used), w[i] (w NULL when wtype is FA_W_NONE), acc[i] (rows x
 * cols of atype each).  Entries may repeat (the same input twice; an output
 * twice gets the later raster).  Two device buffer sets: raster i+1 uploads
 * on one copy stream and raster i-1 downloads on another (PCIe is full
 * duplex) while raster i runs on the device -- the throughput of a queue of
 * rasters is bounded by the larger copy direction, not their sum.  The
 * rasters are independent problems (P:L49-57 per raster); the batch is the
 * host-side pipeline around them.  count == 0: FA_OK; device pointers:
 * FA_E_ARG.  On an error in raster i the message starts "raster i:",
 * outputs of rasters < i are complete, later ones undefined.  fa_get_stats
 * after the call: cells / graph_nodes / launches summed, ms_total the whole
 * batch (first upload to last download), ms_compute the device pipelines,
 * bytes_exchanged the PCIe bytes. */
FA_API fa_status fa_accumulate_batch(fa_ctx* ctx, int count, int64_t rows, int64_t cols,
                                     const float* const* dem, float nodata, const uint8_t* const* dirs,
                                     const void* const* w, fa_wtype wtype, void* const* acc, fa_atype atype);

/* fa_accumulate_streamed with absorption (N3, see fa_accumulate_absorb):
 * alpha is a HOST buffer streamed with the strips (4 more bytes per cell and
 * pass); output f64, w none or f32. */
FA_API fa_status fa_accumulate_absorb_streamed(fa_ctx* ctx, int64_t rows, int64_t cols,
                                               const float* dem, float nodata, const uint8_t* dirs,
                                               const void* w, fa_wtype wtype, const float* alpha,
                                               double* acc, int64_t strip_rows);

/* H4/H5 intermediates for tests and tools: number of tile perimeter slots
 * for a rows x cols raster under the context's tiling (tiles row-major,
 * slots per tile in clockwise perimeter order from the tile's top-left,
 * P = 2h+2w-4, or h*w for a 1-wide tile). */
FA_API int64_t fa_perimeter_slots(const fa_ctx* ctx, int64_t rows, int64_t cols);

/* Run the tiled method and return, per tile perimeter slot ("(a) its
 * flow direction F, (b) its flow accumulation A, and (c) its link L"):
 *   links   (u32): Alg. 2 FollowPath: the perimeter index of
 *                  the exit cell where the slot's in-tile path leaves the
 *                  tile, 0xFFFFFFFE FlowExternal, 0xFFFFFFFF FlowTerminates;
 *   tile_acc(atype): A_T, the tile-local accumulation (Alg. 1 on the tile);
 *   offsets (atype): x, the external inbound flow the global solve returns
 *                  to the slot (P:L220 A', read as a_in, D11).
 * Any of the three may be NULL.  Same inputs as fa_accumulate; `acc` (may be
 * NULL) receives the final accumulation. */
FA_API fa_status fa_perimeter_records(fa_ctx* ctx, int64_t rows, int64_t cols, const float* dem,
                               float nodata, const uint8_t* dirs, const void* w, fa_wtype wtype,
                               fa_atype atype, uint32_t* links, void* tile_acc, void* offsets,
                               void* acc);

/* Multi-GPU (H7): rank 0 calls fa_nccl_unique_id and broadcasts the 128
 * bytes (e.g. with torch.distributed); every rank then calls
 * fa_accumulate_dist collectively with identical global_rows, cols, nranks,
 * wtype, atype and tiling.  Rank r owns rows [row_begin, row_begin +
 * local_rows) (strips contiguous, ordered by rank, each a multiple of the
 * tile height except the last).  dem/dirs/w/acc are the rank's strip.
 * Collectives (dist.cu): C0 a gather of every rank's arguments (all ranks
 * agree on the partition or all return the same error before data moves),
 * C1 two halo rows of z (DEM input) or one row of codes to/from each
 * neighbour strip, C3 a gather of the status flags and integer weight sums
 * (bitwise OR; u32 overflow, D10), C2 ONE all-gather of fixed-size padded
 * buffers of the strips' tile perimeter records, and a final
 * status gather.  The perimeter graph is solved redundantly on every rank
 * (no second exchange).  With a DEM every strip but the last needs >= 2
 * rows.  A rank-local failure (allocation, a kernel error) is reported to
 * every rank at the next status gather, so all ranks return. */
FA_API fa_status fa_nccl_unique_id(void* out128);
FA_API fa_status fa_accumulate_dist(fa_ctx* ctx, const void* nccl_id128, int rank, int nranks,
                             int64_t global_rows, int64_t cols, int64_t row_begin,
                             int64_t local_rows, const float* dem, float nodata,
                             const uint8_t* dirs, const void* w, fa_wtype wtype, void* acc,
                             fa_atype atype);

/* fa_accumulate_dist with absorption (N3, see fa_accumulate_absorb): alpha
 * is the rank's strip (device buffer, f32 in [0,1]), output f64, w none or
 * f32.  The tile records all-gather also carries each slot's alpha path
 * factor; collective like fa_accumulate_dist. */
FA_API fa_status fa_accumulate_absorb_dist(fa_ctx* ctx, const void* nccl_id128, int rank, int nranks,
                                           int64_t global_rows, int64_t cols, int64_t row_begin,
                                           int64_t local_rows, const float* dem, float nodata,
                                           const uint8_t* dirs, const void* w, fa_wtype wtype,
                                           const float* alpha, double* acc);

/* The multi-GPU path with a loopback transport: nranks ranks of
 * fa_accumulate_dist run as host threads inside this call, rank q on
 * ctxs[q] (one distinct context per rank, each with its own stream; the
 * contexts may share a device), exchanging halo rows, status flags and the
 * perimeter records by stream-ordered device copies and events instead of
 * NCCL.  Every rank executes the same code as in fa_accumulate_dist (C0
 * argument agreement, C1 halo rows, phase A, C3 status, C2 record
 * all-gather, the producer graph G2, phase B); only the transport differs
 * (P:L215).  Per-rank arrays of nranks entries: row_begin,
 * local_rows, dem / dirs / w / alpha (each array NULL when that input is
 * absent), acc (required); every pointer is the rank's strip on its
 * context's device.  alpha != NULL selects absorption (f64 output, w none
 * or f32).  Returns FA_OK or the first failing rank's status (its message in
 * fa_last_error of that rank's context); each context keeps its rank's
 * statistics. */
FA_API fa_status fa_accumulate_dist_loopback(fa_ctx* const* ctxs, int nranks, int64_t global_rows,
                                             int64_t cols, const int64_t* row_begin,
                                             const int64_t* local_rows, const float* const* dem,
                                             float nodata, const uint8_t* const* dirs,
                                             const void* const* w, fa_wtype wtype,
                                             const float* const* alpha, void* const* acc,
                                             fa_atype atype);

/* Per-phase statistics of the last call (device-timed with CUDA events).
 * fa_get_stats copies min(out_bytes, sizeof(fa_stats)) bytes into `out`
 * (fields are only ever appended, so a caller built against an older,
 * shorter fa_stats receives its prefix); out_bytes <= 0 -> FA_E_ARG. */
typedef struct {
  double ms_total, ms_pass1, ms_graph, ms_pass2, ms_exchange;
  int64_t cells, blocks, graph_nodes, tile_nodes;
  int64_t peel_rounds, contract_levels, jump_rounds;
  int64_t bytes_exchanged;
  int64_t launches; /* kernels launched by the call */
  double ms_d8;     /* the standalone D8 kernel (single-device path; 0 when D8 is fused into pass 1) */
  double ms_block;  /* the pass-1 block kernel alone (k_pass1), last strip */
  double ms_compute; /* fa_accumulate_batch: the rasters' device pipelines, summed (ms_total: the whole
                        batch, first upload to last download) */
} fa_stats;
FA_API fa_status fa_get_stats(const fa_ctx* ctx, void* out, int64_t out_bytes);

#ifdef __cplusplus
}
#endif
#endif /* FA_H */
