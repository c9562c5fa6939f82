/*
 * skycell_gpu.h -- C ABI of the B200-native SkyCell skyline path.
 *
 * Drop-in for the reference entry point
 *
 *   SkylineResult skycell::compute_skyline(const Dataset& ds, int rho, Mode mode,
 *                                          ThreadPool& pool, bool merge_cross_cell = true);
 *       (/root/reference/proj/include/skycell/refine.hpp:61-62,
 *        /root/reference/proj/src/refine.cpp:108-158)
 *
 * and its only library caller
 *
 *   SkylineResult skycell::quadrant_skyline(const Dataset&, std::span<const double> origin,
 *                                           int rho, Mode, ThreadPool&);
 *       (refine.hpp:66-68, refine.cpp:160-184)
 *
 * Plain pointers and sizes only; no C++ or torch types cross this boundary.
 * The C++ wrapper with the reference's exact signature and exception types is
 * include/skycell_gpu.hpp; the ctypes binding is paper_2107_09993_b200/skycell.py.
 *
 * Every entry point returns a status code and, on failure, writes the
 * reference's exception message into err (truncated to err_len).  The codes map
 * 1:1 onto the reference's exception taxonomy (proj/include/skycell/error.hpp:9-26).
 */
#ifndef SKYCELL_GPU_H_
#define SKYCELL_GPU_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum skycell_status {
  SKYCELL_OK = 0,
  SKYCELL_INPUT = 1,    /* skycell::InputError  (dataset.cpp:23-43)               */
  SKYCELL_CONFIG = 2,   /* skycell::ConfigError (grid.cpp:38-43)                  */
  SKYCELL_USAGE = 3,    /* skycell::UsageError  (refine.cpp:162-163)              */
  SKYCELL_IO = 4,       /* skycell::IoError                                       */
  SKYCELL_CUDA = 5,     /* CUDA runtime failure (no reference equivalent)         */
  SKYCELL_NCCL = 6,     /* collective failure  (no reference equivalent)          */
  SKYCELL_UNSUPPORTED = 7 /* valid for the reference, not (yet) for this build    */
};

/* Mode, refine.hpp:40.  Ids never depend on it; it only selects whether
 * per-layer candidate counts are reported (kSequential reports -1 except at
 * layer rho, refine.cpp:132-135). */
enum skycell_mode { SKYCELL_SEQUENTIAL = 0, SKYCELL_PARALLEL = 1 };

/* Mirrors SkylineResult minus the ids (refine.hpp:19-38).  keys[i] and
 * candidates[i] are |KS_{i+1}| and |CS_{i+1}| for i = 0..n_layers-1. */
typedef struct skycell_gpu_stats {
  double normalize_ms, grid_ms, shrink_ms, refine_ms, total_ms;
  uint64_t points_examined;
  int32_t n_layers;
  int32_t pad_;
  uint64_t keys[64];
  int64_t candidates[64];
  /* diagnostics beyond the reference's SkylineResult */
  uint64_t survivors_stream;   /* points leaving the streaming pass (K1)          */
  uint64_t survivors_filter;   /* points entering the exact dominance pass (K5)   */
  uint64_t kernel_launches;    /* kernels this call launched                      */
  double stream_kernel_ms;     /* CUDA-event time of the streaming kernel K1 alone */
  double filter_kernel_ms;     /* ... of the candidate filter K4 (K4a + K4b)      */
  double dominance_ms;         /* ... of the exact dominance pass K5 (build + query) */
} skycell_gpu_stats;

typedef struct skycell_gpu_ctx skycell_gpu_ctx;

/* Opaque per-device handle: device, stream, scratch buffers.  Not shared across
 * concurrent calls (callers serialise per handle; use one handle per thread). */
int skycell_gpu_create(int device, skycell_gpu_ctx** out, char* err, size_t err_len);
void skycell_gpu_destroy(skycell_gpu_ctx* ctx);

/* compute_skyline over n x d row-major coordinates.
 *   coords      host or device pointer (detected); n*d values
 *   dim_min/max host arrays of d doubles -- the declared normalisation range
 *               (Dataset::dim_min/dim_max, dataset.hpp:24-25)
 *   ids_out     host or device pointer with room for n uint32 ids; receives the
 *               skyline record ids in ascending order
 *   n_out       host pointer; receives the skyline size
 *   stats       optional (NULL)
 * The f32 entry point is the benchmark path: coords are widened to double
 * exactly as the reference would see them, so results are identical to the
 * reference fed Dataset{coords = (double)x, dim_min, dim_max}. */
int skycell_gpu_skyline_f64(skycell_gpu_ctx* ctx, const double* coords, uint64_t n, int d,
                            const double* dim_min, const double* dim_max, int rho, int mode,
                            int merge_cross_cell, uint32_t* ids_out, uint64_t* n_out,
                            skycell_gpu_stats* stats, char* err, size_t err_len);
int skycell_gpu_skyline_f32(skycell_gpu_ctx* ctx, const float* coords, uint64_t n, int d,
                            const double* dim_min, const double* dim_max, int rho, int mode,
                            int merge_cross_cell, uint32_t* ids_out, uint64_t* n_out,
                            skycell_gpu_stats* stats, char* err, size_t err_len);

/* quadrant_skyline (refine.cpp:160-184): skyline of the points >= origin in every
 * dimension, renormalised by the subset's own min/max; ids refer to the
 * original records.  origin has origin_len doubles (must equal d). */
int skycell_gpu_quadrant_f64(skycell_gpu_ctx* ctx, const double* coords, uint64_t n, int d,
                             const double* origin, int origin_len, int rho, int mode,
                             uint32_t* ids_out, uint64_t* n_out, skycell_gpu_stats* stats,
                             char* err, size_t err_len);

/* Bind the context to a caller's CUDA stream (a cudaStream_t; 0 is the
 * legacy default stream), or back to its own stream with use_own = 1.  Every
 * kernel and copy of later calls is enqueued on it, so collectives the caller
 * issues on the same stream (the sharded query below) are ordered without
 * host synchronisation. */
int skycell_gpu_set_stream(skycell_gpu_ctx* ctx, void* stream, int use_own);

/* ---- Sharded query over G devices (one process / context per device).
 * No reference equivalent: the reference is single-process
 * (SURVEY.md §8(e)); the result equals compute_skyline over the
 * concatenation of all shards.  Rank g holds records [id_base, id_base + n)
 * of the global dataset.  The caller performs the two exchanges (NCCL over
 * NVLink in paper_2107_09993_b200/dist.py):
 *
 *   shard_begin        K0 + K1 on the shard; *occ_bytes = size of the
 *                      occupancy region to exchange
 *   shard_export_occ   copy this rank's occupancy region to dev_dst
 *      -- caller: all-gather the regions (rank order) into one buffer --
 *   shard_prune        OR the world regions (K2), prune against the global
 *                      occupancy (K3, K4), local skyline (K5);
 *                      *local_count = its size
 *      -- caller: all-gather the counts; max_count = their maximum --
 *   shard_block_bytes  bytes of one rank's padded local-skyline block
 *   shard_pack         write this rank's block (padded to max_count)
 *      -- caller: all-gather the blocks (rank order) --
 *   shard_finish       this rank's local-skyline points against the union;
 *                      writes this rank's part of the global skyline
 *                      (global ids, ascending) to ids_out; stats hold the
 *                      global per-layer counts and the LOCAL points_examined.
 * coords_f32 selects float (1) or double (0) coordinates.  dim_min/dim_max are
 * the GLOBAL declared range (identical on every rank). */
int skycell_gpu_shard_begin(skycell_gpu_ctx* ctx, const void* coords, int coords_f32, uint64_t n, int d,
                            const double* dim_min, const double* dim_max, int rho, int mode, uint64_t id_base,
                            uint64_t* occ_bytes, char* err, size_t err_len);
int skycell_gpu_shard_export_occ(skycell_gpu_ctx* ctx, void* dev_dst, char* err, size_t err_len);
int skycell_gpu_shard_prune(skycell_gpu_ctx* ctx, const void* dev_gathered, int world, uint64_t* local_count,
                            char* err, size_t err_len);
uint64_t skycell_gpu_shard_block_bytes(skycell_gpu_ctx* ctx, uint64_t max_count);
int skycell_gpu_shard_pack(skycell_gpu_ctx* ctx, void* dev_dst, uint64_t max_count, char* err, size_t err_len);
int skycell_gpu_shard_finish(skycell_gpu_ctx* ctx, const void* dev_recv, int world, uint64_t max_count, int rank,
                             uint64_t own_count, uint32_t* ids_out, uint64_t* n_out, skycell_gpu_stats* stats,
                             char* err, size_t err_len);

/* ---- Single-process multi-device query ("skycell_gpu_create(
 * int n_gpus, ...)"; §8(e)).  One handle owns a context per listed device,
 * shards the records by index and runs the sharded protocol above itself:
 * the exchanges are device-to-device copies (NVLink / NVSwitch peer access
 * when available), one host thread per device.  Same contract as
 * skycell_gpu_skyline_f64 / _f32 (the reference's compute_skyline,
 * refine.hpp:61-62): ids ascending, per-layer counts, points_examined.
 * Queries sharding cannot serve (one device, n < devices, merge_cross_cell =
 * 0, a sparse layer rho) run on the first device.  The same device may be
 * listed more than once (tests run G contexts on one GPU). */
typedef struct skycell_gpu_multi skycell_gpu_multi;
int skycell_gpu_multi_create(const int* devices, int n_devices, skycell_gpu_multi** out, char* err,
                             size_t err_len);
void skycell_gpu_multi_destroy(skycell_gpu_multi* m);
int skycell_gpu_multi_size(const skycell_gpu_multi* m);
/* The context of device slot g (e.g. for quadrant queries); owned by m. */
skycell_gpu_ctx* skycell_gpu_multi_context(skycell_gpu_multi* m, int g);
int skycell_gpu_multi_skyline_f64(skycell_gpu_multi* m, const double* coords, uint64_t n, int d,
                                  const double* dim_min, const double* dim_max, int rho, int mode,
                                  int merge_cross_cell, uint32_t* ids_out, uint64_t* n_out,
                                  skycell_gpu_stats* stats, char* err, size_t err_len);
int skycell_gpu_multi_skyline_f32(skycell_gpu_multi* m, const float* coords, uint64_t n, int d,
                                  const double* dim_min, const double* dim_max, int rho, int mode,
                                  int merge_cross_cell, uint32_t* ids_out, uint64_t* n_out,
                                  skycell_gpu_stats* stats, char* err, size_t err_len);

/* ---- MultiLayerGrid drop-in (proj/include/skycell/grid.hpp:33-70,
 * proj/src/grid.cpp:35-140).  Built on the device from a normalised PointSet
 * (coords n x d doubles in [0, 1 - 2^-32], ids n uint32 or NULL for 0..n-1;
 * host or device pointers): points sorted by the Z-order key of their
 * layer-rho cell, ties by input position (grid.cpp:47-54); the contiguous
 * point range of every non-empty layer-rho cell; occupancy of layers
 * 0..rho-1 by child-OR.  ConfigError on the reference's rho budget
 * (grid.cpp:38-43).  Cells are named by their linear index
 * (CellIndex::linear_index, cell.hpp:102-107).
 *   grid_points          the sorted PointSet (coords, ids; host or device)
 *   grid_nonempty_count  MultiLayerGrid::nonempty_count(layer)
 *   grid_nonempty_cells  nonempty_cells(layer): ascending linear indices
 *                        (enumeration order, lex_less); count entries
 *   grid_lookup          batch of `count` cells of one layer: occupied
 *                        (occupied(), grid.cpp:105-113) and, at layer rho,
 *                        [begin, end) (range(), grid.cpp:115-119; empty cells
 *                        0, 0); begin/end at another layer is UsageError
 *                        "range: only layer-rho cells carry point ranges". */
typedef struct skycell_gpu_grid skycell_gpu_grid;
int skycell_gpu_grid_build(skycell_gpu_ctx* ctx, const double* coords, const uint32_t* ids, uint64_t n, int d,
                           int rho, skycell_gpu_grid** out, char* err, size_t err_len);
void skycell_gpu_grid_destroy(skycell_gpu_grid* g);
int skycell_gpu_grid_shape(const skycell_gpu_grid* g, uint64_t* n, int* d, int* rho);
uint64_t skycell_gpu_grid_nonempty_count(const skycell_gpu_grid* g, int layer);
int skycell_gpu_grid_points(skycell_gpu_grid* g, double* coords_out, uint32_t* ids_out, char* err, size_t err_len);
int skycell_gpu_grid_nonempty_cells(skycell_gpu_grid* g, int layer, uint64_t* lin_out, char* err, size_t err_len);
int skycell_gpu_grid_lookup(skycell_gpu_grid* g, int layer, const uint64_t* lin, uint64_t count, uint8_t* occupied,
                            uint32_t* begin, uint32_t* end, char* err, size_t err_len);

/* On-device synthetic data with the reference generator's streams
 * (skycell::generate, datagen.cpp:62-87): dist 0 independent, 1 correlated,
 * 2 anti-correlated.  kind 0 writes n*d raw doubles, kind 1 writes n*d floats
 * quantised to the 2^-24 grid (x = (float)(floor(v * 2^24) * 2^-24), the
 * benchmark input rule of BASELINE.md §2).  dev_out is a device pointer. */
int skycell_gpu_generate(skycell_gpu_ctx* ctx, int dist, uint64_t n, int d, uint64_t seed, int kind,
                         void* dev_out, char* err, size_t err_len);
/* Records [begin, begin + count) of the same n-record dataset (a shard). */
int skycell_gpu_generate_range(skycell_gpu_ctx* ctx, int dist, uint64_t n, int d, uint64_t seed, int kind,
                               uint64_t begin, uint64_t count, void* dev_out, char* err, size_t err_len);

/* ---- SKYC dataset files (skycell::read_bin / write_bin, datagen.cpp:185-221;
 * declared at proj/include/skycell/datagen.hpp:86-87).
 * Format: "SKYC" | u32 version 1 | u32 d | u64 n | n*d f64, little-endian.
 *
 *   skycell_bin_header   host only: validates the header exactly as read_bin
 *                        does (bad magic, unsupported version, bad
 *                        dimensionality -> SKYCELL_INPUT; cannot open ->
 *                        SKYCELL_IO) and returns n and d
 *   skycell_gpu_read_bin streams the coordinates into dev_coords (a device
 *                        buffer of cap_values doubles) through pinned staging
 *                        and reduces dim_min / dim_max on the device
 *                        (Dataset::compute_minmax, dataset.cpp:10-20); a short
 *                        file is "<path>: truncated file" (SKYCELL_INPUT).
 *                        n >= 2^32 is rejected (the reference truncates
 *                        Dataset::n to uint32).
 *   skycell_gpu_write_bin writes n x d doubles from host or device memory. */
int skycell_bin_header(const char* path, uint64_t* n, int* d, char* err, size_t err_len);
int skycell_gpu_read_bin(skycell_gpu_ctx* ctx, const char* path, double* dev_coords, uint64_t cap_values,
                         uint64_t* n_out, int* d_out, double* dim_min, double* dim_max, char* err, size_t err_len);
int skycell_gpu_write_bin(skycell_gpu_ctx* ctx, const char* path, const double* coords, uint64_t n, int d,
                          char* err, size_t err_len);

/* MultiLayerGrid::default_rho (grid.cpp:30-33). */
int skycell_default_rho(uint64_t n, int d);

/* Host-side argument validation in the reference's order (dataset.cpp:23-24,
 * grid.cpp:38-43) without touching a device; used by CPU tests.  Non-finite
 * coordinates are a device-side check and are not covered here. */
int skycell_validate(uint64_t n, int d, int rho, char* err, size_t err_len);

/* Build identification string (arch, version). */
const char* skycell_gpu_version(void);

#ifdef __cplusplus
}
#endif

#endif /* SKYCELL_GPU_H_ */
