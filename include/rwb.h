/*
 * rwb.h — C ABI of the B200 hierarchical random-walker library (librwb.so).
 *
 * This is the drop-in boundary under the reference's compute-graph operator
 * API (`OperatorNode.kernel(h, input_arrays, out)`,
 * pkg/src/chunkcast/graph.py:18-51, driven by `_generic_compute_body`,
 * pkg/src/chunkcast/engine.py:999-1076).  Every entry point below replaces
 * one operator kernel of the reference (or, for the random walker, the
 * operator the reference's paper describes but the package leaves out,
 * SPEC.md:8).  The Python binding is `paper_2509_26213_b200/_native.py`
 * (ctypes); INTEGRATION.md shows the binding a reference maintainer adds.
 *
 * Conventions
 *  - Plain pointers and sizes only.  All array pointers are DEVICE pointers
 *    (cudaMalloc / torch CUDA storage) unless stated otherwise; the caller
 *    owns all memory, including the solver workspace.
 *  - Arrays are dense row-major with the LAST dimension fastest, like the
 *    reference's chunk payloads (model.py:3-6).  `size[0]` is the slowest
 *    dimension (TensorMetaData.size order, model.py:98-117).  ndim is 2 or 3
 *    (the LOD kernel also takes 1).
 *  - Every call is stream-ordered on `stream` (a cudaStream_t, NULL = legacy
 *    default stream) and reentrant: distinct host threads may call with
 *    distinct streams.  The only blocking call is rwb_solve_level, which
 *    polls convergence on its own stream.
 *  - Return value: RWB_OK (0) on success, a negative RWB_ERR_* code on
 *    failure; rwb_last_error() then returns a thread-local message.
 */
#ifndef RWB_H
#define RWB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RWB_ABI_VERSION 2

enum {
  RWB_OK = 0,
  RWB_ERR_INVALID = -1,     /* bad argument (shape, pointer, parameter) */
  RWB_ERR_CUDA = -2,        /* CUDA runtime error (message has the cause) */
  RWB_ERR_WORKSPACE = -3,   /* workspace too small */
  RWB_ERR_UNSUPPORTED = -4, /* no sm_100 device / unsupported configuration */
};

/* Geometry of one pyramid level and its brick (chunk) grid.
 * Bricks cover [origin + h*brick, origin + (h+1)*brick) ∩ [0, size) per
 * dimension; origin = 0 gives the reference's chunk grid
 * (TensorMetaData.chunk_grid_dims / chunk_logical_region, model.py:125-170).
 * brick == size makes the whole level one brick (the coarsest-level solve). */
typedef struct {
  int32_t ndim;
  int32_t reserved;
  int64_t size[3];
  int64_t brick[3];
  int64_t origin[3]; /* each in (-brick, 0] */
} rwb_geometry_t;

typedef struct {
  float beta;          /* edge weight exp(-beta * dI^2) */
  float min_weight;    /* lower clamp of every edge weight */
  float tol;           /* per-brick stop: ||r|| <= tol * ||b|| (Jacobi-scaled system) */
  int32_t max_iter;    /* per-brick iteration cap */
  int32_t check_every; /* iterations per convergence poll (0 = library default) */
  int32_t flags;       /* RWB_SOLVE_* */
} rwb_solve_params_t;

#define RWB_SOLVE_NO_GRAPH 1  /* streaming solver: launch iterations directly, not via a CUDA graph */
#define RWB_SOLVE_STREAMING 2 /* force the streaming solver even where the brick-resident one applies */
#define RWB_SOLVE_NO_COOP 4   /* whole-level solves: graph-launched passes instead of one cooperative kernel */
#define RWB_SOLVE_CLUSTER16 8 /* brick-resident solver: 16-CTA clusters, 2 CTAs/SM (default 8-CTA, 1 CTA/SM) */
#define RWB_SOLVE_SPLIT_Z 16  /* brick-resident solver: 8-CTA clusters with 512 threads x 8 voxels per CTA */
#define RWB_SOLVE_SETUP2 32   /* build the system with the two-kernel setup instead of the fused per-brick one */
/* Two-phase use of the brick-resident engine (resident path only): SETUP_ONLY builds the level's
   system in `workspace` (and finishes the bricks the setup settles); a later call with the SAME
   arguments and NO_SETUP solves it.  Lets a caller build slab k+1's system on one stream while
   slab k solves on another (device.hierarchical_random_walker, level0_chunks). */
#define RWB_SOLVE_SETUP_ONLY 128
#define RWB_SOLVE_NO_SETUP 256
/* `stats` points to device-accessible memory (device or mapped pinned host memory), filled
   by a kernel on `stream` with no host synchronisation (brick-resident / cooperative paths never
   block the host then; cg_ms from %globaltimer around the solve launches). */
#define RWB_SOLVE_STATS_DEVICE 512
/* brick-resident solver: 4-CTA clusters (8 planes x 8192 voxels per CTA, scaled weights in tensor memory) */
#define RWB_SOLVE_CLUSTER4 1024

/* whole-level (single-brick) solves: Jacobi-PCG (the cooperative kernel, or the graph-launched
   passes with NO_COOP) instead of the default multigrid-preconditioned CG */
#define RWB_SOLVE_NO_MG 2048

/* brick-resident 4-CTA solver: plain Jacobi-PCG instead of the default coarse-corrected PCG
   (Jacobi + an additive correction on the brick's 8^3-voxel aggregates) */
#define RWB_SOLVE_NO_COARSE 4096

/* whole-level solves: multigrid-PCG at any size (default: levels of at least 2^19 voxels; on
   smaller ones the V-cycle's per-iteration barriers cost more than the iterations it saves) */
#define RWB_SOLVE_MG 8192

/* Solver paths (rwb_solve_stats_t.path) */
#define RWB_PATH_STREAMING 0 /* brick-batched CG, state in HBM, 2 launches per iteration */
#define RWB_PATH_RESIDENT 1  /* CG state on chip: one 32^3 brick per 4-CTA cluster (3-D, default), one 64^2 tile per CTA (2-D) */
#define RWB_PATH_COOPERATIVE 2 /* single-brick (whole-level) Jacobi-PCG: all iterations in one cooperative kernel */
#define RWB_PATH_MULTIGRID 3   /* single-brick (whole-level) solve: V-cycle-preconditioned CG, one cooperative kernel */

typedef struct {
  int64_t bricks;          /* bricks solved by this call */
  int64_t converged;       /* reached tol */
  int64_t not_converged;   /* hit max_iter */
  int64_t zero_rhs;        /* ||b|| == 0: exact solution 0, no iterations */
  int64_t iterations_max;  /* max over bricks */
  int64_t iterations_sum;  /* sum over bricks (for algorithmic-byte accounting) */
  int64_t unknowns;        /* unseeded voxels solved for */
  int32_t sweeps;          /* streaming: CG iterations launched (iterations_max rounded up to a poll) */
  float cg_ms;             /* device time of the solve launches (CUDA events on `stream`): streaming =
                              the CG iteration kernels; resident = the whole on-chip brick solve */
  int32_t path;            /* RWB_PATH_* that ran */
  int32_t reserved;
  int64_t unknown_iterations; /* sum over bricks of unknowns x iterations: the PCG work done, in
                                 unknown-voxel iterations (algorithmic-byte accounting) */
} rwb_solve_stats_t;

int rwb_abi_version(void);
const char* rwb_last_error(void);
/* Process-wide count of librwb kernels launched so far (graph replays count
 * every kernel node).  Lets callers report how many of the library's kernels
 * ran inside a timed region. */
int64_t rwb_kernel_launches(void);
/* sm count and compute capability of the current device; RWB_ERR_UNSUPPORTED if not sm_100. */
int rwb_device_info(int32_t* sm_count, int32_t* cc_major, int32_t* cc_minor);

/* One LOD pyramid step, level k -> k+1:
 * f32(downsample_mean(f32(separable_conv(src, [.25,.5,.25]^d, clamp)))).
 * Replaces the separable_conv + downsample_mean pair that build_lod chains
 * per level (ops.py:714-727, kernels ops.py:503-530 and ops.py:642-661);
 * bit-identical to them (same float64 operation order).
 * dst has size ceil(size/2) per dimension. */
int rwb_lod_down_f32(int32_t ndim, const int64_t* size, const float* src, float* dst, void* stream);

/* Seed labels (0 none, 1 fg, 2 bg) of the next coarser level: a coarse voxel
 * is 1 (2) if one of its downsample_mean block children (ops.py:629-636) is
 * 1 (2) and none is 2 (1), else 0.  coarse has size ceil(size/2). */
int rwb_project_seeds_u8(int32_t ndim, const int64_t* size, const uint8_t* fine, uint8_t* coarse,
                         void* stream);

/* Coarse-to-fine prolongation: cell-centred multilinear, fine index g reads
 * parent coordinate g/2 - 1/4, clamped.  fine_size must satisfy
 * ceil(fine_size/2) == parent_size. */
int rwb_upsample_f32(int32_t ndim, const int64_t* parent_size, const float* parent,
                     const int64_t* fine_size, float* fine, void* stream);

/* Windowed prolongation for operator mode, where a chunk kernel only holds
 * the parent chunks around its brick: computes the fine voxels
 * [fine_origin, fine_origin + fine_window) of a level of size fine_size from
 * the parent window [parent_origin, parent_origin + parent_window) of a parent
 * level of size parent_size (taps use global coordinates, identical to
 * rwb_upsample_f32; the parent window must cover them). */
int rwb_upsample_window_f32(int32_t ndim, const int64_t* parent_size, const int64_t* parent_origin,
                            const int64_t* parent_window, const float* parent, const int64_t* fine_size,
                            const int64_t* fine_origin, const int64_t* fine_window, float* fine, void* stream);

/* Forward edge weights, lanes-last (the ElementType(F32, ndim) payload layout,
 * model.py:66-80): weights[i*ndim + k] = max(exp(-beta*(I_i - I_{i+e_k})^2), min_weight),
 * 0 where i+e_k is outside the volume. */
int rwb_edge_weights_f32(int32_t ndim, const int64_t* size, const float* volume, float beta,
                         float min_weight, float* weights, void* stream);

/* labels[i] = prob[i] > 0.5 (cast_array semantics of a boolean, ops.py:44-52). */
int rwb_labels_u8(int64_t n, const float* prob, uint8_t* labels, void* stream);

/* Factor-2 mean downsampling alone (build_lod(smooth=False), downsample_mean,
 * ops.py:611-676): per coarse element, float64 pairwise means along dimension
 * 0, then 1, then 2 of its 2^d block (a trailing odd element passing through),
 * rounded to f32.
 * dst has size ceil(size/2); ndim 1..3. */
int rwb_downsample_mean_f32(int32_t ndim, const int64_t* size, const float* src, float* dst, void* stream);
/* The same over a subset of the dimensions (downsample_mean(input, dims), ops.py:611-616): bit d of
 * dims_mask selects dimension d; unselected dimensions keep their size (dst[d] = size[d]). */
int rwb_downsample_mean_dims_f32(int32_t ndim, const int64_t* size, uint32_t dims_mask, const float* src, float* dst,
                                 void* stream);

/* Chunk payloads <-> dense tensor, for chunked tensor files (PLCT,
 * tensorfile.py:1-13).  A payload is the full chunk box (chunk[0..ndim)),
 * row-major, last dimension fastest, `elem_bytes` per element (scalar width x
 * lanes, lanes innermost: ElementType.payload_shape, model.py:78-80).  Border
 * chunks are clipped to `size` (chunk_logical_region, model.py:158-170).
 * Payload i of the batch belongs to chunk chunk_ids[i] (device int64,
 * row-major chunk index, model.py:138-146), or to chunk first + i when
 * chunk_ids is NULL.  ndim 1..4.
 *  scatter: the clipped part of each payload -> its region of `dense`
 *           (open_chunked's kernel, tensorfile.py:186-195, for a batch)
 *  gather : each chunk's region of `dense` -> its payload, zero outside the
 *           tensor (the payloads _ChunkWriter.write_chunk writes, :126-138) */
int rwb_chunks_scatter(int32_t ndim, const int64_t* size, const int64_t* chunk, int32_t elem_bytes,
                       const void* payloads, const int64_t* chunk_ids, int64_t first, int64_t n, void* dense,
                       void* stream);
int rwb_chunks_gather(int32_t ndim, const int64_t* size, const int64_t* chunk, int32_t elem_bytes,
                      const void* dense, const int64_t* chunk_ids, int64_t first, int64_t n, void* payloads,
                      void* stream);

/* Constant-chunk table of a scalar tensor (build_const_chunk_table, ops.py:777-816): table is
 * dense over the chunk grid (ceil(size/chunk) per dimension, row-major); each element is the
 * chunk's value when every element of its clipped region equals the first one (element-type
 * ==, so NaN never matches), else the sentinel: NaN for floats, the type maximum for integers
 * (sentinel_for, ops.py:770-774).  scalar_code as in PLCT files / model.py:24-29:
 * 0 u8, 1 i16, 2 u16, 3 f32, 4 f64.  ndim 1..4. */
int rwb_const_chunk_table(int32_t ndim, const int64_t* size, const int64_t* chunk, int32_t scalar_code,
                          const void* src, void* table, void* stream);

/* Volume raycaster (the reference's `raycast` / `render_frame` final frame, render.py:101-631):
 * marches n_px rays over an LOD pyramid of n_levels 3-D float32 levels (levels[k] device
 * pointers, sizes 3 per level, spacing 3 per level, finest spacing ascending).  rays: per pixel 10
 * doubles — origin (3), unit direction (3) from the reference's _pixel_rays, then its entry-exit
 * record (t_entry, t_exit, fp0, fps) as float32 values (t_entry = +inf: miss).  compositing 0 =
 * DVR (opacity-corrected front to back, early termination at 0.99), 1 = MOP; grey-ramp transfer
 * function [tf_lo, tf_hi].  out: n_px premultiplied RGBA, uchar4 (out_u8) or float4. */
int rwb_raycast(int32_t n_levels, const float* const* levels, const int64_t* sizes, const double* spacing,
                int64_t n_px, const double* rays, int32_t compositing, double sample_distance_factor,
                double lod_bias, double tf_lo, double tf_hi, int32_t out_u8, void* out, void* stream);

/* Nearest-neighbour pan/zoom view (the reference's viewer: _resample_nn / slice_view /
 * image_view, render.py:640-741): frame pixel (p0, p1) of the (frame_size[0], frame_size[1])
 * frame samples source element floor((p + 0.5) * scale + offset) per axis (float64 math), 0
 * outside the source.  The source is a 2-D image (src_ndim 2, slice_dim < 0) or the slice
 * slice_index along slice_dim of a 3-D level (the remaining axes in order, slice_node
 * semantics).  Elements are opaque elem_bytes-byte items (scalar width x lanes). */
int rwb_resample_nn(int32_t src_ndim, const int64_t* src_size, int32_t slice_dim, int64_t slice_index,
                    int32_t elem_bytes, const void* src, const int64_t* frame_size, const double* scale,
                    const double* offset, void* frame, void* stream);

/* Bytes of solver workspace for n_bricks bricks of `geom` (n_bricks < 0: all)
 * with the given RWB_SOLVE_* flags (the brick-resident path needs almost none). */
size_t rwb_solve_workspace_bytes(const rwb_geometry_t* geom, int64_t n_bricks, int32_t flags);

/* Random-walker solve of the listed bricks of one level.
 *  intensity : f32 level (size)         seeds : u8 level, 0/1/2
 *  bound     : f32 level or NULL.  Values of the Dirichlet nodes outside a
 *              brick and the initial guess inside it (the upsampled parent
 *              level).  NULL only when the geometry has a single brick
 *              (coarsest level), initial guess 0.
 *  brick_list: device int32 row-major brick indices, or NULL for all bricks
 *              (n_bricks then ignored).  Listed bricks must be distinct.
 *  prob      : f32 level output; written only inside the listed bricks.  May
 *              alias `bound` on the streaming path only (all its reads of
 *              bound happen before any write); the brick-resident path
 *              solves bricks at different times and rejects aliasing.
 *  labels    : u8 level output (prob > 0.5) or NULL.
 *  stats     : host pointer or NULL.
 * Path: 3-D levels with 32^3 bricks and more than one brick run the
 * brick-resident solver (unless RWB_SOLVE_STREAMING); whole-level (coarsest,
 * single-brick) solves of at least 2^19 voxels (any size with RWB_SOLVE_MG) run
 * multigrid-preconditioned CG in one cooperative kernel, smaller ones (and
 * RWB_SOLVE_NO_MG) Jacobi-PCG, cooperative unless RWB_SOLVE_NO_COOP;
 * everything else runs the streaming solver with graph-launched passes.
 * Blocking on the host: returns when the listed bricks have converged (or hit
 * max_iter); all work is stream-ordered on `stream`. */
int rwb_solve_level(const rwb_geometry_t* geom, const float* intensity, const uint8_t* seeds,
                    const float* bound, const int32_t* brick_list, int64_t n_bricks,
                    const rwb_solve_params_t* params, float* prob, uint8_t* labels,
                    void* workspace, size_t workspace_bytes, rwb_solve_stats_t* stats,
                    void* stream);

#ifdef __cplusplus
}
#endif

#endif /* RWB_H */
