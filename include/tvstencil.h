/*
 * tvstencil.h — C ABI of libtvstencil.so, the B200 (sm_100a) kernel library
 * behind the drop-in `tvstencil` stencil-run functions.
 *
 * The reference is pure Python; every entry point below
 * replaces the body of one reference function, and a ctypes binding
 * (paper_2010_04868_b200/_native.py) is the "FFI" that
 * calls it.  Plain pointers, sizes and POD structs only; no torch types.
 *
 *   reference interface                                  -> entry point
 *   kernels1d.py:89-93   heat1d_temporal(grid, steps)       -> tvs_run (JACOBI, dim 1)
 *   kernels1d.py:96-103  gs1d_temporal(grid, steps)         -> tvs_run (GAUSS_SEIDEL, dim 1)
 *   kernels_nd.py:38-45  jacobi2d/3d_temporal(grid, steps)  -> tvs_run (JACOBI, dim 2/3)
 *   kernels_nd.py:48-55  gs2d/3d_temporal(grid, steps)      -> tvs_run (GAUSS_SEIDEL, dim 2/3)
 *   baselines.py:43-49   jacobi_plane_update (one step)     -> tvs_jacobi_device(steps=1)
 *   cli.py:156-170       _bench_once (device-resident reps) -> tvs_plan_* API
 *   grid.py:127-133      fnv1a64                            -> tvs_fnv1a64
 *   baselines.py:52-66   life_plane_update (int32 Life)     -> tvs_life_run / tvs_life_device
 *   kernels/lcs.py:32-108 lcs_temporal(a, b) -> int          -> tvs_lcs / tvs_lcs_device
 *   tiling.py:347-371    execute_parallel(kernel, grid, sched) -> tvs_tiled_run / tvs_tiled_life
 *   tiling.py:374-406    lcs_blocked(a, b, sched)           -> tvs_lcs_tiled
 *
 * Arithmetic contract (baselines.py:3-7, 43-49; vec.py:296-298): taps are
 * evaluated in the order given (the caller passes StencilSpec.offsets()
 * order, i.e. sorted), first tap a multiply, every further tap a separately
 * rounded multiply and add.  fma_policy relaxes this only where stated.
 *
 * Status codes (mapped to the reference's exceptions by the binding):
 *   0 ok; 1 size (SizeError); 2 unsupported (UnsupportedError);
 *   3 invalid argument (ValueError); 4 CUDA error / no device (RuntimeError).
 * Every function is re-entrant; the last error message is thread-local.
 */
#ifndef TVSTENCIL_H
#define TVSTENCIL_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TVS_OK 0
#define TVS_ERR_SIZE 1
#define TVS_ERR_UNSUPPORTED 2
#define TVS_ERR_INVALID 3
#define TVS_ERR_CUDA 4

#define TVS_JACOBI 0
#define TVS_GAUSS_SEIDEL 1

#define TVS_MAX_TAPS 27

/* fma_policy */
#define TVS_FMA_NEVER 0 /* always mul then add: bit-exact vs the reference  */
#define TVS_FMA_EXACT 1 /* fuse only when every coefficient is 0 or +-2^k:
                           bit-identical except for subnormal products      */
#define TVS_FMA_ALLOW 2 /* fuse always (rel. error ~1e-15, tolerance mode) */

/* gs_order (Gauss-Seidel update order) */
#define TVS_GS_LEXICOGRAPHIC 0 /* row-major in-place loop (model.py:150-156) */
#define TVS_GS_REFERENCE 1     /* anti-diagonal gather/scatter (baselines.py:83-107) */

/* algo */
#define TVS_ALGO_AUTO 0
#define TVS_ALGO_NAIVE 1    /* one step per launch (Jacobi) / hyperplane (GS) */
#define TVS_ALGO_BLOCKED 2  /* temporal blocking / warp pipelines          */

/* One stencil: StencilSpec (model.py:76-132) flattened.
 * offsets[k] / coeffs[k] in evaluation order (StencilSpec.offsets()). */
typedef struct tvs_stencil {
  int32_t dim;    /* 1..3 */
  int32_t kind;   /* TVS_JACOBI | TVS_GAUSS_SEIDEL */
  int32_t ntaps;  /* 1..27 */
  int32_t radius; /* must be 1 */
  int32_t offsets[TVS_MAX_TAPS][3];
  double coeffs[TVS_MAX_TAPS];
  double boundary; /* constant Dirichlet value of every non-interior cell */
} tvs_stencil;

/* Host array in the reference Grid layout (grid.py:27-37): a C-contiguous
 * padded array of `shape`, interior origin at `offset` on every axis. */
typedef struct tvs_layout {
  int32_t dim;
  int32_t pad_;
  int64_t extents[3];
  int64_t shape[3];
  int64_t offset;
} tvs_layout;

/* tvs_exec.flags */
#define TVS_EXEC_EMULATE_SHARDS 1 /* n_gpus shards may share devices (round
                                     robin from `device`): the one-GPU test
                                     form of the sharded path */

typedef struct tvs_exec {
  int32_t device;         /* CUDA ordinal (first device of a sharded run) */
  int32_t fma_policy;     /* TVS_FMA_* */
  int32_t temporal_depth; /* 0 = auto */
  int32_t gs_order;       /* TVS_GS_* */
  int32_t algo;           /* TVS_ALGO_* */
  int32_t n_gpus;         /* 0/1: one GPU.  N > 1: 2D/3D Jacobi (star/box)
                             is split into N axis-0 slabs on devices
                             device .. device+N-1; 1D and
                             Gauss-Seidel run on `device` ("replicas only") */
  int32_t flags;          /* TVS_EXEC_* */
  int32_t reserved;
} tvs_exec;

/* Device layout of one (local) block: last axis padded by 32 elements on each
 * side (256-byte aligned interior rows), other axes by one halo cell. */
typedef struct tvs_geometry {
  int32_t dim;
  int32_t pad_;
  int64_t extents[3];    /* local interior extents (axis 0 incl. ghost rows) */
  int64_t strides[3];    /* element strides of axes 0..dim-1 (last = 1)   */
  int64_t origin;        /* element index of interior (0,..,0)           */
  int64_t alloc_elems;   /* allocation size in elements                  */
  int64_t axis0_offset;  /* global axis-0 index of local position 0      */
  int64_t axis0_global;  /* global axis-0 extent (Dirichlet edges)       */
} tvs_geometry;

/* ---- one-call path: host Grid in, host Grid out (ctypes drop-in) ---------
 * Uploads the interior of `in`, runs `steps` updates on the GPU, downloads
 * the interior into `out` (pads/halo of `out` untouched).  `in == out` is
 * allowed (Gauss-Seidel runs in place).  Device buffers are cached per
 * thread and geometry. */
int tvs_run(const tvs_stencil* st, const tvs_layout* lay, const double* in, double* out,
            int64_t steps, const tvs_exec* ex);

/* ---- problem-struct form (the SURVEY.md §8(b) signatures) --------------
 * One struct for the stencil and the host Grid layout; the same work as
 * tvs_run.  tvs_gauss_seidel runs in place; order = TVS_GS_*. */
typedef struct tvs_problem {
  int32_t dim;                     /* 1..3 */
  int32_t ntaps;                   /* 1..27 */
  int64_t extents[3];              /* interior extents */
  int32_t radius;                  /* 1 */
  int32_t pad_;
  double boundary;                 /* Dirichlet value (grid.boundary) */
  int32_t offsets[TVS_MAX_TAPS][3]; /* StencilSpec.offsets() order */
  double coeffs[TVS_MAX_TAPS];
  int64_t padded_shape[3];         /* Grid.data.shape */
  int64_t offset;                  /* Grid.offset */
} tvs_problem;
int tvs_jacobi(const tvs_problem* p, const double* in_padded, double* out_padded, int64_t steps, const tvs_exec* ex);
int tvs_gauss_seidel(const tvs_problem* p, double* inout_padded, int64_t steps, int32_t order, const tvs_exec* ex);

/* ---- plan path: device-resident repetitions (cli.py:198-227 timing) ----- */
typedef struct tvs_plan tvs_plan;
int tvs_plan_create(const tvs_stencil* st, int32_t dim, const int64_t extents[3], const tvs_exec* ex,
                    tvs_plan** out);
int tvs_plan_upload(tvs_plan* p, const tvs_layout* lay, const double* host);
int tvs_plan_download(tvs_plan* p, const tvs_layout* lay, double* host);
int tvs_plan_run(tvs_plan* p, int64_t steps);            /* async on the plan stream */
int tvs_plan_synchronize(tvs_plan* p);
/* device time of the last tvs_plan_run (CUDA events on the plan stream), ms */
int tvs_plan_last_ms(tvs_plan* p, float* ms);
/* launches issued by the last tvs_plan_run (your kernels only) */
int tvs_plan_last_launches(tvs_plan* p, int64_t* n);
/* the plan's CUDA stream (cudaStream_t), e.g. for torch.cuda.ExternalStream */
int tvs_plan_stream(tvs_plan* p, void** stream);
int tvs_plan_destroy(tvs_plan* p);

/* ---- sharded Jacobi: axis-0 slabs across GPUs ----------
 * A shard holds the owned rows [row_begin, row_end) of a global 2D/3D grid
 * plus `ghost` (= temporal depth) rows on each side, on one device.  A pass
 * of up to `ghost` levels computes the owned rows and the same kernel stores
 * the rows that are a neighbour's ghost rows straight into the neighbour's
 * buffer through peer memory (NVLink P2P stores: the halo exchange is fused
 * into the compute kernel).  Passes are ordered by pass counters that the
 * neighbours write into each other's memory and stream waits
 * (cuStreamWaitValue32) — no host synchronisation between passes.
 * Connect shards of one process with tvs_shard_connect_local; one process
 * per GPU exchanges tvs_shard_export handles (CUDA IPC) and calls
 * tvs_shard_connect.  Every shard of a group must run the same step counts;
 * upload / download only while every shard of the group is idle.
 * Replaces nothing in the reference (no distributed path); the
 * single-process caller shape is tiling.execute_parallel
 * (tiling.py:347-371). */
typedef struct tvs_shard tvs_shard;
typedef struct tvs_shard_handle {
  unsigned char bytes[256];
} tvs_shard_handle;
int tvs_shard_create(const tvs_stencil* st, int32_t dim, const int64_t global_extents[3], int32_t n_shards,
                     int32_t index, const tvs_exec* ex, tvs_shard** out);
int tvs_shard_info(const tvs_shard* s, int64_t* row_begin, int64_t* row_end, int32_t* ghost, int32_t* device);
int tvs_shard_export(tvs_shard* s, tvs_shard_handle* h);
/* left == NULL for shard 0, right == NULL for the last shard */
int tvs_shard_connect(tvs_shard* s, const tvs_shard_handle* left, const tvs_shard_handle* right);
int tvs_shard_connect_local(tvs_shard* s, tvs_shard* left, tvs_shard* right);
/* host Grid of the WHOLE grid (reference layout): the shard copies its rows */
int tvs_shard_upload(tvs_shard* s, const tvs_layout* global_lay, const double* host);
int tvs_shard_download(tvs_shard* s, const tvs_layout* global_lay, double* host);
int tvs_shard_run(tvs_shard* s, int64_t steps); /* async on the shard stream */
int tvs_shard_synchronize(tvs_shard* s);
int tvs_shard_last_ms(tvs_shard* s, float* ms);
int tvs_shard_last_launches(tvs_shard* s, int64_t* n);
int tvs_shard_stream(tvs_shard* s, void** stream);
int tvs_shard_destroy(tvs_shard* s);

/* ---- device path: caller-owned device buffers (halo-exchange module) ---- */
int tvs_geometry_init(int32_t dim, const int64_t extents[3], int64_t axis0_offset, int64_t axis0_global,
                      tvs_geometry* g);
/* Fill every non-interior cell of a device block with `value`. */
int tvs_fill_halo(const tvs_geometry* g, double* dev, double value, void* stream);
/* Jacobi: `steps` updates, ping-ponging src <-> dst (like the reference's
 * swap at baselines.py:122-124; a temporally blocked launch advances several
 * steps per swap); *result_in_dst reports which buffer holds the result.  Axis-0
 * positions outside [0, axis0_global) are boundary; positions outside the
 * local block but inside the domain are ghost cells whose influence spreads
 * one cell per step (callers exchange `steps` ghost rows first). */
int tvs_jacobi_device(const tvs_stencil* st, const tvs_geometry* g, double* src, double* dst, int64_t steps,
                      const tvs_exec* ex, void* stream, int32_t* result_in_dst);
/* One temporally blocked pass (`steps` <= the kernel's depth: 2D <= 12, 3D
 * <= 2) writing only axis-0 rows [row_lo, row_hi) of dst: the interior /
 * edge split that lets a halo exchange overlap the interior compute. */
int tvs_jacobi_device_rows(const tvs_stencil* st, const tvs_geometry* g, const double* src, double* dst,
                           int64_t steps, const tvs_exec* ex, void* stream, int64_t row_lo, int64_t row_hi);
/* Gauss-Seidel in place on one device block (single GPU, no ghosts). */
int tvs_gauss_seidel_device(const tvs_stencil* st, const tvs_geometry* g, double* grid, int64_t steps,
                            const tvs_exec* ex, void* stream);
/* Host <-> device interior copies between the Grid layout and a geometry. */
int tvs_upload(const tvs_geometry* g, double* dev, const tvs_layout* lay, const double* host, void* stream);
int tvs_download(const tvs_geometry* g, const double* dev, const tvs_layout* lay, double* host, void* stream);

/* ---- integer kernels ------------------------------
 * Life-like automaton (StencilSpec.is_life, model.py): n = wrapping int32
 * sum over `offsets` (StencilSpec.offsets(): the box neighbours, centre
 * excluded); n in birth -> 1, else n in survive -> own state, else 0
 * (baselines.py:52-66).  Masks: bit v set <=> count v in the set (v <= 8). */
typedef struct tvs_life_rule {
  int32_t dim;
  int32_t ntaps; /* 1..26 */
  int32_t offsets[26][3];
  int32_t birth_mask;
  int32_t survive_mask;
  int32_t boundary; /* constant value of every non-interior cell */
  int32_t pad_;
} tvs_life_rule;
/* one call: host int32 Grid in (reference layout), host Grid out */
int tvs_life_run(const tvs_life_rule* r, const tvs_layout* lay, const int32_t* in, int32_t* out, int64_t steps,
                 const tvs_exec* ex);
/* caller-owned device blocks (geometry as for fp64, 4-byte cells); ping-pong
 * like tvs_jacobi_device */
int tvs_life_device(const tvs_life_rule* r, const tvs_geometry* g, int32_t* src, int32_t* dst, int64_t steps,
                    const tvs_exec* ex, void* stream, int32_t* result_in_dst);
int tvs_fill_halo_i32(const tvs_geometry* g, int32_t* dev, int32_t value, void* stream);
int tvs_upload_i32(const tvs_geometry* g, int32_t* dev, const tvs_layout* lay, const int32_t* host, void* stream);
int tvs_download_i32(const tvs_geometry* g, const int32_t* dev, const tvs_layout* lay, int32_t* host, void* stream);
/* LCS length of int32 sequences a (na) and b (nb) (kernels/lcs.py:32). */
int tvs_lcs(const int32_t* a, int64_t na, const int32_t* b, int64_t nb, const tvs_exec* ex, int64_t* length);
/* device-resident form: a, b device pointers, *result written on `stream` */
int tvs_lcs_device(const int32_t* a, int64_t na, const int32_t* b, int64_t nb, int32_t* result, void* stream);

/* ---- tile-schedule executor ----------------------
 * One tile of a schedule (tiling.py Tile): time levels [t0, t1); axis d at
 * time t covers [lo[d] + slope_lo[d]*(t-t0), hi[d] + slope_hi[d]*(t-t0))
 * clipped to the grid.  Tiles are listed wave by wave; wave w is
 * tiles[wave_start[w] .. wave_start[w+1]).  Every wave is one launch (one
 * CTA per tile) over a full time history in device memory; Gauss-Seidel
 * uses the lexicographic in-place semantics. */
typedef struct tvs_tile {
  int32_t t0, t1;
  int32_t lo[3], hi[3];
  int32_t slope_lo[3], slope_hi[3];
} tvs_tile;
int tvs_tiled_run(const tvs_stencil* st, const tvs_layout* lay, const double* in, double* out, int64_t steps,
                  const tvs_tile* tiles, const int64_t* wave_start, int64_t nwaves, const tvs_exec* ex);
int tvs_tiled_life(const tvs_life_rule* r, const tvs_layout* lay, const int32_t* in, int32_t* out, int64_t steps,
                   const tvs_tile* tiles, const int64_t* wave_start, int64_t nwaves, const tvs_exec* ex);
/* LCS over rectangle tiles: time = A index (t -> row t+1), axis 0 = B index */
int tvs_lcs_tiled(const int32_t* a, int64_t na, const int32_t* b, int64_t nb, const tvs_tile* tiles,
                  const int64_t* wave_start, int64_t nwaves, const tvs_exec* ex, int64_t* length);

/* ---- misc -------------------------------------------------------------- */
/* Free the calling thread's cached tvs_run / tvs_lcs device buffers, streams,
 * events and captured graphs (they are otherwise kept per thread between
 * calls).  Thread-pool workers (tiling.py:363-367) call it before exiting. */
int tvs_release_thread_cache(void);
const char* tvs_last_error(void);
int tvs_device_count(int32_t* n);
int tvs_host_register(void* ptr, size_t bytes);   /* pin a host buffer */
int tvs_host_unregister(void* ptr);
/* page-locked host allocation (cudaHostAlloc) for Grid storage: both copy
   directions at once run at ~97 GB/s from it vs ~83 GB/s from registered
   pageable memory (tools/pinned_probe.py).  Replaces the numpy allocation in
   the reference Grid constructor (tvstencil/grid.py:24-50) when the caller
   asks for pinned storage. */
int tvs_host_alloc(size_t bytes, void** ptr);
int tvs_host_free(void* ptr);
/* 64-bit FNV-1a continuing from `state` (grid.py:127-133). Host only. */
uint64_t tvs_fnv1a64(const void* data, size_t n, uint64_t state);
/* kernels launched by this thread since the last call (resets the counter) */
int64_t tvs_launch_counter(void);
const char* tvs_version(void);

#ifdef __cplusplus
}
#endif
#endif /* TVSTENCIL_H */
