/*
 * nglod_b200 -- C ABI of the B200 (sm_100a) NGLOD render hot path.
 *
 * The reference (arxiv/paper_2101_10994, package `octfield`) is pure Python
 * and exposes no FFI: its boundary is the Python module API
 * (octfield/__init__.py:11-164). These entry points are what a ctypes / cffi
 * binding of that API needs; each names the reference function it replaces.
 * The Python host package `paper_2101_10994_b200` binds them with ctypes
 * (INTEGRATION.md shows the binding a maintainer would add to octfield).
 *
 * Conventions
 *  - Plain C types only. Every pointer argument is DEVICE memory owned by
 *    the caller (PyTorch allocates it); nothing here frees caller memory.
 *  - `stream` is a cudaStream_t passed as void*. Calls are asynchronous on
 *    that stream unless documented otherwise.
 *  - Every function returns an int status (NG_OK = 0). NG_ERR_* map 1:1 to
 *    the reference exception classes (octfield/errors.py:4-29); the message
 *    of the last failure on the calling thread is ng_last_error().
 *  - Variable-length outputs use two-phase sizing: counts are written to
 *    device memory; when a count exceeds the capacity the caller passed,
 *    the data is not written and the caller retries with larger buffers.
 */
#ifndef NGLOD_B200_H
#define NGLOD_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NG_OK 0
#define NG_ERR_STRUCTURAL 1  /* octfield.errors.StructuralError */
#define NG_ERR_CONFIG 2      /* octfield.errors.ConfigError */
#define NG_ERR_CAPACITY 3    /* internal: grow buffers and retry */
#define NG_ERR_CUDA 4        /* CUDA runtime failure */
#define NG_ERR_OCTFIELD 5    /* octfield.errors.OctfieldError (e.g. non-finite decoder input) */

#define NG_MAX_TLEVELS 16    /* virtual + stored traversal levels */
#define NG_FEAT_PAD 32       /* feature rows are padded to 32 fp32 channels (128 B) */
#define NG_W1_STRIDE 36      /* packed decoder row: 3 x-weights, 32 feature weights, b1 */
#ifndef NG_MAX_BATCH
#define NG_MAX_BATCH 16      /* cameras per ng_render_batch launch (_lib.MAX_BATCH mirrors it) */
#endif

/* Device-resident sparse voxel octree (octree.py:100-131).
 * Traversal level t = level + n_virtual; levels -n_virtual..-1 are the
 * virtual coarse grids above the stored root (octree.py:1-8, 208-212). */
typedef struct ng_octree {
  int32_t r0;
  int32_t max_level;
  int32_t n_virtual;            /* log2(r0) */
  int32_t n_tlevels;            /* n_virtual + max_level + 1 */
  int64_t count[NG_MAX_TLEVELS];              /* voxels per traversal level */
  const uint64_t* codes[NG_MAX_TLEVELS];      /* strictly ascending Morton codes */
  const int32_t* child_start[NG_MAX_TLEVELS]; /* index of first child in level t+1 */
  const uint8_t* child_mask[NG_MAX_TLEVELS];  /* occupied-octant bits (bit = code & 7) */
  const uint64_t* bitmap[NG_MAX_TLEVELS];     /* occupancy bit per Morton code (res^3 bits) */
  const uint32_t* rank[NG_MAX_TLEVELS];       /* exclusive popcount per 64-bit bitmap word */
  const int32_t* corners[NG_MAX_TLEVELS];     /* feature levels: (count, 8) global corner ids */
  double region_lo[3];          /* occupied finest-level AABB (octree.py:204-206) */
  double region_hi[3];
  double half_diag_finest;      /* 0.5*sqrt(3)*edge(max_level) (octree.py:123-124) */
} ng_octree;

/* Neural field parameters (field.py:30-48, 242-269), packed for the device.
 *  Z:        (corner_count, 32) fp32, channels >= m zero.
 *  decoders: n_decoders blocks of dec_stride floats; block L-1 holds
 *            W1b[h][36] (x weights, feature weights padded to 32, b1),
 *            W2[h], b2, zero padding. */
typedef struct ng_field {
  const float* Z;
  const float* decoders;
  int32_t m;
  int32_t h;
  int32_t n_decoders;
  int32_t dec_stride;
  int64_t corner_count;
  /* Optional presummed feature tables for the sphere tracer (ng_field_presum):
   * S_L on the level-`presum_level` corner ids for each L in presum_mask
   * (ascending), (n, presum_corners, 32) fp32. Used by the march / normals
   * when their gather level and output levels match; NULL disables. */
  const float* presum;
  int64_t presum_offset;   /* first corner id of the level */
  int64_t presum_corners;  /* corners of the level */
  int32_t presum_level;
  int32_t presum_mask;
} ng_field;

/* EvalCounter (field.py:79-90) plus a non-finite-input tally; device int64. */
typedef struct ng_counters {
  int64_t decoder_evals;
  int64_t evals_missing_level;
  int64_t empty_fallbacks;
  int64_t nonfinite_inputs;
} ng_counters;

/* One batched SDF query. Modes:
 *  - predict / forward (field.py:194-218, 337-357): out_levels selects the
 *    decoder levels L to output (bit L-1), one fp64 column per set bit in
 *    ascending L; each column equals predict(x, L).
 *  - blend (field.py:226-239): blend_base >= 1 and blend_alpha in (0,1)
 *    outputs one column (1-a)*predict(base) + a*predict(base+1).
 *  - query_field (render.py:155-171): inside_level >= 0 answers points that
 *    are not inside that level's voxels with empty_space_value. */
typedef struct ng_query_args {
  int32_t out_levels;
  int32_t inside_level;
  int32_t blend_base;
  int32_t pad;
  double blend_alpha;
} ng_query_args;

/* Ray record (traversal.py:40-56): origin, unit direction, 1/direction,
 * flags bits 0-2 = (d<0) per axis (traversal.py:147-154), bits 3-5 = (d==0). */
typedef struct ng_ray {
  double o[3];
  double d[3];
  double inv[3];
  int32_t flags;
  int32_t pad;
} ng_ray;

/* (ray, voxel) pair at one traversal level (traversal.py:59-70). */
typedef struct ng_pair {
  int32_t ray;
  int32_t voxel;
} ng_pair;

/* Final-level hit with its entry/exit distances (traversal.py:233-246). */
typedef struct ng_hit_pair {
  int32_t ray;
  int32_t voxel;
  double t_enter;
  double t_exit;
} ng_hit_pair;

/* Pinhole camera (render.py:43-88); basis precomputed on the host in fp64.
 * Image tiling for multi-GPU frames: the image is cut into bands of
 * band_rows rows; this camera generates the rays of bands b with
 * b % band_stride == band_offset, in order (band_stride = 1: whole frame). */
typedef struct ng_camera {
  double position[3];
  double fwd[3];
  double right[3];
  double up[3];
  double tan_half;
  double aspect;
  int32_t width;
  int32_t height;
  int32_t band_rows;
  int32_t band_stride;
  int32_t band_offset;
  int32_t local_rows;   /* rows this camera generates */
} ng_camera;

/* RenderConfig (render.py:91-114), resolved on the host. */
typedef struct ng_render_cfg {
  double delta;
  double far_plane;
  double skip_eps;
  double osc_tol;         /* osc_factor * delta */
  double lod;             /* resolved detail level, >= 1 */
  double normal_eps;
  double light[3];        /* normalised */
  double albedo[3];
  double ambient;
  double background[3];
  int32_t max_iters;
  int32_t trace_level;    /* min(ceil(lod), max_level) */
  /* Secondary shadow rays (BASELINE.json configs[4]; not in the reference):
   * from p + shadow_offset * n toward the light, traced with the same rules;
   * a hit means the pixel is shaded with the ambient term only. */
  double shadow_offset;
  int32_t shadows;
  int32_t pad;
} ng_render_cfg;

/* Per-pixel frame outputs (render.py:117-128), device arrays of n pixels. */
typedef struct ng_frame {
  uint8_t* hit;           /* (n,) */
  double* t;              /* (n,) nan on miss */
  double* normal;         /* (n, 3), zero where invalid */
  uint8_t* normal_ok;     /* (n,) */
  int32_t* iterations;    /* (n,) */
  int32_t* evals;         /* (n,) */
  uint8_t* color;         /* (n, 3) */
} ng_frame;

/* Scratch for traversal and tracing; sized by ng_render_workspace_bytes. */
typedef struct ng_workspace {
  void* base;
  size_t bytes;
  int64_t pair_capacity;  /* per ping-pong pair buffer */
  int64_t hit_capacity;   /* final hit-pair list */
  void* ev_trace_done;    /* optional cudaEvent_t recorded between march and normals */
  void* ev_march_begin;   /* optional cudaEvent_t recorded just before the march kernel */
} ng_workspace;

/* Device-side frame statistics (FrameReport, render.py:131-137). */
typedef struct ng_frame_stats {
  int64_t pairs[NG_MAX_TLEVELS + 1]; /* list length entering each level; [target+1] = hits */
  int64_t visible;
  int64_t active_rays;
  ng_counters counters;
  int64_t overflow;              /* nonzero: a pair list exceeded its capacity */
  int64_t shadow_pairs[NG_MAX_TLEVELS + 1]; /* shadow-ray traversal (when cfg.shadows) */
  int64_t shadowed;              /* hit pixels whose shadow ray hit the surface */
  int64_t pair_need;             /* after an overflow: pair capacity a rerun needs (tile traversal arena) */
} ng_frame_stats;

/* ---- library ----------------------------------------------------------- */
int ng_abi_version(void);
const char* ng_last_error(void);
int ng_sm_count(int device);

/* ---- Morton / binning / locate (octree.py:35-85, 134-143, 259-282) ----- */
int ng_morton_encode(const int64_t* ijk, int64_t n, uint64_t* codes, void* stream);
int ng_morton_decode(const uint64_t* codes, int64_t n, int64_t* ijk, void* stream);
int ng_locate(const ng_octree* tree, const double* pts, int64_t n, int32_t level,
              int64_t* out_index, void* stream);
/* ray_aabb_batch (octree.py:311-333): rows matched; t_enter/t_exit fp64, hit u8. */
int ng_ray_aabb(const double* o, const double* d, const double* lo, const double* hi,
                int64_t n, double* t_enter, double* t_exit, uint8_t* hit, void* stream);

/* ---- octree build (octree.py:146-256) ----------------------------------- */
/* Set the finest-level bit of every sample's cell (octree.py:170-175). */
int ng_build_mark_samples(const double* pts, int64_t n, int32_t res, uint64_t* bitmap,
                          void* stream);
/* Corner test (octree.py:225-246) from an fp32 |d| lattice of (res+1)^3 in
 * (i,j,k) C order: set cells whose min corner |d| <= tol (fp64 compare). */
int ng_build_mark_lattice(const float* absd, int32_t res, double tol, uint64_t* bitmap,
                          void* stream);
/* |d| of a built-in analytic SDF on the corner lattice, as fp32.
 * kind 1 sphere (r), 2 torus (R, r), 3 closed polyline tube (params =
 * [tube, x0,y0,z0, x1,...], nverts = (n_params-1)/3, params in device memory). */
int ng_sdf_lattice(int32_t kind, const double* params, int32_t n_params, int32_t res,
                   float* absd, void* stream);
int ng_sdf_eval(int32_t kind, const double* params, int32_t n_params, const double* pts,
                int64_t n, double* out, void* stream);
/* Parent closure: parent bit p = OR of child bits 8p..8p+7 (octree.py:183-187). */
int ng_bitmap_parent(const uint64_t* child_bitmap, int64_t child_words, uint64_t* parent_bitmap,
                     int64_t parent_words, void* stream);
/* Exclusive popcount prefix per word; total written to *d_total (device). */
int ng_bitmap_rank(const uint64_t* bitmap, int64_t n_words, uint32_t* rank, int64_t* d_total,
                   void* scratch, size_t scratch_bytes, void* stream);
/* Sorted set-bit positions -> codes (np.unique order). */
int ng_bitmap_extract(const uint64_t* bitmap, const uint32_t* rank, int64_t n_words,
                      uint64_t* codes, void* stream);
/* parents (octree.py:197) from the parent level's bitmap/rank. */
int ng_level_parents(const uint64_t* codes, int64_t n, const uint64_t* parent_bitmap,
                     const uint32_t* parent_rank, int32_t* parents, void* stream);
/* child_start / child_mask for traversal (children_ranges, octree.py:303-308). */
int ng_level_children(const uint64_t* codes, int64_t n, const uint64_t* child_bitmap,
                      const uint32_t* child_rank, int32_t* child_start, uint8_t* child_mask,
                      void* stream);
/* Corner keys of every voxel into a (2*res)^3-bit corner bitmap (octree.py:249-253). */
int ng_corner_mark(const uint64_t* codes, int64_t n, uint64_t* corner_bitmap, void* stream);
/* Corner table: offset + rank of each corner key (octree.py:254-256). */
int ng_corner_table(const uint64_t* codes, int64_t n, const uint64_t* corner_bitmap,
                    const uint32_t* corner_rank, int32_t offset, int32_t* corners, void* stream);
/* Min / max cell coordinate of a level (for the region AABB, octree.py:204-206). */
int ng_cell_extent(const uint64_t* codes, int64_t n, int32_t* d_minmax6, void* stream);

/* ---- scans (traversal.py:113-144) --------------------------------------- */
size_t ng_scan_scratch_bytes(int64_t n);
int ng_exclusive_sum_i64(const int64_t* in, int64_t n, int64_t* out, void* scratch,
                         size_t scratch_bytes, void* stream);

/* ---- field (field.py:104-239, 337-357; render.py:155-171) -------------- */
int ng_query(const ng_octree* tree, const ng_field* fld, const ng_query_args* args,
             const double* pts, int64_t n, double* out, ng_counters* d_counters, void* stream);
/* sum_features / trilinear: z = sum of levels [level_lo, level_hi] as fp64
 * (n, m) and per-level presence mask (n, level_hi-level_lo+1). */
int ng_interp(const ng_octree* tree, const ng_field* fld, const double* pts, int64_t n,
              int32_t level_lo, int32_t level_hi, double* z, uint8_t* mask, void* stream);
/* empty_space_value (field.py:185-191). */
int ng_empty_value(const ng_octree* tree, const double* pts, int64_t n, double* out,
                   void* stream);

/* ---- traversal (traversal.py:95-255) ------------------------------------ */
/* Build ray records from origins/directions (n,3) fp64. */
int ng_rays_from_arrays(const double* o, const double* d, int64_t n, ng_ray* rays,
                        void* stream);
/* One BFS pass at traversal level t: decide + exclusive scan + subdivide
 * (or, when final != 0, decide + compactify + entry/exit distances).
 * in == NULL means the implicit root list (i, 0) of d_count_in rays.
 * Counts live in device memory; writes past the capacity are dropped and
 * the full count is still reported. */
size_t ng_level_scratch_bytes(int64_t max_pairs);
int ng_traverse_level(const ng_octree* tree, const ng_ray* rays, int32_t t, int32_t final,
                      const ng_pair* in, const int64_t* d_count_in, int64_t in_capacity,
                      ng_pair* out_pairs, ng_hit_pair* out_hits, int64_t* d_count_out,
                      int64_t out_capacity, void* scratch, size_t scratch_bytes, void* stream);
/* ray_segments (traversal.py:250-255) over a final hit list (device count). */
int ng_segments(const ng_hit_pair* hits, const int64_t* d_count, int64_t capacity,
                int64_t n_rays, int64_t* seg_start, int64_t* seg_end, void* stream);

/* ---- the field API in float64 (field.py:104-239, 337-357; render.py:155-171)
 * Reference semantics computed in fp64 from the caller's parameters: Z is
 * (C, m) fp64 row-major; decoders are fp64 blocks of dec_stride doubles in
 * the training layout W1b[h][36] (x weights, m feature weights, b1 in
 * column 35), W2[h], b2. Serves predict / blend / forward / query_field /
 * trilinear / sum_features / decode (the hot paths use ng_query and
 * ng_render_frame). */
int ng_interp64(const ng_octree* tree, const double* Z, int32_t m, const double* pts, int64_t n,
                int32_t level_lo, int32_t level_hi, double* z, uint8_t* mask, void* stream);
int ng_decode64(const double* decoder, int32_t h, int32_t m, const double* x, const double* z, int64_t n,
                double* out, int64_t* d_nonfinite, void* stream);
int ng_query64(const ng_octree* tree, const double* Z, int32_t m, const double* decoders, int32_t h,
               int32_t n_decoders, int32_t dec_stride, const ng_query_args* args, const double* pts, int64_t n,
               double* out, ng_counters* d_counters, void* stream);

/* ---- rendering (render.py:43-448) --------------------------------------- */
int ng_camera_rays(const ng_camera* cam, ng_ray* rays, void* stream);
size_t ng_render_workspace_bytes(int64_t n_rays, int64_t pair_capacity, int64_t hit_capacity);
/* Byte offsets into a frame workspace of what the last frame's traversal
 * left there (render path, traversal.py:207-255): out[0] the final hit list
 * (ng_hit_pair, tile order; .ray holds the voxel's packed cell
 * x | y << 10 | z << 20 on the tile path, the ray id otherwise), out[1] /
 * out[2] the per-ray segments [start, end) into it (int64), out[3] the total
 * size, out[4] the tile traversal's control words (u64 at +128: the
 * continuation records pushed << 32 | finished). n_out <= 5 entries are
 * written. Lets callers and tests read the render path's per-ray voxel
 * lists back without re-running a traversal. */
int ng_render_workspace_offsets(int64_t n_rays, int64_t pair_capacity, int64_t hit_capacity,
                                int64_t* out, int32_t n_out);
/* sphere_trace (render.py:174-274) over an existing final list. */
int ng_sphere_trace(const ng_octree* tree, const ng_field* fld, const ng_render_cfg* cfg,
                    const ng_ray* rays, int64_t n_rays, const ng_hit_pair* hits,
                    const int64_t* d_hit_count, const int64_t* seg_start,
                    const int64_t* seg_end, uint8_t* hit, double* t_hit, int32_t* iters,
                    int32_t* evals, ng_counters* d_counters, void* stream);
/* normals (render.py:277-300) at hit points p (k,3) fp64 -> normal fp64, ok u8. */
int ng_normals(const ng_octree* tree, const ng_field* fld, const ng_render_cfg* cfg,
               const double* pts, int64_t k, double* normal, uint8_t* ok,
               ng_counters* d_counters, void* stream);
/* shade (render.py:303-314). */
int ng_shade(const uint8_t* hit, const double* normal, int64_t n, const ng_render_cfg* cfg,
             uint8_t* color, void* stream);
/* Whole frame: rays -> traversal -> march -> normals -> shade, with no host
 * synchronisation (capturable in a CUDA graph). Statistics are written to
 * *d_stats (device); stats.overflow != 0 means retry with more capacity. */
int ng_render_frame(const ng_octree* tree, const ng_field* fld, const ng_render_cfg* cfg,
                    const ng_camera* cam, const ng_frame* frame, const ng_workspace* ws,
                    ng_frame_stats* d_stats, void* stream);
/* A batch of frames in one launch sequence (render.py:342-448 per camera,
 * for a camera sequence): cams[0..n_cams) share width, height and band
 * layout (NG_ERR_CONFIG otherwise), 1 <= n_cams <= NG_MAX_BATCH. Frame f's
 * pixels are pixels [f n, (f + 1) n) of every `frame` buffer and of the
 * workspace's per-ray arrays (n = width * local_rows; size the workspace for
 * n_cams * n rays). Each frame's outputs equal ng_render_frame's for its
 * camera; the statistics cover the batch. One traversal and one march cover
 * every frame, so one frame's longest rays overlap the others' work. */
int ng_render_batch(const ng_octree* tree, const ng_field* fld, const ng_render_cfg* cfg,
                    const ng_camera* cams, int32_t n_cams, const ng_frame* frame,
                    const ng_workspace* ws, ng_frame_stats* d_stats, void* stream);
/* CUDA graphs of launch sequences (render.py's frame graphs): capture on a
 * non-default stream (thread-local mode), instantiate, replay on any stream.
 * exec handles are opaque; ng_graph_destroy releases one. */
int ng_graph_capture_begin(void* stream);
int ng_graph_capture_end(void* stream, void** exec_out);
int ng_graph_launch(void* exec, void* stream);
int ng_graph_destroy(void* exec);
/* Same, for arbitrary rays (metrics.trace_field_rays, metrics.py:135-142). */
int ng_render_rays(const ng_octree* tree, const ng_field* fld, const ng_render_cfg* cfg,
                   const ng_ray* rays, int64_t n_rays, const ng_frame* frame,
                   const ng_workspace* ws, ng_frame_stats* d_stats, int32_t do_normals,
                   void* stream);
/* Standalone decoder (decode, field.py:172-182) on given inputs: x (n,3),
 * z (n,m) fp64 -> out (n,) fp64; decoder is one packed block. Non-finite
 * inputs are counted in *d_nonfinite (device int64). */
int ng_decode(const float* decoder, int32_t h, int32_t m, const double* x, const double* z, int64_t n,
              double* out, int64_t* d_nonfinite, void* stream);
/* decide (traversal.py:95-110) for an explicit pair list at traversal level t. */
int ng_decide(const ng_octree* tree, const ng_ray* rays, int32_t t, int32_t final, const ng_pair* pairs,
              int64_t n, int64_t* decisions, void* stream);
/* subdivide (traversal.py:165-191) from decisions D and their exclusive sum S. */
int ng_subdivide(const ng_octree* tree, const ng_ray* rays, int32_t t, const ng_pair* pairs, int64_t n,
                 const int64_t* D, const int64_t* S, ng_pair* out, void* stream);
/* compactify (traversal.py:194-204). */
int ng_compactify(const ng_pair* pairs, int64_t n, const int64_t* D, const int64_t* S, ng_pair* out,
                  void* stream);
/* Debug (NG_MARCH_PROFILE=1): per tile group of the last march launches
 * {steps, busy lanes, first ns, last ns, acquire ns, eval ns, 0, 0}; copies and resets. */
int ng_march_profile(unsigned long long* host_out, int max_groups);
/* Hit positions o + t*d for hit rays (FrameBuffer.points, render.py:395-396). */
int ng_hit_points(const ng_ray* rays, const uint8_t* hit, const double* t, int64_t n,
                  double* points, void* stream);

/* Presummed feature tables: S_L(c) = sum_{l <= L} psi_l(c) at every level-`level`
 * corner c, for each L in out_mask (ascending), fp32 (n_out, n_corners, 32).
 * Exact reassociation of sum_features (field.py:154-169) for points inside a
 * level-`level` voxel (see presum.cu). owner_scratch: n_corners int32. */
int ng_field_presum(const ng_octree* tree, const float* Z, int32_t level, int32_t out_mask, int64_t offset,
                    int64_t n_corners, float* S, int32_t* owner_scratch, void* stream);

/* ---- evaluation (metrics.py) ------------------------ */
/* trace_oracle_rays (metrics.py:145-178) for a built-in SDF (kinds as in
 * ng_sdf_lattice): hit u8, t_hit fp64 (nan on miss). */
int ng_trace_sdf(int32_t kind, const double* params, int32_t n_params, const double* origins, const double* dirs,
                 int64_t n, double delta, double far_plane, int32_t max_iters, uint8_t* hit, double* t_hit,
                 void* stream);
/* Nearest occupied voxel of `level` for each point (first minimum of the
 * squared box distance, metrics.py:236-250): the clamped anchor (n,3) and the
 * separation (n,). */
int ng_nearest_voxel(const ng_octree* tree, int32_t level, const double* pts, int64_t n, double* anchor, double* gap,
                     void* stream);
/* sample_surface_sdf's tracer (sampling.py:109-149) for a built-in SDF: the
 * surface point of each ray, NaN where the ray found none. */
int ng_surface_trace(int32_t kind, const double* params, int32_t n_params, const double* origins,
                     const double* dirs, int64_t n, double tol, double t_max, int32_t max_iters,
                     int32_t bisect_iters, double* points, void* stream);
/* Distance from each query to its nearest point (PointGrid.nearest_dist, metrics.py:64-112). */
int ng_nn_dist(const double* queries, int64_t nq, const double* points, int64_t np_, double* out, void* stream);

/* ---- training (field.py:286-409, trainer.py:87-296) ------- */
/* fp64 master parameters and Adam moments (trainer.py:62-84, 176-190), all
 * device memory owned by the caller. Z rows are padded to 32 channels; each
 * decoder block holds W1b[h][36] (x weights, feature weights, b1 in column
 * 35), W2[h], b2, zero padding to dec_stride doubles. */
typedef struct ng_train_params {
  double* Z;
  double* Zm;
  double* Zv;
  int32_t* Zlast;           /* per row: last Adam step applied (lazy zero-gradient steps) */
  double* dec;
  double* decm;
  double* decv;
  int32_t m;
  int32_t h;
  int32_t n_decoders;
  int32_t dec_stride;
  int64_t corner_count;
} ng_train_params;

/* One batch (loss_batch + backward + adam_step, trainer.py:106-144, 87-103). */
typedef struct ng_train_step {
  int32_t active_mask;      /* loss levels, bit L-1 (trainer.py:119-125) */
  int32_t update_decoders;  /* 0 for the frozen_decoder schedule (trainer.py:197) */
  int32_t mode;             /* 0: Adam step; 1: gradients only (accumulated); 2: forward cache */
  int32_t pad;
  double denom;             /* loss denominator (trainer.py:127) */
  double lr;
  int64_t step;             /* Adam step of this batch, 1-based (trainer.py:91) */
  const double* adam_c;     /* device: (1 - beta1^t, 1 - beta2^t) of step t at [2(t-1)] (trainer.py:92-93) */
  int64_t batch_index;      /* reported through status on divergence */
} ng_train_step;

/* The workspace must be zero-filled once before its first use. */
size_t ng_train_workspace_bytes(const ng_octree* tree, int64_t batch_capacity, int32_t h, int32_t n_decoders,
                                int64_t corner_count, int32_t dec_stride);
/* One batch. upstream != NULL selects backward(cache, upstream) semantics
 * (field.py:360-394) for the single level in active_mask. Mode 0 adds the
 * per-level residual sums to level_sums[L-1] and runs Adam unless *status
 * != 0; a non-finite loss or gradient sets *status = 1 + batch_index and
 * stops all later updates (TrainingDiverged). Mode 1 writes level_sums,
 * accumulates grad_Z (corner_count x 32) and grad_dec (n_decoders x
 * dec_stride) and sets dec_touched[L-1] = 1 for decoders that received a
 * gradient. psi_out (optional, n x max_active_level x 32) receives the
 * per-level interpolated features. */
int ng_train_batch(const ng_octree* tree, const ng_train_params* P, const ng_train_step* st, const double* pts,
                   const double* dist, const double* upstream, int64_t n, int64_t batch_capacity, void* ws,
                   size_t ws_bytes, double* level_sums, double* grad_Z, double* grad_dec, int32_t* dec_touched,
                   double* psi_out, int64_t* status, void* stream);
/* All mini-batches of one epoch (trainer.py:223-241) on already-permuted
 * device points; Adam steps step0+1, step0+2, ... (adam_c must cover them).
 * Rows are flushed to the current step every flush_every batches and at the
 * end, so P is fully up to date when the stream reaches the end. */
int ng_train_epoch(const ng_octree* tree, const ng_train_params* P, const double* pts, const double* dist,
                   int64_t n, int64_t batch_size, int32_t active_mask, int32_t update_decoders, double lr,
                   int64_t step0, const double* adam_c, int32_t flush_every, void* ws, size_t ws_bytes,
                   double* level_sums, int64_t* status, void* stream);
/* Apply the zero-gradient Adam steps every row has missed, up to `step`. */
int ng_train_flush(const ng_train_params* P, int64_t step, const double* adam_c, double lr, void* stream);
/* ForwardCache (field.py:321-357) of forward(x, level) with batch capacity
 * n: per-level corner ids (n, level, 8; -1 where absent) and trilinear
 * weights, per-level features psi (n, level, 32), pre-activations (n, h)
 * and decoder inputs [x, z, 1] (n, 36); rows that are not decoded are 0. */
int ng_train_export(const ng_octree* tree, const ng_train_params* P, int32_t level, const double* pts, int64_t n,
                    void* ws, size_t ws_bytes, int32_t* ids, double* weights, double* psi, double* pre, double* inp,
                    void* stream);
/* Debug (NG_TRAIN_EVENTS=1): mean device ms per batch of each training kernel
 * (locate, rowprep, gather, dec, reduce, update) since the last call; resets. */
int ng_train_profile(double* host_out6);
/* adam_step (trainer.py:87-103) on one fp64 array; *d_bad = 1 (and no
 * update) when the gradient has a non-finite entry. */
int ng_adam_step(double* param, double* m, double* v, const double* grad, int64_t n, double lr, double c1,
                 double c2, int64_t* d_bad, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* NGLOD_B200_H */
