/*
 * ss_abi.h -- C ABI of the B200-native 3DSS surface-splatting hot path.
 *
 * libss_b200.so (built from paper_2605_05876_b200/csrc/) exports these entry
 * points.  They are the seams of the reference package's Python hot path
 * (surfsplat 0.1.0, a CPU numpy/numba package with no native ABI of its own):
 * each function replaces one reference routine, cited per entry below, and the
 * Python host mirror (paper_2605_05876_b200/) binds them with ctypes the way a
 * maintainer would bind them from the reference.
 *
 * Conventions
 *  - Every pointer is a DEVICE pointer owned by the caller (the torch
 *    allocator in the host mirror); the library never allocates.  Scratch
 *    buffers are sized by the caller from the formulas documented per entry.
 *    Exceptions, passed by value from the HOST: the struct arguments
 *    (SsCamera/SsCloud/SsEnv/... themselves, whose members are device
 *    pointers), `background` (3 floats) and `origin3` (3 floats).
 *  - `stream` is a cudaStream_t passed as void*.  All work is stream-ordered,
 *    asynchronous and CUDA-graph capturable (no host synchronisation inside).
 *  - Return value: SS_OK, SS_ERR_INVALID (bad argument, checked on the host
 *    before any launch), or SS_ERR_CUDA (launch error; see ss_last_error()).
 *  - Surfel parameters are float32 struct-of-arrays (surfels.py:80-105).
 *    Per-view records are indexed by SOURCE surfel index (culled rows carry
 *    rect = 0 and emit no pairs); the reference compacts kept rows in
 *    ascending source order (preprocess.py:296), which is order-isomorphic,
 *    so sort orders and tile lists are identical after the host re-indexes.
 */
#ifndef SS_ABI_H
#define SS_ABI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { SS_OK = 0, SS_ERR_INVALID = 1, SS_ERR_CUDA = 2 };

#define SS_REC_FLOATS 24  /* 96-byte record, see SsRecord in csrc/ss_common.cuh */
#define SS_ACC_FLOATS 20  /* per-record backward accumulator: 17 grads + ss + touch + layout flag */
/* slot 19 of an accumulator row: 0 = slots 0..8 hold dL/dt1, dt2, dt4;
 * SS_ACC_MOMENTS = they hold sum gp, sum (x - cx) gp, sum (y - cy) gp of the
 * ray-plane gradient, (cx, cy) = (t1.z / t4.z, t2.z / t4.z) the projected
 * centre (record-parallel backward; ss_chain_backward converts) */
#define SS_ACC_MOMENTS 1.0f
/* slot 19 = SS_ACC_F64: the row's channels live in float64 in the caller's
 * rec_acc64 buffer (ss_train_backward_records), row index = the int bits of
 * slot 0, SS_ACC64_WIDTH doubles per row in channel order dt1 dt2 dt4,
 * dSigma^-1, dn_f, dcolour, screen |g| sum, dview_z (slot 17 still holds
 * the float screen sum, slot 18 the touch count) */
#define SS_ACC_F64 2.0f
#define SS_ACC64_WIDTH 18
#define SS_KMAX_CAP 16    /* largest k_max the kernels accept (= reference default K_MAX) */

typedef struct SsCamera {
    double view[16];   /* row-major world->view (camera.py:28-48) */
    double proj[16];   /* row-major view->clip, GL style (camera.py:17-25) */
    int width, height;
} SsCamera;

typedef struct SsCloud {
    const float *centers;       /* (n,3) */
    const float *quats;         /* (n,4) wxyz */
    const float *log_scales;    /* (n,2) */
    const float *albedo_raw;    /* (n,3) pre-sigmoid */
    const float *metallic_raw;  /* (n,)  */
    const float *roughness_raw; /* (n,)  */
    int n;
} SsCloud;

/* Prefiltered environment (shading.py:334-379) as consumed by shading. */
typedef struct SsEnv {
    const float *diffuse;   /* (He,We,3) */
    const float *specular;  /* (L,He,We,3) */
    const float *lut;       /* (R,R,2) BRDF LUT, row = roughness (shading.py:118-156) */
    int he, we, levels, lut_res;
    /* nullable: the same maps padded to 4 floats per texel (16-byte texel
     * loads in the shading kernels) */
    const float *diffuse4;  /* (He,We,4) */
    const float *specular4; /* (L,He,We,4) */
    /* nullable: the float64 maps (ss_env_refresh), read by the float64 shading */
    const double *diffuse64;  /* (He,We,3) */
    const double *specular64; /* (L,He,We,3) */
} SsEnv;

typedef struct SsPreprocessOpts {
    float r_cut;       /* preprocess.py:19 */
    float mip_sigma;   /* preprocess.py:34 */
    int mip_enabled;
    int tile;          /* rasterizer.py:22 */
} SsPreprocessOpts;

/* Colour sources of render() (rasterizer.py:341-350). */
enum { SS_COLOR_EXPLICIT = 0, SS_COLOR_IBL = 1, SS_COLOR_ALBEDO = 2, SS_COLOR_IBL_F32 = 3 };

/* Optional per-surfel outputs of preprocess (ProjectedSurfels fields,
 * preprocess.py:195-228), all (n, ...) and nullable. */
typedef struct SsProjAux {
    float *c_cam, *tu_cam, *tv_cam;   /* (n,3) */
    float *eps_z;                     /* (n,)  */
    float *center_ndc;                /* (n,2) */
    float *jac;                       /* (n,2,2) */
    uint8_t *jac_ok;                  /* (n,)  */
    float *colors;                    /* (n,3) the per-surfel colours used */
    int32_t *cells;                   /* (n,15) shading branch signature (shading.py:490-497) */
    /* (n,4) uint32, the same branch state packed for ss_chain_backward:
     * diffuse cell i0 | j0 << 16, specular cell, LUT cell, roughness level
     * | flags << 8 (bit 0 diffuse dv_ok, 1 specular dv_ok, 2 LUT du_ok,
     * 3 LUT dv_ok, 4 n.w_o > 0, 5 n.w_o < 1) -- from the float64 forward */
    uint32_t *cells_packed;
} SsProjAux;

/* ---- preprocess + shade + tile count --------------------------------------
 * Replaces preprocess() (preprocess.py:231-309), shade_surfels()
 * (shading.py:447-503) and the count half of bin_and_sort()
 * (rasterizer.py:92-106).  Writes one 96-byte record per surfel, the cull code
 * (0-4, preprocess.py:23-27), the per-record pair count and accumulates the
 * per-tile pair histogram `tile_counts` (ntiles ints, zeroed by the caller).
 * color_source: SS_COLOR_EXPLICIT reads `colors_in` (n,3); SS_COLOR_IBL shades
 * against `env` in float64 like the reference; SS_COLOR_IBL_F32 shades in
 * float32 (the training step: colours within ~1e-6 relative, the forward
 * state the float32 shading adjoint of ss_chain_backward recomputes);
 * SS_COLOR_ALBEDO uses sigmoid(albedo_raw).  `flags` (int[4],
 * zeroed by caller) receives [0] zero-norm quaternion seen, [1] non-finite
 * colour seen.  bininfo (n x 4 uint32, nullable): the binning input of
 * ss_bin_sort (packed rect, order-preserving z_start bits). */
int ss_preprocess(const SsCloud *cloud, const SsCamera *cam, const SsPreprocessOpts *opt,
                  int color_source, const float *colors_in, const SsEnv *env,
                  float *records, int8_t *cull, int32_t *pair_count, int32_t *tile_counts,
                  uint32_t *bininfo, const SsProjAux *aux, int32_t *flags, void *stream);

/* ---- per-step surfel prepass ----------------------------------------------
 * The view-independent part of ss_preprocess for one optimisation step
 * (every view of a step sees the same parameters): the float32 scaled
 * tangent frame (quat_to_frame and exp(log_scales), surfels.py:40-51,
 * preprocess.py:38-60), the finiteness test, and -- with the float64 env maps
 * -- the float64 activations, normal and diffuse lookup of shade_surfels
 * (shading.py:463-471).  `prepass`: ss_surfel_prepass_bytes(n) of caller
 * scratch, 16-byte aligned.  ss_preprocess_prepared is ss_preprocess reading
 * it instead of recomputing: records, colours and branch state are
 * bit-identical. */
size_t ss_surfel_prepass_bytes(int n);
int ss_surfel_prepass(const SsCloud *cloud, const SsEnv *env, void *prepass, void *stream);
int ss_preprocess_prepared(const SsCloud *cloud, const SsCamera *cam, const SsPreprocessOpts *opt,
                           int color_source, const float *colors_in, const SsEnv *env,
                           float *records, int8_t *cull, int32_t *pair_count, int32_t *tile_counts,
                           uint32_t *bininfo, const SsProjAux *aux, int32_t *flags, const void *prepass,
                           void *stream);

/* ---- records from a ProjectedSurfels ---------------------------------------
 * render(..., proj=P) reuse and bin_and_sort(P) (rasterizer.py:92-116,
 * :331-339): packs the k compacted rows of a ProjectedSurfels (t1, t2, t4,
 * sinv (k,3); n_f, view_z, eps_z (k,); rect (k,4) int32) into records
 * source_index[j] (nullable: row j), colours from `colors` (per SOURCE row,
 * (n,3), nullable: 0), with the preprocess kernel's certified coverage
 * margin, bin info and tile histogram (tile_counts zeroed by the caller).
 * Rows not named by source_index are left as the caller initialised them
 * (zero rect, its cull code). */
int ss_pack_records(int k, const float *t1, const float *t2, const float *t4, const float *sinv,
                    const float *n_f, const float *view_z, const float *eps_z, const int32_t *rect,
                    const int32_t *source_index, const float *colors, int width, int height, int tile,
                    float *records, uint32_t *bininfo, int32_t *tile_counts, void *stream);

/* ---- tile binning with deterministic order ---------------------------------
 * Replaces the rest of bin_and_sort() (rasterizer.py:106-116): exclusive scan
 * of tile_counts into tile_offsets (ntiles+1 int32), bucket scatter of
 * (z_start, record) keys, and a per-tile sort by (z_start, record index) so
 * the result equals np.lexsort((rec, z_start, tile)) bit for bit.
 * pair_capacity bounds pair_rec/keys; flags[2] is set when it overflowed
 * and flags[3] receives max(flags[3], pairs this view needs).  On overflow
 * the offsets are clamped to the capacity (the excess pairs are dropped, the
 * results are wrong but every kernel stays inside the caller's buffers):
 * the caller grows the buffers to flags[3] and re-runs the view.
 * keys: uint64 scratch of pair_capacity entries; cursors: ntiles ints scratch.
 * pair_rect (2 uint32 per pair) receives each pair's record rect packed as
 * (x0 | y0 << 16, x1 | y1 << 16), the rasterisers' cull input.  bininfo: the
 * preprocess output (n x 4 uint32: packed rect, order-preserving z_start
 * bits, 0) -- 16 bytes per record instead of the 96-byte record. */
int ss_bin_sort(int n, const uint32_t *bininfo, const int8_t *cull, int width, int height, int tile,
                const int32_t *tile_counts, int32_t *tile_offsets, int32_t *cursors,
                uint64_t *keys, int32_t *pair_rec, uint32_t *pair_rect, int64_t pair_capacity,
                int32_t *flags, int32_t *tile_order, void *stream);
/* tile_order (ntiles int32, nullable): a launch order for the rasterisers,
 * tiles grouped by descending pair count (heavy first). */

/* ---- raster forward -------------------------------------------------------
 * Replaces _forward_kernel (rasterizer.py:119-249), interval depth mode.
 * rgb (H,W,3), alpha/depth (H,W) float32, nlayers (H,W) int32 are written for
 * every pixel.  Nullable extras: pair_cover (per pair int32, with_cover_counts),
 * stacks (collect_stacks; st_w/st_z/st_z2 (H,W,k), st_c (H,W,k,3), st_n (H,W,k)),
 * discarded (1 int64, the discarded_overflow statistic). */
typedef struct SsStacks { float *w, *c, *z, *z2; int32_t *n; } SsStacks;
int ss_raster_forward(int width, int height, int tile, const int32_t *tile_offsets,
                      const int32_t *pair_rec, const uint32_t *pair_rect, const float *records, const float *background,
                      int k_max, float *rgb, float *alpha, float *depth, int32_t *nlayers,
                      int32_t *pair_cover, const SsStacks *stacks, unsigned long long *discarded,
                      void *stream);

/* ---- raster backward ------------------------------------------------------
 * Replaces _backward_kernel (backward.py:48-321) and the pair reduction
 * (backward.py:382-396).  g_rgb (H,W,3) / g_alpha (H,W) float32 upstream
 * gradients (g_alpha nullable).  Accumulates into rec_acc (n x 20 float,
 * zeroed by the caller): [0:3] dt1, [3:6] dt2, [6:9] dt4, [9:12] dSigma^-1,
 * [12] dn_f, [13:16] dcolour, [16] dview_z, [17] screen-space |g| sum,
 * [18] covering-pixel count (as float bits of an int32 counter).  cons_loss
 * (1 double, zeroed) receives the consolidation penalty value. */
int ss_raster_backward(int width, int height, int tile, const int32_t *tile_offsets,
                       const int32_t *pair_rec, const uint32_t *pair_rect, const float *records, const float *background,
                       int k_max, const float *g_rgb, const float *g_alpha, float cons_scale,
                       float *rec_acc, double *cons_loss, void *stream);

/* ---- fused training step (SURVEY §8d "fwd+bwd view") ----------------------
 * ss_train_forward: the forward walk fused with the L1 photometric loss
 * (losses.py:94-108, lambda_ssim=0) against `target` (H,W,3) and with the
 * per-pixel suffix recursion of backward.py:201-238.  Writes per pixel and
 * layer the float4 (A_hi, dL/dC_raw rgb) into `coef` (k_max*H*W*9 floats:
 * k_max layer-major float4 planes, then k_max float planes of A_lo, then
 * k_max float4 planes the deferred variant uses for the low parts of its
 * float64 layer sums; A = A_hi + A_lo is formed from the float-rounded
 * dL/dC_raw so that the backward's g_w = A + dL/dC_raw . colour keeps the
 * record colour - layer mean colour difference exactly), per pixel a packed header `pix_hdr` (H*W x 8
 * int32: number of closed layers, then the depths at which layers 0..6
 * closed, as float bits; words past the closed count are not written) and
 * the closing depths of layers >= 7 into `thr` (k_max*H*W floats, plane j), and adds sum|rgb - target| into loss_sum (1 double).
 * rgb (H,W,3) is nullable.
 * ss_train_backward_records: pass 2 of backward.py:240-320 without the walk:
 * a covering record with interval start zs belongs to layer
 * #{j : closing depth_j < zs}; records are counting-sorted
 * by rect area and an 8-lane group per record sweeps its rect.  The rec_acc row of every kept record is OVERWRITTEN (committed once,
 * no atomics, no memset needed; culled rows untouched -- ss_chain_backward
 * skips them); channel 16 (dview_z) is 0 without a consolidation term.
 * pixel_ndc: scratch of ss_train_backward_scratch_words(n, width, height)
 * 32-bit words (0 on invalid sizes). */
int ss_train_forward(int width, int height, int tile, const int32_t *tile_offsets,
                     const int32_t *pair_rec, const uint32_t *pair_rect, const float *records,
                     const float *background, int k_max, const float *target, float *coef, float *thr,
                     int32_t *pix_hdr, double *loss_sum, float *rgb, float *alpha, const int32_t *tile_order,
                     void *stream);
/* ss_train_forward with target == NULL is the DEFERRED-loss variant (any
 * image loss, e.g. the reference fit loss of train.py:194-206): it writes rgb
 * (required), alpha (nullable) and, per pixel and layer, the raw layer sums
 * (W, C rgb) into coef; after the loss has produced g_rgb (and g_alpha),
 * ss_train_coefs turns them into the backward coefficients in place (suffix
 * recursion of backward.py:201-238 incl. the coverage term).  pix_hdr.x =
 * closed layers | layer count << 8. */
/* g_rgb64 (nullable): the same image gradient in float64 (ss_photometric_loss
 * grad64), used instead of g_rgb -- the layer coefficients' colour terms
 * cancel, so a float32-rounded gradient biases them by ~1e-5 */
int ss_train_coefs(int width, int height, int k_max, const int32_t *pix_hdr, float *coef, const float *g_rgb,
                   const double *g_rgb64, const float *g_alpha, const float *background, void *stream);
/* The same three steps with the consolidation penalty (backward.py:160-320
 * with cons_scale > 0): ss_train_forward_zstats is the deferred forward that
 * also writes, per pixel and layer, the depth moments (z0, sum w dz,
 * sum w dz^2, 0), dz = view_z - z0 of the layer's first covering member,
 * into `zstats` (k_max*H*W float4); ss_train_coefs_cons turns coef and zstats
 * in place into the layer coefficients and the penalty's per-layer
 * (B, Q, z_bar, var) and adds the penalty value into cons_loss (1 double);
 * ss_train_backward_records_cons adds the penalty's weight and depth terms
 * (accumulator slot 16 = dL/dview_z). */
int ss_train_forward_zstats(int width, int height, int tile, const int32_t *tile_offsets,
                            const int32_t *pair_rec, const uint32_t *pair_rect, const float *records,
                            const float *background, int k_max, float *coef, float *thr, int32_t *pix_hdr,
                            float *rgb, float *alpha, const int32_t *tile_order, float *zstats, void *stream);
int ss_train_coefs_cons(int width, int height, int k_max, const int32_t *pix_hdr, float *coef, float *zstats,
                        const float *g_rgb, const double *g_rgb64, const float *g_alpha, const float *background,
                        double cons_scale, double *cons_loss, void *stream);
int ss_train_backward_records_cons(int n, const int8_t *cull, const float *records, int width, int height,
                                   int k_max, const float *coef, const float *thr, const int32_t *pix_hdr,
                                   const float *zcoef, float *pixel_ndc, float *rec_acc, double *rec_acc64,
                                   void *stream);
size_t ss_train_backward_scratch_words(int n, int width, int height);
/* rec_acc64: n x SS_ACC64_WIDTH doubles (no initialisation needed): the
 * float64 channel sums of the big records (rects > 512 px, ~0.1% of them,
 * evaluated with the reference's own per-item arithmetic), referenced from
 * their rec_acc rows (SS_ACC_F64); pass the same buffer to
 * ss_chain_backward. */
int ss_train_backward_records(int n, const int8_t *cull, const float *records, int width, int height,
                              int k_max, const float *coef, const float *thr, const int32_t *pix_hdr,
                              float *pixel_ndc, float *rec_acc, double *rec_acc64, void *stream);

/* ---- image losses ---------------------------------------
 * Replace the reference's numpy/scipy losses: tone_map / tone_map_backward
 * (shading.py:54-79; tone_mode 0 = 'ldr', 1 = 'hdr-loss', -1 = identity),
 * ssim_loss / photometric_loss (losses.py:45-108) and silhouette_loss
 * (losses.py:111-123).  Images (H, W, C) float32, C in {1, 3}; float64
 * internally.  ss_photometric_loss: loss = (1 - l) mean|T(x) - T(y)| +
 * l (1 - mean SSIM(T(x), T(y))), its gradient w.r.t. x (through T) into grad
 * (and, nullable, in float64 into grad64),
 * out[3] = {loss, L1, 1 - SSIM} (device doubles, no host sync); lambda = 1
 * gives ssim_loss.  workspace: ss_photometric_workspace() bytes.
 * ss_silhouette_loss: out[1] = 1 - soft IoU, grad d/d alpha; workspace 2 doubles. */
size_t ss_photometric_workspace(int height, int width, int channels);
int ss_photometric_loss(int height, int width, int channels, const float *x, const float *y, int tone_mode,
                        double lambda_ssim, double *out, float *grad, double *grad64, double *workspace,
                        void *stream);
int ss_tone_map(int64_t n, const float *img, int tone_mode, float *out, void *stream);
int ss_tone_map_backward(int64_t n, const float *img, int tone_mode, const float *g_out, float *g_in, void *stream);
int ss_silhouette_loss(int64_t n, const float *alpha, const float *mask, double *out, float *grad,
                       double *workspace, void *stream);

/* ---- oriented KNN index + normal consistency ------------
 * ss_knn_oriented replaces NeighborIndex.rebuild (knn.py:31-81): for every
 * surfel the k (<= 16) nearest other surfels with n_i . n_j > 0, ascending
 * (distance, index), -1 padded, into neighbors (n, k) int64; mean_dist (n)
 * float64 = mean accepted distance, or the distance to the nearest other
 * surfel when none qualifies.  The grid is the caller's: cells of
 * ss_grid_cells (origin3, cell, dim <= 1024), sorted (sorted_cells, order).
 * ss_normal_consistency replaces normal_consistency_loss (losses.py:189-220):
 * loss (1 double), g_quats (n, 4) float32; g_normals: n*3 float64 scratch. */
int ss_knn_oriented(int n, const float *centers, const float *quats, const int32_t *order,
                    const int32_t *sorted_cells, const float *origin3, float cell, int dim, int k,
                    int64_t *neighbors, double *mean_dist, void *stream);
int ss_normal_consistency(int n, int k, const float *centers, const float *quats, const int64_t *neighbors,
                          const double *mean_dist, double *loss, double *g_normals, float *g_quats, void *stream);

/* Dense cell grid for the neighbour queries (no host round trip, no binary
 * searches): ss_cell_grid_build sizes cubic cells over the centres'
 * bounding box on the device and counting-sorts the surfels into dim^3
 * cells (per-cell [start, end) table); `grid`: ss_cell_grid_words(n, dim)
 * int32 words of caller scratch, dim <= 512; it also keeps a cell-ordered
 * float4 copy of the centres (x, y, z, source index).  ss_knn_dense is
 * ss_knn_oriented on it (queries in cell order; grid_coarse: a second grid
 * of the same centres with wider cells, dim_coarse ~ dim / 4, on which the
 * queries whose k-th oriented neighbour lies beyond a few fine shells are
 * finished; workspace: ss_knn_workspace_bytes(n) of caller scratch, 8-byte
 * aligned), ss_isolation_dense the isolation test of densify.py:118-123. */
size_t ss_cell_grid_words(int n, int dim);
int ss_cell_grid_build(int n, const float *centers, int dim, int32_t *grid, void *stream);
size_t ss_knn_workspace_bytes(int n);
int ss_knn_dense(int n, const float *centers, const float *quats, const int32_t *grid, int dim,
                 const int32_t *grid_coarse, int dim_coarse, int k, void *workspace, int64_t *neighbors,
                 double *mean_dist, void *stream);
int ss_isolation_dense(int n, const float *centers, const float *log_scales, const int32_t *grid, int dim,
                       uint8_t *isolated, void *stream);

/* ---- chain backward -------------------------------------------------------
 * Replaces the per-surfel tail of backward_image() (backward.py:398-461,
 * 473-548), shade_backward() (shading.py:525-616) and quat_frame_backward()
 * (surfels.py:54-77).  Reads rec_acc and ADDS into the parameter gradients
 * (so multi-view steps accumulate in place): g_centers (n,3), g_quats (n,4),
 * g_log_scales (n,2), g_albedo_raw (n,3), g_metallic_raw, g_roughness_raw,
 * g_colors (n,3, nullable), ss_grad (n), touched (n int32 covering-pixel
 * counts, nullable), view_count (n float32, nullable: +1 for every surfel
 * that covers at least one pixel of this view -- the per-view `touched` bool
 * of backward.py:432-441 summed over a step's views, as DensifyStats
 * accumulates it, densify.py:35-37).  With
 * SS_COLOR_IBL it also scatters the derived-map gradients into d_diffuse
 * (He,We,3) and d_specular (L,He,We,3) (float64, accumulated with fp64
 * atomics: a step sums 64 views x N surfels x 36 scatters into them). */
typedef struct SsGrads {
    float *centers, *quats, *log_scales, *albedo_raw, *metallic_raw, *roughness_raw;
    float *colors;     /* nullable */
    float *ss_grad;
    int32_t *touched;
    double *d_diffuse, *d_specular;  /* nullable unless SS_COLOR_IBL */
    /* nullable: per-view float32 derived-map accumulators with 16-byte texels
     * ((He,We,4) and (L,He,We,4), zero on entry); when given, the shading
     * adjoint scatters into them with vector float32 reductions and
     * ss_env_grad_merge later folds them into d_diffuse / d_specular */
    float *d_diffuse4, *d_specular4;
    float *view_count;  /* nullable */
} SsGrads;
/* shade_cells (nullable, SS_COLOR_IBL): the SsProjAux.cells_packed of this
 * view's preprocess; the shading adjoint then runs in float32 on the
 * forward's own float64 branch decisions (texel cells, level, clip flags)
 * instead of re-deriving them in float64. */
int ss_chain_backward(const SsCloud *cloud, const SsCamera *cam, const SsPreprocessOpts *opt,
                      int color_source, const SsEnv *env, const int8_t *cull,
                      const float *rec_acc, const double *rec_acc64, const uint32_t *shade_cells,
                      const SsGrads *grads, void *stream);
/* ss_chain_backward inside a training step whose prepass (ss_surfel_prepass,
 * this step's parameters and env) is given: the shading adjoint takes the
 * normal's diffuse lookup, texel derivatives and coord_grad_to_dir map from
 * the prepass, and instead of scattering the diffuse-lookup upstream into
 * grads->d_diffuse4 through the four bilinear taps per view it adds it per
 * surfel into g_ld (n x 4 floats, rgb + pad; zero before the step's first
 * view); ss_diffuse_scatter then applies the (view independent) taps once per
 * step into d_diffuse (He x We x 3 doubles, +=) and zeroes g_ld.  Same result
 * as the per-view scatter up to float summation order
 * (bilinear_scatter, shading.py:248-260, 583-597). */
int ss_chain_backward_prepared(const SsCloud *cloud, const SsCamera *cam, const SsPreprocessOpts *opt,
                               int color_source, const SsEnv *env, const int8_t *cull,
                               const float *rec_acc, const double *rec_acc64, const uint32_t *shade_cells,
                               const SsGrads *grads, const void *prepass, float *g_ld, void *stream);
int ss_diffuse_scatter(int n, const SsEnv *env, const void *prepass, float *g_ld, double *d_diffuse, void *stream);

/* ss_env_grad_merge: dst[3 t + c] += src4[4 t + c] (float64 += float32) for
 * t < texels, c < 3, and zeroes src4 (the per-view derived-map accumulators
 * of SsGrads.d_diffuse4 / d_specular4). */
int ss_env_grad_merge(int64_t texels, float *src4, double *dst, void *stream);

/* ---- environment ----------------------------------------------------------
 * ss_brdf_lut: brdf_lut() (shading.py:118-156) -> lut (res,res,2) float.
 * ss_env_refresh: EnvironmentLight.refresh (shading.py:369-379): base_log
 *   (He,We,3) -> base, diffuse (He,We,3), specular (L,He,We,3).
 * ss_env_adjoint: env_gradient (shading.py:381-394): d_diffuse, d_specular
 *   -> d_base_log (He,We,3) and d_base (He,We,3 doubles, also the scratch of
 *   the accumulation).
 * The prefilter operators of the reference (build_diffuse_operator /
 * build_specular_operator, shading.py:275-331: dense T x T float64) are
 * passed as a caller-owned bundle, built once per env shape:
 *   rowsum  (He*We doubles) diffuse row sums, from ss_env_rowsums;
 *   khat    (nullable) the diffuse kernel's spectrum, ss_env_khat_words(He,We)
 *           doubles filled by ss_env_khat (0 words: odd widths / too large;
 *           NULL selects the O(T^2) N-body quadrature);
 *   row_ptr/col/rval, col_ptr/row/cval (nullable) the sparse specular
 *           operators of ss_spec_op_count / ss_spec_op_fill and their per-level
 *           transpose (CSC by a stable sort); NULL regenerates the GGX samples
 *           on the fly;
 *   work    3*He*We doubles of scratch.
 * The library keeps no state and allocates nothing. */
typedef struct SsEnvOps {
    const double *rowsum;
    const double *khat;
    const int64_t *row_ptr; const int32_t *col; const double *rval;
    const int64_t *col_ptr; const int32_t *row; const double *cval;
    double *work;
} SsEnvOps;
int ss_brdf_lut(int res, int samples, float *lut, void *stream);
size_t ss_env_khat_words(int he, int we);
int ss_env_khat(int he, int we, double *khat, void *stream);
int ss_env_rowsums(int he, int we, const double *khat, double *rowsum, double *work, void *stream);
/* The maps are computed in float64 like the reference's (base = exp(base_log),
 * dense float64 operator products, shading.py:369-379) into base64 (He,We,3),
 * diffuse64 (He,We,3), specular64 (L,He,We,3) -- read by the float64 shading
 * (SsEnv.diffuse64/specular64) -- and rounded into the float maps. */
int ss_env_refresh(int he, int we, int levels, int samples, const float *base_log, const SsEnvOps *ops,
                   float *base, float *diffuse, float *specular, double *base64, double *diffuse64,
                   double *specular64, void *stream);
/* ss_env_refresh64: ss_env_refresh from a float64 base_log (the optimiser's
 * float64 master of the environment, like the reference's float64 env). */
int ss_env_refresh64(int he, int we, int levels, int samples, const double *base_log, const SsEnvOps *ops,
                     float *base, float *diffuse, float *specular, double *base64, double *diffuse64,
                     double *specular64, void *stream);
int ss_env_adjoint(int he, int we, int levels, int samples, const double *base64, const SsEnvOps *ops,
                   const double *d_diffuse, const double *d_specular, double *d_base, float *d_base_log,
                   void *stream);

/* Specular prefilter operators S_l (l = 1..L-1) as a sparse matrix, built
 * once per (He, We, L, samples) instead of regenerating 128 GGX samples per
 * texel per call.  Rows r = (l-1)*T + i; duplicate columns are kept (the SpMV
 * sums them); weights are divided by the row weight sum; empty rows hold one
 * identity entry.  ss_spec_op_count -> row_nnz ((L-1)*T int32), the caller
 * scans it into row_ptr ((L-1)*T+1 int64), ss_spec_op_fill -> col (int32),
 * val (double).  The caller builds the per-level transpose (CSC: col_ptr over
 * (l-1)*T + j, row, val) with a stable sort and passes both in SsEnvOps.
 * ss_spec_apply / ss_spec_apply_t expose the two products directly. */
int ss_spec_op_count(int he, int we, int levels, int samples, int32_t *row_nnz, void *stream);
int ss_spec_op_fill(int he, int we, int levels, int samples, const int64_t *row_ptr, int32_t *col, double *val,
                    void *stream);
int ss_spec_apply(int he, int we, int levels, const int64_t *row_ptr, const int32_t *col, const double *val,
                  const double *base, double *specular, float *specular_f, void *stream);
int ss_spec_apply_t(int he, int we, int levels, const int64_t *col_ptr, const int32_t *row, const double *val,
                    const double *d_specular, double *d_base, void *stream);

/* ---- optimiser ------------------------------------------------------------
 * Adam.step (adam.py:21-41) fused over one parameter tensor of `count`
 * floats; m, v float32 state; bias corrections from step t (>= 1). */
int ss_adam_step(int64_t count, float *param, const float *grad, float *m, float *v,
                 int t, float lr, float beta1, float beta2, float eps, void *stream);
/* ss_adam_multi: the same update for up to 8 tensors in ONE launch (params[k],
 * grads[k], m[k], v[k] of counts[k] floats, step count steps[k], lr lrs[k]);
 * tensors with quat_flags[k] != 0 (n x 4) are renormalised right after their
 * update (train.py:241-246). */
int ss_adam_multi(int ntensors, float *const *params, const float *const *grads, float *const *m,
                  float *const *v, const int64_t *counts, const int *steps, const float *lrs,
                  const int *quat_flags, float beta1, float beta2, float eps, void *stream);
/* The same two entry points with float64 moments, the reference's state
 * precision (adam.py:26-28: np.float64 m, v); parameters and gradients stay
 * float32, the update is float64 in both variants. */
int ss_adam_step_f64(int64_t count, float *param, const float *grad, double *m, double *v,
                     int t, float lr, float beta1, float beta2, float eps, void *stream);
int ss_adam_multi_f64(int ntensors, float *const *params, const float *const *grads, double *const *m,
                      double *const *v, const int64_t *counts, const int *steps, const float *lrs,
                      const int *quat_flags, float beta1, float beta2, float eps, void *stream);
/* ss_adam_multi_master: the same multi-tensor step on float64 MASTER
 * parameters `masters` (the reference's fit keeps its parameters in float64,
 * train.py:168-174): the reference's numpy update operation by operation
 * (adam.py:31-41; c1s / c2s = 1 - beta^t per tensor, lrs in float64),
 * quaternion segments renormalised in float64 (surfels.py:31-37); `params`
 * receives the float32 rounding of each updated master value. */
int ss_adam_multi_master(int ntensors, float *const *params, double *const *masters, const float *const *grads,
                         double *const *m, double *const *v, const int64_t *counts, const double *c1s,
                         const double *c2s, const double *lrs, const int *quat_flags, double beta1, double beta2,
                         double eps, void *stream);
/* q <- q / |q| after the step (train.py:246). */
int ss_normalize_quats(int n, float *quats, void *stream);

/* ---- refinement scan (densify.py:101-202) ---------------------------------
 * Isolation prune (densify.py:118-123): isolated[i] = 1 iff no other centre
 * lies within 3 * max(exp(log_scales[i])).  Fixed-radius existence query on a
 * uniform grid: ss_grid_cells writes each centre's linear cell id
 * ((x*dim + y)*dim + z, axes clamped to [0, dim), dim <= 1024); the caller
 * sorts the ids (sorted_cells, with the permutation `order`); ss_isolation
 * visits the cells overlapping each query ball by binary search. */
int ss_grid_cells(int n, const float *centers, const float *origin3, float cell, int dim,
                  int32_t *cell_of, void *stream);
int ss_isolation(int n, const float *centers, const float *log_scales, const int32_t *order,
                 const int32_t *sorted_cells, const float *origin3, float cell, int dim,
                 uint8_t *isolated, void *stream);
/* The same query with the grid kept on the device (no host round trip):
 * ss_grid_fit writes origin (3 floats), cell, dim (int bits) into `grid`
 * (16 words of device scratch) from the centres' bounding box and the mean
 * support; ss_grid_cells_d / ss_isolation_d read it from there. */
int ss_grid_fit(int n, const float *centers, const float *log_scales, float *grid, void *stream);
int ss_grid_cells_d(int n, const float *centers, const float *grid, int32_t *cell_of, void *stream);
int ss_isolation_d(int n, const float *centers, const float *log_scales, const int32_t *order,
                   const int32_t *sorted_cells, const float *grid, uint8_t *isolated, void *stream);
/* Split children (densify.py:60-98): parent rows `parents` (nsplit) produce
 * the (+) child at out row plus_row0+k and the (-) child at minus_row0+k;
 * only centres and log-scales differ from the parent (the caller copies the
 * other attributes). `origin3` is a HOST pointer. */
int ss_split_children(int nsplit, const int32_t *parents, const float *centers, const float *quats,
                      const float *log_scales, float *out_centers, float *out_log_scales,
                      int64_t plus_row0, int64_t minus_row0, void *stream);

/* ---- refinement scan on the device (densify.py:168-202, adam.py:43-58) -----
 * ss_refine_plan: prune_keep_mask (stale: grad_sum <= 0; isolated: the
 * ss_isolation flags; floater: front > 0 && outside >= front, votes
 * nullable together), mean gradient grad_sum / max(view_count, 1),
 * select_split (threshold max(np.quantile(mean_grad[active], q), floor)
 * with numpy's 'linear' method; candidates mean_grad >= threshold and
 * max scale > mean_neighbor_dist) and the budget (the max_surfels - kept
 * largest mean gradients, ties in index order).  Per row: kind (0 removed,
 * 1 stay, 2 split) and dst (stay: output row; split: rank among the split
 * rows: +child at n_stay + rank, -child at n_stay + n_split + rank).
 * counts (9 int64, device): n_out, kept, split, stale, isolated, floater,
 * active, candidates, then the threshold's float64 bits.  workspace:
 * ss_refine_workspace_bytes(n).  No host synchronisation; a fixed launch
 * sequence (order statistics by an 8-bit radix select on the float64 bits).
 * ss_refine_apply: the new rows of up to 32 row-major tensors (src[t] n
 * rows, dst[t] capacity >= n_out rows, row_bytes[t] a multiple of 4) by
 * role: 0 children copy the parent row, 1 children zero (Adam moments),
 * 2 centres (children +-(s_max / 2) along the longer tangent axis), 3 log
 * scales (that axis x 0.7) -- split_cloud (densify.py:60-98); index_map
 * (capacity int64, nullable): source row of each new row, -1 for children
 * (workspace: the one ss_refine_plan filled). */
size_t ss_refine_workspace_bytes(int n);
int ss_refine_plan(int n, const double *grad_sum, const int64_t *view_count, const uint8_t *isolated,
                   const int64_t *outside_votes, const int64_t *front_votes, const float *log_scales,
                   const double *mean_neighbor_dist, int64_t max_surfels, double quantile, double grad_floor,
                   int32_t *dst, uint8_t *kind, int64_t *counts, void *workspace, void *stream);
int ss_refine_apply(int n, const uint8_t *kind, const int32_t *dst, const float *centers, const float *quats,
                    const float *log_scales, int ntensors, const void *const *src, void *const *dst_tensors,
                    const int *row_bytes, const int *roles, int64_t *index_map, const void *workspace,
                    void *stream);

/* Diagnostic for the rasterisers' fast coverage test: counts[0] (pixel,
 * in-rect record) evaluations, counts[1] decisions differing from the exact
 * reference arithmetic (0 by construction), counts[2] exact fallbacks taken.
 * counts: 3 uint64, zeroed by the caller. */
/* Per-CTA (forward) / per-warp (record backward) timestamps for the tail
 * analysis: only in a library built with -DSS_CTA_TIMING (else
 * SS_ERR_INVALID); buf = 3 uint64 (start ns, end ns, SM id) per CTA / warp
 * of the next launches, nullptr to stop. */
int ss_debug_set_fwd_timing(void *buf);
int ss_debug_set_bwd_timing(void *buf);
int ss_debug_cover_check(int width, int height, int tile, const int32_t *tile_offsets,
                         const int32_t *pair_rec, const uint32_t *pair_rect, const float *records,
                         unsigned long long *counts, void *stream);

const char *ss_last_error(void);
int ss_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SS_ABI_H */
