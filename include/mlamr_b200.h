/*
 * mlamr_b200 — C ABI of the B200 multilayer-AMR hot path.
 *
 * Plain pointers and sizes only.  All array pointers are DEVICE pointers
 * unless the parameter name starts with `h_`.  `stream` is a cudaStream_t
 * passed as void*.  Every entry point is asynchronous on `stream` and
 * returns 0 on a successful launch; device-side faults (CFL violation,
 * geometry errors) are reported through the int32 status word described
 * below, which the host shim maps onto the reference's exception types
 * (errors.py:4-37 of /root/reference/pkg/src/mlamr).
 *
 * Data layout: one pool per level.  Patch p of a level owns a
 * (ny+4) x (nx+4) row-major block (x fastest, ghost width 2, mesh.py:181-186)
 * starting at element offset[p]; the 3M state fields (h_0..h_{M-1},
 * hu_0.., hv_0..) are planes `field_stride` elements apart; bathymetry is
 * one more plane of the same shape.  Boxes are inclusive global indices
 * (lo_i, lo_j, hi_i, hi_j) of the patch interior (mesh.py:40-113).
 *
 * Owner maps are int32 arrays over a level's index space extended by the
 * 2-cell frame: cell (i, j) is at [(j + 2) * (level_nx + 4) + (i + 2)].
 */
#ifndef MLAMR_B200_H
#define MLAMR_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MLAMR_MAX_LAYERS 4

/* status word bits (device int32) */
#define MLAMR_ST_CFL 1        /* CflViolationError  (physics.py:342-347) */
#define MLAMR_ST_GEOMETRY 2   /* GeometryError      (refine.py:210-225)  */
#define MLAMR_ST_NONFINITE 4  /* NumericalAbortError (driver.py:286-297) */
#define MLAMR_ST_BATHY 8      /* AssertionError: bathymetry does not telescope (coarsen.py:79-100) */

/* boundary kinds, per side in the order left, right, bottom, top */
#define MLAMR_BC_WALL 0
#define MLAMR_BC_OUTFLOW 1

typedef struct mlamr_params {
    int32_t num_layers;                 /* M (1..4)                           */
    int32_t pad_;
    double gravity;                     /* g                                  */
    double dry_tolerance;               /* tol                                */
    double densities[MLAMR_MAX_LAYERS]; /* top to bottom (state.py:19-53)     */
} mlamr_params;

typedef struct mlamr_level {
    int32_t num_patches;
    int32_t num_layers;
    int32_t level_nx, level_ny;   /* level index space                   */
    double dx, dy;
    int64_t field_stride;         /* elements between state planes       */
    const int32_t *box;           /* [P*4]                               */
    const int64_t *offset;        /* [P]                                 */
    double *state;                /* [3M * field_stride]                 */
    double *bathy;                /* [field_stride]                      */
    const int32_t *own;           /* interior-owner map (last wins)      */
    const int32_t *gown;          /* frame-owner map (first wins) or NULL */
} mlamr_level;

/* ---- patch table: the handle-based runtime -------------
 * A stateful level/patch manager over the kernels below, for callers that
 * hold the reference's host Patch arrays (mesh.py:158-232): every argument
 * is a HOST pointer or a size.  Per patch, h/hu/hv are (M, ny+4, nx+4) and
 * bathy (ny+4, nx+4) row-major float64 arrays, ghost frames included.
 * Return values: 0, a CUDA error code, -1 (bad handle/level), -2 (out of
 * memory), or MLAMR_ST_* status bits (CFL violation: nothing was written,
 * as physics.py:342-347 raises before touching a patch).
 *   create / destroy / set_level(level, nx, ny, dx, dy, r_x, r_y, r_t of
 *   the ratio to level+1) / set_level_bathymetry(in-domain [ny][nx], used
 *   by regrid for new patches) / upload_patches (replaces the level's
 *   patches) / download (current state incl. frames) / num_patches /
 *   max_speed (stable_dt's speeds, physics.py:261-289) / stash(t0, dt)
 *   (the current state becomes the time-blend source of the children,
 *   driver.py:260-264) / fill_ghosts(t) (driver.py:175-190) / step_level
 *   (out_counters[M+2] = clipped depth sums per layer, shear fixes,
 *   wet-prefix repairs) / average_down(fine level) / regrid(level, new
 *   boxes) (regrid.rebuild_child_level's data movement, refine and
 *   derefine mass deltas [M]) / composite_mass(out[M]) / check_finite. */
typedef struct mlamr_pt mlamr_pt;
mlamr_pt *mlamr_pt_create(mlamr_params prm, const int32_t *h_bcs, void *stream);
void mlamr_pt_destroy(mlamr_pt *pt);
int mlamr_pt_set_level(mlamr_pt *pt, int level, int nx, int ny, double dx, double dy, int r_x, int r_y, int r_t);
int mlamr_pt_set_level_bathymetry(mlamr_pt *pt, int level, const double *h_bathy);
int mlamr_pt_upload_patches(mlamr_pt *pt, int level, int n, const int32_t *h_boxes, const double *const *h,
                            const double *const *hu, const double *const *hv, const double *const *h_bathy);
int mlamr_pt_download(mlamr_pt *pt, int level, double *const *h, double *const *hu, double *const *hv);
int mlamr_pt_num_patches(mlamr_pt *pt, int level);
int mlamr_pt_max_speed(mlamr_pt *pt, int level, double *h_out_speed);
int mlamr_pt_stash(mlamr_pt *pt, int level, double t0, double dt);
int mlamr_pt_clear_stash(mlamr_pt *pt, int level);
int mlamr_pt_fill_ghosts(mlamr_pt *pt, int level, double t);
int mlamr_pt_step_level(mlamr_pt *pt, int level, double dt, int y_first, double *h_out_counters,
                        int *h_bad_patch);
int mlamr_pt_average_down(mlamr_pt *pt, int fine_level);
int mlamr_pt_regrid(mlamr_pt *pt, int level, int n, const int32_t *h_new_boxes, double *h_out_refine,
                    double *h_out_derefine);
int mlamr_pt_composite_mass(mlamr_pt *pt, double *h_out);
int mlamr_pt_check_finite(mlamr_pt *pt);
int mlamr_pt_status(mlamr_pt *pt);

/* ---- library ------------------------------------------------------------ */
/* Number of exported entry points / a version string (for smoke checks). */
int mlamr_version(void);
const char *mlamr_build_info(void);

/* ---- owner maps (replace the O(P^2) box scans of ghost.py:186-196,
 *      regrid.py:311-323, coarsen.py:57-75) -------------------------------
 * Paint the boxes of a level into an owner map that was pre-set to -1.
 * grow = 0 paints interiors, 2 interiors plus the ghost frame; first_wins
 * selects the smallest patch index (gather's ghost fallback, ghost.py:
 * 73-84) instead of the largest (later interiors overwrite, ghost.py:64-72).
 * r_x/r_y > 1 paints coarsened boxes into the parent's index space.
 * max_cells bounds the painted cells per box (grid sizing). */
int mlamr_paint_owner(int32_t *map, int map_nx, int map_ny, const int32_t *box,
                      int num_patches, int grow, int first_wins, int r_x, int r_y,
                      int max_cells, void *stream);

/* ---- K1: batched patch step (physics.step_patch, physics.py:330-386) -----
 * Reads `src_state` (ghosts filled), writes the stepped interior into
 * `dst_state`.  `tiles` is an int32 [n_tiles*3] work list (patch, j0, i0)
 * of interior tiles of tile_tx columns (32: 16x32 tiles, 320 threads; 16:
 * 16x16 tiles, 192 threads, for narrow-patch levels -- see
 * mlamr_step_tile).  Per-patch observed speeds of the pre-step state
 * go to `speed_bits` (int64 bit patterns, pre-set to -1 = all dry);
 * per-tile partials (sum of clipped negative depth per layer, hyperbolicity
 * fixes, wet-prefix repairs) to `tile_acc` [n_tiles * (M + 2)].
 * With a ghost plan (mlamr_ghost_plan's ghost_base/ghost_plan; NULL = read
 * the patch's own ghost frame), halo cells that have a sibling source are
 * read from the sibling's interior directly, so the sibling copy of the
 * ghost fill need not run for this level (patches that need physical BCs
 * excepted: their BC corners read the copied frame).
 * The call enqueues two kernels on `stream`: the work list expanded into
 * 32-byte tile descriptors (library-owned scratch per device and stream,
 * grown with the stream-ordered allocator), then the step.  Safe to call
 * from several host threads, also on one stream (the reference steps its
 * patches from a thread pool, driver.py:231-232).
 * Does nothing when *status != 0. */
int mlamr_step(mlamr_level lv, const double *src_state, double *dst_state,
               const int32_t *tiles, int n_tiles, int tile_tx, double dt, int y_first,
               mlamr_params prm, long long *speed_bits, double *tile_acc,
               const int32_t *status, const int64_t *ghost_base, const int64_t *ghost_plan,
               void *stream);

/* Select the K1 form for 32-column tiles and M <= 2: 0 = phase kernel
 * (default; per-cell phases between block barriers), 1 = line walker
 * (bit-identical, one interface per register window; env MLAMR_STEP=walk).
 * Returns the previous form, or -1 for an unknown one. */
int mlamr_set_step_form(int form);

/* Interior tile shape (rows, columns) the step kernel uses for a level
 * whose widest patch interior is max_patch_nx cells and num_layers layers;
 * the host builds that level's `tiles` with it and passes tx as tile_tx. */
int mlamr_step_tile(int max_patch_nx, int num_layers, int *ty, int *tx);

/* CFL guard (physics.py:342-347) + deterministic reduction of a step's
 * partials into acc[M + 2].  A patch whose speed*dt/min(dx,dy) > 1 gets its
 * interior restored from src (the reference raises before touching it),
 * MLAMR_ST_CFL is set and the smallest such patch index is atomically
 * min-ed into *bad_patch. */
int mlamr_step_finalize(mlamr_level lv, const double *src_state, double *dst_state,
                        const int32_t *tiles, int n_tiles, double dt,
                        mlamr_params prm, long long *speed_bits,
                        const double *tile_acc, double *acc, int32_t *status,
                        int32_t *bad_patch, int reset_speeds, void *stream);

/* Deterministic column sums of per-block partials (row-major [rows][cols]):
 * s_c = (sum over rows, fixed order) * scale; acc[c] = init ? s_c : acc[c]
 * + s_c, and acc2[c] += s_c when acc2 is given.  One launch in place of the
 * framework reductions the driver used for mass and refine/derefine
 * deltas. */
int mlamr_memset(void *ptr, int byte, long long nbytes, void *stream);  /* cudaMemsetAsync */
/* Host: the step tile list (patch, j0, i0) of int64 boxes [n][4] for tiles
 * of tile_y x tile_x, patch-major; returns the count (out NULL: count only). */
long long mlamr_tile_list(const int64_t *boxes, int n, int tile_y, int tile_x, int32_t *out);
int mlamr_sum_partials(const double *part, long long rows, int cols, double scale, double *acc,
                       double *acc2, int init, void *stream);

/* ---- K6: per-patch observed max wave speed (physics.py:261-278) --------- */
int mlamr_max_speed_tiles(mlamr_level lv, const double *state, const int32_t *tiles,
                          int n_tiles, int tile_tx, mlamr_params prm, long long *speed_bits,
                          void *stream);

/* ---- K2: ghost filling (ghost.py:145-197, driver.py:157-190) -------------
 * Coarse interpolation from the parent level, time-blended as
 * (1-theta)*old + theta*new when `parent_old_state` (the stash) is given
 * (ghost.py:68-71); then sibling copies; then physical BCs.  `parent` NULL
 * = coarsest level.  `bcs` is a HOST int32[4] (left, right, bottom, top). */
int mlamr_fill_ghosts(mlamr_level lv, const mlamr_level *parent,
                      const double *parent_old_state, double theta,
                      int r_x, int r_y, const int32_t *bcs,
                      mlamr_params prm, const int32_t *status,
                      const int32_t *patch_list, int n_list, void *stream);

/* K2 as a per-layout plan + three lean kernels.  mlamr_ghost_plan writes,
 * for every ghost cell of every patch (gbase = prefix sums of
 * 4*(nx+4)+4*ny per patch), the element offset of the sibling interior
 * cell covering it, -1 (in-domain, interpolate from the parent) or -2
 * (outside the level box, boundary condition).  mlamr_fill_ghosts_planned
 * then copies sibling cells, interpolates the compacted `interp_cells`
 * (int32 pairs patch, ghost index) from the (blended) parent and applies
 * the BCs of `bc_patches` -- the same values as mlamr_fill_ghosts.  With
 * `n_interp_dev` (device int32, e.g. from mlamr_plan_interp_cells) the
 * list's length is read on the device and n_interp is its capacity; NULL =
 * n_interp cells.  mlamr_plan_interp_cells compacts the plan's -1 cells of
 * the listed patches (NULL = all) into `cells` (int32 pairs, unordered) and
 * their number into *count, without a host round trip. */
int mlamr_ghost_plan(mlamr_level lv, const int64_t *gbase, int64_t *plan, int max_ghost, void *stream);
int mlamr_plan_interp_cells(mlamr_level lv, const int64_t *gbase, const int64_t *plan,
                            const int32_t *patch_list, int n_list, int max_ghost, int32_t *cells,
                            int32_t *count, void *stream);
int mlamr_fill_ghosts_planned(mlamr_level lv, const mlamr_level *parent, const double *parent_old_state,
                              double theta, int r_x, int r_y, const int32_t *bcs, mlamr_params prm,
                              const int32_t *status, const int64_t *gbase, const int64_t *plan,
                              const int32_t *patch_list, int n_list, int max_ghost,
                              const int32_t *interp_cells, int n_interp, const int32_t *n_interp_dev,
                              const int32_t *bc_patches, int n_bc, void *stream);

/* Patch bathymetry (frame included) from a level-wide array of in-domain
 * values, then ghost.apply_bathymetry_bcs (ghost.py:118-129). */
int mlamr_fill_bathymetry(mlamr_level lv, const double *level_bathy,
                          const int32_t *bcs, void *stream);

/* ---- K4: coarsening (coarsen.average_down, coarsen.py:30-76) ------------
 * Block means of every fine patch written over the coarse interiors that
 * own them (coarse.own); per-(fine patch, block) mass-change partials
 * [P_fine * blocks_per_patch * M]. */
int mlamr_average_down(mlamr_level fine, mlamr_level coarse, int r_x, int r_y,
                       mlamr_params prm, double *patch_delta, int blocks_per_patch,
                       const int32_t *status, void *stream);

/* The same coarsening over a flat list of all coarse cells of the fine
 * level (coarse_base[p] = first coarse cell of fine patch p, prefix sums;
 * n_coarse in total), without the mass-change partials: the driver's path,
 * whose blocks stay full for small patches. */
int mlamr_average_down_flat(mlamr_level fine, mlamr_level coarse, int r_x, int r_y, mlamr_params prm,
                            const int64_t *coarse_base, int64_t n_coarse, const int32_t *status,
                            void *stream);

/* check_bathymetry_consistency (coarsen.py:79-100) for every patch of a new
 * fine level against the coarse level's interiors: block_mean of the fine
 * bathymetry (the reference's numpy order, r <= 4) vs the coarse value,
 * |diff| > atol sets MLAMR_ST_BATHY and the smallest offending fine patch
 * index in *bad_patch.  `coarse_base` = prefix sums of the coarse cells
 * under each fine patch (as mlamr_average_down_flat). */
int mlamr_check_bathymetry(mlamr_level fine, mlamr_level coarse, int r_x, int r_y, double atol,
                           const int64_t *coarse_base, int64_t n_coarse, int32_t *status,
                           int32_t *bad_patch, void *stream);

/* ---- K3 + K5: regrid data movement (regrid.py:270-353) -------------------
 * Every new-patch interior cell is copied from the old patch covering it
 * (old.own), else refined from the parent's interiors (gather with
 * include_ghosts=False).  Refine-delta partials [P_new * blocks * M]. */
int mlamr_regrid_fill(mlamr_level newlv, mlamr_level oldlv, mlamr_level parent,
                      int r_x, int r_y, mlamr_params prm, double *refine_delta,
                      int blocks_per_patch, int32_t *status,
                      const int32_t *patch_list, int n_list, void *stream);
/* Derefine delta (regrid.py:329-348); new_child = the new patches'
 * coarsened owner map in the parent's index space. */
int mlamr_derefine_delta(mlamr_level oldlv, mlamr_level parent, const int32_t *new_child,
                         int r_x, int r_y, mlamr_params prm, double *derefine_delta,
                         int blocks_per_patch, const int32_t *patch_list, int n_list,
                         void *stream);

/* Standalone interpolate_state (refine.py:158-190) over a gathered coarse
 * array [M][cny][cnx] with availability mask; fine outputs [M][fny][fnx]. */
int mlamr_interpolate_box(int M, const double *ch, const double *chu, const double *chv,
                          const double *cb, const uint8_t *cavail,
                          int clo_i, int clo_j, int cnx, int cny,
                          int flo_i, int flo_j, int fnx, int fny,
                          const double *fb, int r_x, int r_y, mlamr_params prm,
                          double *oh, double *ohu, double *ohv, int32_t *status,
                          void *stream);

/* ---- K6: level reductions (driver.py:138-153, 286-297) ------------------
 * Per-(patch, block) uncovered-interior depth sums [P * blocks * M] (child
 * = coarsened owner map of the finer level in this level's index space, or
 * NULL) and a non-finite scan of interiors (`interior_state`) and frames
 * (`ghost_state`) that sets MLAMR_ST_NONFINITE. */
int mlamr_level_reduce(mlamr_level lv, const double *interior_state,
                       const double *ghost_state, const int32_t *child,
                       double *patch_mass, int blocks_per_patch,
                       int32_t *status, const int32_t *patch_list, int n_list,
                       void *stream);

/* As mlamr_level_reduce, for a level whose sibling ghost cells were never
 * copied because its step read them through the ghost plan (mlamr_step with
 * ghost_base/ghost_plan): frame cells with a plan entry >= 0 are checked at
 * that sibling cell of `ghost_state` -- the value the copy would have
 * written -- so the non-finite scan covers the same values as the
 * reference's isfinite over whole patch arrays (driver.py:286-297). */
int mlamr_level_reduce_planned(mlamr_level lv, const double *interior_state,
                               const double *ghost_state, const int32_t *child,
                               double *patch_mass, int blocks_per_patch,
                               int32_t *status, const int32_t *patch_list,
                               int n_list, const int64_t *ghost_base,
                               const int64_t *ghost_plan, void *stream);

/* Reference flag rule, per-cell part (regrid.flag_cells, regrid.py:58-101):
 * cell_bits over the level index space (no frame): bit0 amplitude flag
 * |eta_m - eta_rest_m| > wave_tol_m, bit(1+m) layer m wet, bit7 covered.
 * The dilations are applied by the host. */
int mlamr_flag_cells(mlamr_level lv, const double *state, mlamr_params prm,
                     const double *eta_rest, const double *wave_tol,
                     uint8_t *cell_bits, int blocks_per_patch,
                     const int32_t *patch_list, int n_list, void *stream);

/* Multi-GPU shadow exchange: copy whole patch blocks of `nplanes` planes
 * between a pool (plane stride = field_stride) and a packed buffer (plane
 * stride = packed length); segments = int64 [n][3] (src offset, dst
 * offset, length).  Patch lists (patch_list/n_list) above restrict a launch
 * to the patches a rank owns; NULL = every patch of the pool. */
/* Checkpoints: copy the interiors of every patch of a level (all 3M state
 * planes of `state`) to `packed` (unpack = 0) or back (unpack = 1).
 * packed is [3M][n_total], patch p's interior at pbase[p] (prefix sums of
 * nx*ny), rows x-fastest.  Replaces copying whole buffers in
 * Simulation.snapshot/restore: ghost frames and padding are refilled
 * before use (driver.py:175-190 fills every level first in its advance). */
int mlamr_pack_interiors(mlamr_level lv, double *state, double *packed,
                         const int64_t *pbase, int64_t n_total, int max_interior,
                         int unpack, void *stream);

int mlamr_copy_segments(const double *src, int64_t src_stride, double *dst, int64_t dst_stride,
                        const int64_t *segments, int n_segments, int max_len, int nplanes,
                        void *stream);

/* Harness Bernoulli flag rule on the device (C5):
 * flags = dilate^dilate_w(u < p) & covered & allowed and allowed =
 * erode(covered, 1), with u the splitmix64 counter hash of (seed,
 * stream_id, j, i) -- bit-identical to problems.hash_uniform -- and covered
 * read from the level's interior owner map `own` (frame-extended, >= 0 =
 * covered).  0/1 byte maps [ny][nx]; scratch is 3*ny*nx bytes. */
int mlamr_flags_bernoulli(const int32_t *own, int ny, int nx, unsigned long long seed,
                          unsigned long long stream_id, double p, int dilate_w, uint8_t *flags,
                          uint8_t *allowed, uint8_t *scratch, void *stream);

/* Harness gradient flag rule on the device (C1/C3): with
 * eta_m = (h_{M-1} + ... + h_m) + B of the layers in layer_mask on the
 * level grid (interior owner wins), a covered cell is flagged when
 * |eta difference| / spacing across a face shared with another covered
 * cell exceeds tol in any of those layers; then flags = dilate^dilate_w &
 * covered & allowed, allowed = erode(covered, 1).  0/1 byte maps
 * [ny][nx]; scratch 3*ny*nx bytes, eta_scratch popcount(layer_mask)*ny*nx
 * doubles. */
int mlamr_flags_gradient(mlamr_level lv, const double *state, mlamr_params prm, unsigned layer_mask,
                         double tol, int dilate_w, uint8_t *flags, uint8_t *allowed, uint8_t *scratch,
                         double *eta_scratch, void *stream);

/* The gradient rule for a sharded level, in two halves around the union
 * (uint8 MAX all-reduce) of the ranks' raw flags: _raw evaluates the rule
 * on the rank's local pool and keeps the owned cells' flags
 * (owned_patches: uint8 per local patch, NULL = all); _finish dilates the
 * union and masks it with the level's GLOBAL coverage (0/1 map) and its
 * one-cell erosion (allowed).  bits: ny*nx bytes; scratch: 3*ny*nx. */
int mlamr_flags_gradient_raw(mlamr_level lv, const double *state, mlamr_params prm, unsigned layer_mask,
                             double tol, const uint8_t *owned_patches, uint8_t *raw, uint8_t *bits,
                             double *eta_scratch, void *stream);
int mlamr_flags_finish(const uint8_t *raw, const uint8_t *covered, int ny, int nx, int dilate_w,
                       uint8_t *flags, uint8_t *allowed, uint8_t *scratch, void *stream);

/* Summed-area table for the clustering bisection (regrid.cluster_flags,
 * regrid.py:129-182): sat is int32 [(ny+1)*(nx+1)] with
 * sat[(j+1)*(nx+1)+(i+1)] = sum over [0,j]x[0,i] of map (invert=0) or
 * 1-map (invert=1), zero first row/column; scratch is int32
 * [ceil(ny/32)*nx].  Exact integer sums. */
int mlamr_sat_u8(const uint8_t *map, int ny, int nx, int invert, int32_t *sat, int32_t *scratch,
                 void *stream);

/* Sibling copies as a flat gather/scatter.  mlamr_copy_pairs_of_plan
 * writes, for every ghost cell of the listed patches (all when NULL), the
 * pair (destination, source) of element offsets, or (-1, src<0) when the
 * cell has no sibling source; list_base[k] is the first pair slot of list
 * entry k (prefix sum of its ghost counts).  mlamr_fill_copy_pairs then
 * copies the 3M planes for the n_pairs compacted pairs -- the sibling part
 * of the ghost fill (ghost.py:186-196) with one thread per cell. */
int mlamr_copy_pairs_of_plan(mlamr_level lv, const int64_t *gbase, const int64_t *plan,
                             const int32_t *patch_list, int n_list, const int64_t *list_base,
                             int max_ghost, int64_t *pairs, void *stream);
int mlamr_fill_copy_pairs(double *state, int64_t field_stride, const int64_t *pairs, int64_t n_pairs,
                          int num_layers, const int32_t *status, void *stream);

/* Frame records of one level (frames.frame_from_hierarchy + write_frame,
 * frames.py:72-100, 141-163): for each patch p (or each entry of
 * patch_list), writes at out + rec_off[p] (8-byte units) the five int64
 * (level_index, lo_i, lo_j, hi_i, hi_j) and the interior planes bathymetry,
 * h_0, hu_0, hv_0, h_1, ... (row-major, x fastest) -- the reference's binary
 * patch record, so the host writes header + one contiguous body. */
int mlamr_pack_frame(mlamr_level lv, const double *state, int level_index, const int64_t *rec_off,
                     const int32_t *patch_list, int n_list, int blocks_per_patch, double *out,
                     void *stream);

/* Full reference flag rule on the device (regrid.flag_cells +
 * nesting_allowed, regrid.py:58-101, 185-211): from mlamr_flag_cells' bits,
 * flags = dilate(amplitude | wet_m & dilate(dry_m)) & covered & allowed and
 * allowed = erode(covered, 1), as 0/1 byte maps [ny][nx]; scratch is 3*ny*nx
 * bytes. */
int mlamr_flags_reference(const uint8_t *bits, int ny, int nx, int M, int buffer_width,
                          uint8_t *flags, uint8_t *allowed, uint8_t *scratch, void *stream);

/* Self-test: counts quotients where the shared-reciprocal division used by
 * the kernels differs bitwise from div.rn.f64 (`bad`, must stay 0) and how
 * often its fast path declined (`slow`). */
int mlamr_selftest_div(const double *a, const double *b, int n, unsigned long long *bad,
                       unsigned long long *slow, void *stream);

/* Host-side (no GPU) recursive-bisection clustering of a flag map
 * (regrid.cluster_flags, regrid.py:129-182).  flags/allowed are HOST uint8
 * [ny][nx] (allowed may be NULL); writes (lo_i, lo_j, hi_i, hi_j) boxes
 * sorted by (lo_j, lo_i) into h_out_boxes.  Returns the box count, -1 if
 * more than max_boxes, -2 if a flag lies outside `allowed`. */
int mlamr_cluster_flags(const uint8_t *h_flags, int ny, int nx, double efficiency_target,
                        const uint8_t *h_allowed, int32_t *h_out_boxes, int max_boxes);

/* The same clustering from summed-area tables built on the device: HOST
 * int32 (ny+1) x (nx+1) tables of the flags and of the cells outside
 * `allowed` (h_sat_bad NULL = all allowed), zero first row/column. */
int mlamr_cluster_sat(const int32_t *h_sat_flags, const int32_t *h_sat_bad, int ny, int nx,
                      double efficiency_target, int32_t *h_out_boxes, int max_boxes);

/* Host-side max-patch-size chop of boxes (SURVEY.md App. B harness rule);
 * HOST int32 [n*4] in, HOST int32 [cap*4] out sorted by (lo_j, lo_i).
 * Returns the count or -1 when it exceeds cap. */
int mlamr_chop_boxes(const int32_t *h_boxes, int n, int max_nx, int max_ny, int aligned,
                     int32_t *h_out, int cap);

/* Host-side: out[k] = 1 when HOST box a[k] (int64 [na][4], inclusive)
 * intersects any box of b (multi-GPU shadow planning).  Returns 0, or -1
 * when the bucket grid would be too large. */
int mlamr_boxes_meet_any(const int64_t *h_a, int na, const int64_t *h_b, int nb, int bucket,
                         uint8_t *h_out);

#ifdef __cplusplus
}
#endif

#endif /* MLAMR_B200_H */
