// K2 ghost filling, K3/K5 regrid data movement, K4 coarsening, K6 level
// reductions, owner-map painting and the reference flag rule.
//
// All batched over every patch of a level in one launch.  Patch-to-patch
// relations (siblings, parents, old/new patches, fine/coarse overlaps) are
// resolved through int32 owner maps over each level's index space instead
// of the reference's O(P^2) box scans (ghost.py:186-196, regrid.py:311-323,
// coarsen.py:57-75); the painting order reproduces the reference's
// list-order precedence (interiors: last wins; ghost fallback: first wins).

#include <algorithm>

#include "interp.cuh"

namespace mlamr {

constexpr int NTA = 256;

// ---------------------------------------------------------------------------
// owner maps
// ---------------------------------------------------------------------------
__global__ void k_paint(int32_t *map, int map_nx, int map_ny, const int32_t *box, int grow,
                        int first_wins, int r_x, int r_y, int nrows) {
    const int p = grid_row();
    if (p >= nrows) return;
    const int32_t *b = box + 4 * p;
    int lo_i = b[0], lo_j = b[1], hi_i = b[2], hi_j = b[3];
    if (r_x > 1 || r_y > 1) {  // coarsened footprint (aligned boxes)
        lo_i = floordiv(lo_i, r_x);
        lo_j = floordiv(lo_j, r_y);
        hi_i = floordiv(hi_i + 1, r_x) - 1;
        hi_j = floordiv(hi_j + 1, r_y) - 1;
    }
    lo_i -= grow; lo_j -= grow; hi_i += grow; hi_j += grow;
    const int nx = hi_i - lo_i + 1, ny = hi_j - lo_j + 1;
    const int W = map_nx + 2 * MLAMR_G;
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < nx * ny; idx += gridDim.x * blockDim.x) {
        const int j = lo_j + idx / nx, i = lo_i + idx % nx;
        if (i < -MLAMR_G || j < -MLAMR_G || i >= map_nx + MLAMR_G || j >= map_ny + MLAMR_G) continue;
        int32_t *cell = map + (int64_t)(j + MLAMR_G) * W + (i + MLAMR_G);
        if (first_wins) {
            // map pre-set to -1: take the smallest index
            int cur = *cell;
            while (cur < 0 || p < cur) {
                const int prev = atomicCAS(cell, cur, p);
                if (prev == cur) break;
                cur = prev;
            }
        } else {
            atomicMax(cell, p);
        }
    }
}

// ---------------------------------------------------------------------------
// K2: ghost filling (ghost.fill_ghosts, ghost.py:156-197)
// ---------------------------------------------------------------------------
__device__ __forceinline__ void ghost_cell_of(int idx, int NX, int NY, int ny, int &J, int &I) {
    if (idx < 2 * NX) {  // bottom rows
        J = idx / NX;
        I = idx % NX;
    } else if (idx < 4 * NX) {  // top rows
        const int q = idx - 2 * NX;
        J = NY - 2 + q / NX;
        I = q % NX;
    } else {  // left/right columns on interior rows
        const int q = idx - 4 * NX;
        J = MLAMR_G + q / 4;
        const int s = q % 4;
        I = (s == 0) ? 0 : (s == 1) ? 1 : (s == 2) ? NX - 2 : NX - 1;
    }
}

// one side of the physical BCs (ghost._mirror_or_copy, ghost.py:89-106)
template <int M>
__device__ void bc_side(double *st, int64_t FS, int64_t off, int NX, int NY, int side, int kind,
                        double *bathy_only) {
    const int t = threadIdx.x;
    const bool xs = side < 2;
    const int n_lines = xs ? NY : NX;
    const int nq = (bathy_only != nullptr) ? 1 : 3 * M;
    // BU items per thread per round, all loads before the stores (sources
    // are interior cells, destinations ghost cells): a long level-1 side
    // was a chain of dependent load/store pairs
    constexpr int BU = 4;
    const int n_items = n_lines * 2 * nq;
    for (int base = t; base < n_items; base += NTA * BU) {
        double val[BU];
        double *dstp[BU];
#pragma unroll
        for (int u = 0; u < BU; ++u) {
            const int idx = base + u * NTA;
            dstp[u] = nullptr;
            if (idx >= n_items) continue;
        const int q = idx / (n_lines * 2);
        const int rem = idx - q * n_lines * 2;
        const int line = rem >> 1;
        const int k = rem & 1;
        double *a = (bathy_only != nullptr) ? bathy_only : st + q * FS;
        double sign = 1.0;
        if (bathy_only == nullptr) {
            const int fam = q / M;  // 0 h, 1 hu, 2 hv
            if (fam == 1 && xs) sign = -1.0;
            if (fam == 2 && !xs) sign = -1.0;
        }
        int dst_rc, src_rc;
        const int g = MLAMR_G;
        if (side == 0) {         // left: col g-1-k <- col g+k | col g
            dst_rc = g - 1 - k; src_rc = (kind == MLAMR_BC_WALL) ? g + k : g;
        } else if (side == 1) {  // right: col NX-g+k <- col NX-g-1-k | col NX-g-1
            dst_rc = NX - g + k; src_rc = (kind == MLAMR_BC_WALL) ? NX - g - 1 - k : NX - g - 1;
        } else if (side == 2) {  // bottom rows
            dst_rc = g - 1 - k; src_rc = (kind == MLAMR_BC_WALL) ? g + k : g;
        } else {                 // top rows
            dst_rc = NY - g + k; src_rc = (kind == MLAMR_BC_WALL) ? NY - g - 1 - k : NY - g - 1;
        }
        int64_t d, s;
        if (xs) {
            d = off + (int64_t)line * NX + dst_rc;
            s = off + (int64_t)line * NX + src_rc;
        } else {
            d = off + (int64_t)dst_rc * NX + line;
            s = off + (int64_t)src_rc * NX + line;
        }
        val[u] = (kind == MLAMR_BC_WALL) ? sign * a[s] : a[s];
        dstp[u] = a + d;
        }
#pragma unroll
        for (int u = 0; u < BU; ++u)
            if (dstp[u] != nullptr) *dstp[u] = val[u];
    }
}

template <int M>
__device__ void apply_bcs(const mlamr_level &lv, const PatchView &pv, const int4 bcs,
                          double *bathy_only) {
    // sides touching the level box, x sides first (ghost.py:109-121)
    const bool touch[4] = {pv.lo_i == 0, pv.lo_i + pv.nx == lv.level_nx, pv.lo_j == 0,
                           pv.lo_j + pv.ny == lv.level_ny};
    const int kinds[4] = {bcs.x, bcs.y, bcs.z, bcs.w};
#pragma unroll 1
    for (int side = 0; side < 4; ++side) {
        if (!touch[side]) continue;
        bc_side<M>(lv.state, lv.field_stride, pv.off, pv.NX, pv.NY, side, kinds[side], bathy_only);
        __syncthreads();
    }
}

template <int M>
__global__ void __launch_bounds__(NTA) k_fill_ghosts(mlamr_level lv, mlamr_level par, int has_parent,
                                                     const double *par_old, double theta, int r_x,
                                                     int r_y, int4 bcs, mlamr_params prm,
                                                     const int32_t *status, const int32_t *plist) {
    if (status != nullptr && *status != 0) return;
    const int p = plist ? plist[blockIdx.x] : (int)blockIdx.x;
    const PatchView pv = patch_view(lv, p);
    const int64_t FS = lv.field_stride;
    const double tol = prm.dry_tolerance;
    const int nghost = 4 * pv.NX + 4 * pv.ny;
    for (int idx = threadIdx.x; idx < nghost; idx += NTA) {
        int J, I;
        ghost_cell_of(idx, pv.NX, pv.NY, pv.ny, J, I);
        const int gi = pv.lo_i - MLAMR_G + I, gj = pv.lo_j - MLAMR_G + J;
        if (gi < 0 || gj < 0 || gi >= lv.level_nx || gj >= lv.level_ny) continue;
        const int64_t k = pv.off + (int64_t)J * pv.NX + I;
        const int sib = owner_at(lv.own, lv.level_nx, lv.level_ny, gi, gj);
        if (sib >= 0 && sib != p) {
            const int32_t *b = lv.box + 4 * sib;
            const int SNX = b[2] - b[0] + 1 + 2 * MLAMR_G;
            const int64_t ks = lv.offset[sib] + (int64_t)(gj - b[1] + MLAMR_G) * SNX + (gi - b[0] + MLAMR_G);
#pragma unroll
            for (int q = 0; q < 3 * M; ++q) lv.state[q * FS + k] = lv.state[q * FS + ks];
        } else if (has_parent) {
            const int pi = floordiv(gi, r_x), pj = floordiv(gj, r_y);
            Coarse5<M> c;
            gather5<M>(par, par.state, par_old, theta, true, pi, pj, c);
            Slopes<M> s;
            parent_slopes<M>(c, tol, s);
            double h[M], hu[M], hv[M];
            fine_cell<M>(s, child_offset(gi, pi, r_x), child_offset(gj, pj, r_y), lv.bathy[k], tol, h, hu, hv);
#pragma unroll
            for (int m = 0; m < M; ++m) {
                lv.state[m * FS + k] = h[m];
                lv.state[(M + m) * FS + k] = hu[m];
                lv.state[(2 * M + m) * FS + k] = hv[m];
            }
        }
    }
    __syncthreads();
    apply_bcs<M>(lv, pv, bcs, nullptr);
}

// ---------------------------------------------------------------------------
// K2 split into a per-layout plan and three lean kernels.
// Ghost cells of patch p are enumerated 0..nghost(p)-1 exactly as
// ghost_cell_of(); gbase[p] is the prefix sum of nghost over the pool.
// plan[gbase[p] + idx] = element offset of the sibling cell that covers it
// (interior owner, ghost.py:186-196), -1 = in-domain but no sibling
// (coarse interpolation, ghost.py:167-185), -2 = outside the level box
// (physical BC, ghost.py:132-142).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(NTA) k_ghost_plan(mlamr_level lv, const int64_t *gbase, int64_t *plan) {
    const int p = grid_row();
    if (p >= lv.num_patches) return;
    const PatchView pv = patch_view(lv, p);
    const int nghost = 4 * pv.NX + 4 * pv.ny;
    for (int idx = blockIdx.x * NTA + threadIdx.x; idx < nghost; idx += gridDim.x * NTA) {
        int J, I;
        ghost_cell_of(idx, pv.NX, pv.NY, pv.ny, J, I);
        const int gi = pv.lo_i - MLAMR_G + I, gj = pv.lo_j - MLAMR_G + J;
        int64_t v;
        if (gi < 0 || gj < 0 || gi >= lv.level_nx || gj >= lv.level_ny) {
            v = -2;
        } else {
            const int sib = owner_at(lv.own, lv.level_nx, lv.level_ny, gi, gj);
            if (sib >= 0 && sib != p) {
                const int32_t *b = lv.box + 4 * sib;
                const int SNX = b[2] - b[0] + 1 + 2 * MLAMR_G;
                v = lv.offset[sib] + (int64_t)(gj - b[1] + MLAMR_G) * SNX + (gi - b[0] + MLAMR_G);
            } else {
                v = -1;
            }
        }
        plan[gbase[p] + idx] = v;
    }
}

// Compacted list of the plan's interpolated cells (-1 entries): int32 pairs
// (patch, ghost idx), appended with warp-aggregated atomics, the count in
// *count.  The order is not deterministic, and need not be: every listed
// cell is interpolated independently into its own location.  Keeps the
// compaction on the device (no host round trip for the count).
__global__ void __launch_bounds__(NTA) k_plan_interp_cells(mlamr_level lv, const int64_t *gbase,
                                                           const int64_t *plan, const int32_t *patch_list,
                                                           int n_rows, int32_t *cells, int32_t *count) {
    const int row = grid_row();
    if (row >= n_rows) return;
    const int p = patch_list ? patch_list[row] : row;
    const int32_t *b = lv.box + 4 * p;
    const int nghost = 4 * (b[2] - b[0] + 1 + 2 * MLAMR_G) + 4 * (b[3] - b[1] + 1);
    const int lane = threadIdx.x & 31;
    for (int base = blockIdx.x * NTA; base < nghost; base += gridDim.x * NTA) {
        const int idx = base + threadIdx.x;
        const bool want = idx < nghost && plan[gbase[p] + idx] == -1;
        const unsigned mask = __ballot_sync(0xffffffffu, want);
        if (mask == 0u) continue;
        const int leader = __ffs(mask) - 1;
        int pos = 0;
        if (lane == leader) pos = atomicAdd(count, __popc(mask));
        pos = __shfl_sync(0xffffffffu, pos, leader) + __popc(mask & ((1u << lane) - 1u));
        if (want) {
            cells[2 * pos] = p;
            cells[2 * pos + 1] = idx;
        }
    }
}

// sibling copies (ghost.py:186-196): one CTA of NTC threads per patch.  A
// thread moves ghost cells in PAIRS -- consecutive plan entries are
// neighbouring cells of a frame row (or the two cells of a side band on one
// row), and their sibling sources are neighbours in the sibling's interior
// -- so an aligned pair is one 16-byte load and store per plane.  Each
// thread takes two pairs per round and issues all plan loads, then all
// source loads, then the stores: the kernel is latency-bound (a plan load,
// then the dependent data loads), so independent pairs in flight are what
// reaches the bandwidth.
constexpr int NTC = 128;

// ghost index of an even idx -> (J, I) of the pair's first cell and whether
// the second cell is its right neighbour in memory (ghost_cell_of order)
__device__ __forceinline__ bool ghost_pair_of(int idx, int NX, int NY, int &J, int &I) {
    if (idx < 4 * NX) {  // bottom rows, then top rows
        const int q = idx < 2 * NX ? idx : idx - 2 * NX;
        const int r = q / NX;
        J = idx < 2 * NX ? r : NY - 2 + r;
        I = q - r * NX;
        return I + 1 < NX;
    }
    const int q = idx - 4 * NX;  // side bands: (0, 1) then (NX-2, NX-1) per row
    J = MLAMR_G + (q >> 2);
    I = (q & 2) ? NX - 2 : 0;
    return true;
}

template <int M>
__global__ void __launch_bounds__(NTC) k_fill_copy(mlamr_level lv, const int64_t *gbase, const int64_t *plan,
                                                   const int32_t *plist, const int32_t *status) {
    if (status != nullptr && *status != 0) return;
    const int p = plist ? plist[blockIdx.x] : (int)blockIdx.x;
    const int32_t *b = lv.box + 4 * p;
    const int NX = b[2] - b[0] + 1 + 2 * MLAMR_G, ny = b[3] - b[1] + 1, NY = ny + 2 * MLAMR_G;
    const int npair = 2 * NX + 2 * ny;  // nghost / 2 (nghost = 4 NX + 4 ny)
    const int64_t FS = lv.field_stride;
    const int64_t off = lv.offset[p];
    const int64_t *pl = plan + gbase[p];
    double *st = lv.state;
    for (int q0 = threadIdx.x; q0 < npair; q0 += 2 * NTC) {
        int64_t src[2][2], dst[2][2];
        bool vec[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int q = q0 + u * NTC;
            const bool in = q < npair;
            const int idx = 2 * (in ? q : q0);
            src[u][0] = in ? pl[idx] : -1;
            src[u][1] = in ? pl[idx + 1] : -1;
            int J, I;
            const bool adj = ghost_pair_of(idx, NX, NY, J, I);
            dst[u][0] = off + (int64_t)J * NX + I;
            if (adj) {
                dst[u][1] = dst[u][0] + 1;
            } else {
                int J1, I1;
                ghost_cell_of(idx + 1, NX, NY, ny, J1, I1);
                dst[u][1] = off + (int64_t)J1 * NX + I1;
            }
            vec[u] = adj && src[u][0] >= 0 && src[u][1] == src[u][0] + 1 && ((dst[u][0] | src[u][0]) & 1) == 0;
        }
        double2 v[2][3 * M];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
#pragma unroll
            for (int k = 0; k < 3 * M; ++k) {
                if (vec[u]) {
                    v[u][k] = *reinterpret_cast<const double2 *>(st + k * FS + src[u][0]);
                } else {
                    v[u][k].x = src[u][0] >= 0 ? st[k * FS + src[u][0]] : 0.0;
                    v[u][k].y = src[u][1] >= 0 ? st[k * FS + src[u][1]] : 0.0;
                }
            }
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
#pragma unroll
            for (int k = 0; k < 3 * M; ++k) {
                if (vec[u]) {
                    *reinterpret_cast<double2 *>(st + k * FS + dst[u][0]) = v[u][k];
                } else {
                    if (src[u][0] >= 0) st[k * FS + dst[u][0]] = v[u][k].x;
                    if (src[u][1] >= 0) st[k * FS + dst[u][1]] = v[u][k].y;
                }
            }
        }
    }
}

// sibling copies from a flat list of (destination, source) element offsets
// built from the plan (every ghost cell with a sibling source, owned
// patches only): a pure gather/scatter over all patches of the level, with
// no per-patch blocks left idle by small patches (C5's 16x16 patches have
// 144 ghost cells per 256-thread block in the per-patch kernel).
template <int M>
__global__ void __launch_bounds__(NTA) k_fill_copy_pairs(double *__restrict__ state, int64_t FS,
                                                         const int64_t *__restrict__ pairs, int64_t n,
                                                         const int32_t *status) {
    if (status != nullptr && *status != 0) return;
    for (int64_t c = blockIdx.x * (int64_t)NTA + threadIdx.x; c < n; c += (int64_t)gridDim.x * NTA) {
        const int64_t dst = pairs[2 * c], src = pairs[2 * c + 1];
        double v[3 * M];
#pragma unroll
        for (int q = 0; q < 3 * M; ++q) v[q] = state[q * FS + src];
#pragma unroll
        for (int q = 0; q < 3 * M; ++q) state[q * FS + dst] = v[q];
    }
}

// the (destination, source) pairs of a plan: one thread per ghost cell of
// the listed patches writes its pair, or (-1, -1) when it has no sibling
__global__ void __launch_bounds__(NTA) k_copy_pairs_of_plan(mlamr_level lv, const int64_t *gbase,
                                                            const int64_t *plan, const int32_t *plist,
                                                            const int64_t *pbase, int64_t *pairs, int nrows) {
    const int row = grid_row();
    if (row >= nrows) return;
    const int p = plist ? plist[row] : row;
    const PatchView pv = patch_view(lv, p);
    const int nghost = 4 * pv.NX + 4 * pv.ny;
    const int64_t out0 = pbase[row];
    for (int idx = blockIdx.x * NTA + threadIdx.x; idx < nghost; idx += gridDim.x * NTA) {
        const int64_t src = plan[gbase[p] + idx];
        int J, I;
        ghost_cell_of(idx, pv.NX, pv.NY, pv.ny, J, I);
        const int64_t dst = pv.off + (int64_t)J * pv.NX + I;
        pairs[2 * (out0 + idx)] = src >= 0 ? dst : -1;
        pairs[2 * (out0 + idx) + 1] = src;
    }
}

// coarse interpolation of the cells of a compacted list (patch, ghost idx)
#ifndef MLAMR_INTERP_MINB
#define MLAMR_INTERP_MINB 1
#endif
template <int M>
__global__ void __launch_bounds__(NTA, MLAMR_INTERP_MINB) k_fill_interp(mlamr_level lv, mlamr_level par, const double *par_old,
                                                     double theta, int r_x, int r_y, const int32_t *cells,
                                                     int n_cells, const int32_t *n_cells_dev, mlamr_params prm,
                                                     const int32_t *status) {
    if (status != nullptr && *status != 0) return;
    if (n_cells_dev != nullptr) n_cells = min(n_cells, *n_cells_dev);
    const double tol = prm.dry_tolerance;
    const int64_t FS = lv.field_stride;
    for (int c = blockIdx.x * NTA + threadIdx.x; c < n_cells; c += gridDim.x * NTA) {
        const int p = cells[2 * c], idx = cells[2 * c + 1];
        const int32_t *b = lv.box + 4 * p;
        const int NX = b[2] - b[0] + 1 + 2 * MLAMR_G, ny = b[3] - b[1] + 1;
        int J, I;
        ghost_cell_of(idx, NX, ny + 2 * MLAMR_G, ny, J, I);
        const int gi = b[0] - MLAMR_G + I, gj = b[1] - MLAMR_G + J;
        const int64_t k = lv.offset[p] + (int64_t)J * NX + I;
        const int pi = floordiv(gi, r_x), pj = floordiv(gj, r_y);
        Coarse5<M> cc;
        gather5<M>(par, par.state, par_old, theta, true, pi, pj, cc);
        Slopes<M> sl;
        parent_slopes<M>(cc, tol, sl);
        double h[M], hu[M], hv[M];
        fine_cell<M>(sl, child_offset(gi, pi, r_x), child_offset(gj, pj, r_y), lv.bathy[k], tol, h, hu, hv);
#pragma unroll
        for (int m = 0; m < M; ++m) {
            lv.state[m * FS + k] = h[m];
            lv.state[(M + m) * FS + k] = hu[m];
            lv.state[(2 * M + m) * FS + k] = hv[m];
        }
    }
}

// physical BCs of the patches touching the level box (block per patch)
template <int M>
__global__ void __launch_bounds__(NTA) k_fill_bc(mlamr_level lv, const int32_t *plist, int4 bcs,
                                                 const int32_t *status) {
    if (status != nullptr && *status != 0) return;
    const int p = plist[blockIdx.x];
    const PatchView pv = patch_view(lv, p);
    apply_bcs<M>(lv, pv, bcs, nullptr);
}

__global__ void __launch_bounds__(NTA) k_fill_bathy(mlamr_level lv, const double *level_bathy, int4 bcs) {
    const int p = blockIdx.x;
    const PatchView pv = patch_view(lv, p);
    for (int idx = threadIdx.x; idx < pv.NX * pv.NY; idx += NTA) {
        const int J = idx / pv.NX, I = idx % pv.NX;
        const int gi = pv.lo_i - MLAMR_G + I, gj = pv.lo_j - MLAMR_G + J;
        double v = 0.0;
        if (gi >= 0 && gj >= 0 && gi < lv.level_nx && gj < lv.level_ny)
            v = level_bathy[(int64_t)gj * lv.level_nx + gi];
        lv.bathy[pv.off + idx] = v;
    }
    __syncthreads();
    apply_bcs<1>(lv, pv, bcs, lv.bathy);
}

// ---------------------------------------------------------------------------
// K4: coarsening (coarsen.average_down, coarsen.py:30-76)
// One thread per coarse cell of a fine patch's footprint.
// ---------------------------------------------------------------------------
// RX/RY > 0: compile-time ratios (fully unrolled, all loads in flight);
// 0: runtime ratios.  Same summation order either way (coarsen.py:21-27).
// One coarse cell of average_down: block-mean the fine children of coarse
// cell (clo_i + I, clo_j + J) into the coarse owner's interior (if any) and
// accumulate the mass change into dsum.
// numpy's pairwise_sum over n contiguous doubles (numpy/_core/src/umath/
// loops_utils.h.src), n <= 128: sequential from 0.0 below 8 elements, else
// eight running accumulators, ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), then a
// sequential tail.  block_mean of a patch ONE coarse cell wide sums its
// r_y x r_x block this way (numpy coalesces the two reduced axes into one
// contiguous run); wider patches use the per-row-then-rows order.
__device__ __forceinline__ double np_pairwise(const double *a, int n) {
    if (n < 8) {
        double res = 0.0;
        for (int i = 0; i < n; ++i) res = res + a[i];
        return res;
    }
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int i = 8;
    for (; i < n - (n % 8); i += 8)
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = r[j] + a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res = res + a[i];
    return res;
}

template <int M, int RX, int RY>
__device__ __forceinline__ void avg_cell(const mlamr_level &fine, const mlamr_level &coarse, const PatchView &fv,
                                         int r_x, int r_y, int cnx, int clo_i, int clo_j, int idx, double tol,
                                         double nblk, bool vec2, double (&dsum)[M]) {
    const int64_t FF = fine.field_stride, CF = coarse.field_stride;
    do {
        const int J = idx / cnx, I = idx - (idx / cnx) * cnx;
        const int ci = clo_i + I, cj = clo_j + J;
        const int o = owner_at(coarse.own, coarse.level_nx, coarse.level_ny, ci, cj);
        if (o < 0) break;
        const int64_t base = fv.off + (int64_t)(MLAMR_G + J * r_y) * fv.NX + (MLAMR_G + I * r_x);
        double avg[3][M];
#pragma unroll
        for (int f = 0; f < 3; ++f)
#pragma unroll
            for (int m = 0; m < M; ++m) {
                const double *a = fine.state + (f * M + m) * FF + base;
                double s = 0.0;
                if (RX > 0 && RY > 0) {
                    double v[RY > 0 ? RY : 1][RX > 0 ? RX : 1];
                    if (RX % 2 == 0 && vec2) {
                        // even ratios: fine rows of a refined box start on
                        // even elements of 256-element aligned patches, so a
                        // block row is RX/2 aligned 16-byte loads
#pragma unroll
                        for (int q = 0; q < (RY > 0 ? RY : 1); ++q)
#pragma unroll
                            for (int pp = 0; pp < (RX > 0 ? RX : 1); pp += 2) {
                                const double2 w = *reinterpret_cast<const double2 *>(a + (int64_t)q * fv.NX + pp);
                                v[q][pp] = w.x;
                                v[q][pp + 1] = w.y;
                            }
                    } else {
#pragma unroll
                        for (int q = 0; q < (RY > 0 ? RY : 1); ++q)
#pragma unroll
                            for (int pp = 0; pp < (RX > 0 ? RX : 1); ++pp) v[q][pp] = a[(int64_t)q * fv.NX + pp];
                    }
                    if (cnx == 1) {
                        s = np_pairwise(&v[0][0], (RY > 0 ? RY : 1) * (RX > 0 ? RX : 1));
                    } else {
#pragma unroll
                        for (int q = 0; q < (RY > 0 ? RY : 1); ++q) {
                            double rs = v[q][0];
#pragma unroll
                            for (int pp = 1; pp < (RX > 0 ? RX : 1); ++pp) rs = rs + v[q][pp];
                            s = (q == 0) ? rs : s + rs;
                        }
                    }
                } else if (cnx == 1 && r_x * r_y <= 64) {
                    double blk[64];
                    for (int q = 0; q < r_y; ++q)
                        for (int pp = 0; pp < r_x; ++pp) blk[q * r_x + pp] = a[(int64_t)q * fv.NX + pp];
                    s = np_pairwise(blk, r_x * r_y);
                } else {
                    for (int q = 0; q < r_y; ++q) {
                        const double *row = a + (int64_t)q * fv.NX;
                        double rs = row[0];
                        for (int pp = 1; pp < r_x; ++pp) rs = rs + row[pp];
                        s = (q == 0) ? rs : s + rs;
                    }
                }
                avg[f][m] = s / nblk;
            }
        const int32_t *b = coarse.box + 4 * o;
        const int CNX = b[2] - b[0] + 1 + 2 * MLAMR_G;
        const int64_t kc = coarse.offset[o] + (int64_t)(cj - b[1] + MLAMR_G) * CNX + (ci - b[0] + MLAMR_G);
#pragma unroll
        for (int m = 0; m < M; ++m) {
            if (avg[0][m] <= tol) {
                avg[1][m] = 0.0;
                avg[2][m] = 0.0;
            }
            dsum[m] = dsum[m] + (avg[0][m] - coarse.state[m * CF + kc]);
            coarse.state[m * CF + kc] = avg[0][m];
            coarse.state[(M + m) * CF + kc] = avg[1][m];
            coarse.state[(2 * M + m) * CF + kc] = avg[2][m];
        }
    } while (false);
}

template <int M, int RX, int RY>
__global__ void __launch_bounds__(NTA) k_average_down(mlamr_level fine, mlamr_level coarse, int r_x_, int r_y_,
                                                      mlamr_params prm, double *patch_delta,
                                                      const int32_t *status) {
    __shared__ double red[NTA];
    if (status != nullptr && *status != 0) return;
    const int r_x = RX > 0 ? RX : r_x_;
    const int r_y = RY > 0 ? RY : r_y_;
    const int p = grid_row();
    if (p >= fine.num_patches) return;
    const PatchView fv = patch_view(fine, p);
    const int cnx = fv.nx / r_x, cny = fv.ny / r_y;
    const int clo_i = floordiv(fv.lo_i, r_x), clo_j = floordiv(fv.lo_j, r_y);
    const double tol = prm.dry_tolerance;
    const double nblk = (double)(r_x * r_y);
    const bool vec2 = !((fv.NX | fv.off | fine.field_stride) & 1);
    double dsum[M];
#pragma unroll
    for (int m = 0; m < M; ++m) dsum[m] = 0.0;
    for (int idx = blockIdx.x * NTA + threadIdx.x; idx < cnx * cny; idx += gridDim.x * NTA)
        avg_cell<M, RX, RY>(fine, coarse, fv, r_x, r_y, cnx, clo_i, clo_j, idx, tol, nblk, vec2, dsum);
#pragma unroll
    for (int m = 0; m < M; ++m) {
        const double s = block_sum<NTA>(dsum[m], red);
        if (threadIdx.x == 0) patch_delta[((int64_t)p * gridDim.x + blockIdx.x) * M + m] = s;
    }
}

// average_down over a flat list of all coarse cells of the fine level
// (cbase[p] = first coarse cell of fine patch p, prefix sums), without the
// per-patch mass-change partials (the driver does not use them,
// driver.py:280): small patches (C5's 16x16 fine patches have 32 coarse
// cells) no longer leave most of a per-patch block idle.
template <int M, int RX, int RY>
__global__ void __launch_bounds__(NTA) k_average_down_flat(mlamr_level fine, mlamr_level coarse, int r_x_,
                                                           int r_y_, mlamr_params prm, const int64_t *cbase,
                                                           int64_t n_coarse, const int32_t *status) {
    __shared__ int first_patch;
    if (status != nullptr && *status != 0) return;
    const int r_x = RX > 0 ? RX : r_x_;
    const int r_y = RY > 0 ? RY : r_y_;
    const double tol = prm.dry_tolerance;
    const double nblk = (double)(r_x * r_y);
    double dsum[M];
#pragma unroll
    for (int m = 0; m < M; ++m) dsum[m] = 0.0;
    for (int64_t c0 = (int64_t)blockIdx.x * NTA; c0 < n_coarse; c0 += (int64_t)gridDim.x * NTA) {
        __syncthreads();
        if (threadIdx.x == 0) {  // patch of the block's first cell: last p with cbase[p] <= c0
            int lo = 0, hi = fine.num_patches - 1;
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (cbase[mid] <= c0) lo = mid; else hi = mid - 1;
            }
            first_patch = lo;
        }
        __syncthreads();
        const int64_t c = c0 + threadIdx.x;
        if (c >= n_coarse) continue;
        int p = first_patch;
        while (p + 1 < fine.num_patches && cbase[p + 1] <= c) ++p;
        const PatchView fv = patch_view(fine, p);
        const int cnx = fv.nx / r_x;
        const int clo_i = floordiv(fv.lo_i, r_x), clo_j = floordiv(fv.lo_j, r_y);
        const bool vec2 = !((fv.NX | fv.off | fine.field_stride) & 1);
        avg_cell<M, RX, RY>(fine, coarse, fv, r_x, r_y, cnx, clo_i, clo_j, (int)(c - cbase[p]), tol, nblk, vec2,
                            dsum);
    }
}

// check_bathymetry_consistency (coarsen.py:79-100): one thread per coarse
// cell under a new fine patch (flat list, as k_average_down_flat); the fine
// block mean in the reference's numpy order against the coarse interior
// value, atol absolute.
__global__ void __launch_bounds__(NTA) k_check_bathy(mlamr_level fine, mlamr_level coarse, int r_x, int r_y,
                                                     double atol, const int64_t *__restrict__ cbase,
                                                     int64_t n_coarse, int32_t *status, int32_t *bad) {
    const double nblk = (double)(r_x * r_y);
    for (int64_t c = (int64_t)blockIdx.x * NTA + threadIdx.x; c < n_coarse; c += (int64_t)gridDim.x * NTA) {
        int lo = 0, hi = fine.num_patches - 1;   // last p with cbase[p] <= c
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (cbase[mid] <= c) lo = mid; else hi = mid - 1;
        }
        const int p = lo;
        const PatchView fv = patch_view(fine, p);
        const int cnx = fv.nx / r_x;
        const int idx = (int)(c - cbase[p]);
        const int J = idx / cnx, I = idx - (idx / cnx) * cnx;
        const int ci = floordiv(fv.lo_i, r_x) + I, cj = floordiv(fv.lo_j, r_y) + J;
        const int o = owner_at(coarse.own, coarse.level_nx, coarse.level_ny, ci, cj);
        if (o < 0) continue;
        const double *a = fine.bathy + fv.off + (int64_t)(MLAMR_G + J * r_y) * fv.NX + (MLAMR_G + I * r_x);
        double s = 0.0;
        if (cnx == 1 && r_x * r_y <= 64) {   // numpy's coalesced block (np_pairwise)
            double blk[64];
            for (int q = 0; q < r_y; ++q)
                for (int pp = 0; pp < r_x; ++pp) blk[q * r_x + pp] = a[(int64_t)q * fv.NX + pp];
            s = np_pairwise(blk, r_x * r_y);
        } else {
            for (int q = 0; q < r_y; ++q) {
                double rs = a[(int64_t)q * fv.NX];
                for (int pp = 1; pp < r_x; ++pp) rs = rs + a[(int64_t)q * fv.NX + pp];
                s = (q == 0) ? rs : s + rs;
            }
        }
        const double mean = s / nblk;
        const int32_t *b = coarse.box + 4 * o;
        const int CNX = b[2] - b[0] + 1 + 2 * MLAMR_G;
        const double cv = coarse.bathy[coarse.offset[o] + (int64_t)(cj - b[1] + MLAMR_G) * CNX + (ci - b[0] + MLAMR_G)];
        if (fabs(mean - cv) > atol) {
            atomicOr(status, MLAMR_ST_BATHY);
            atomicMin(bad, p);
        }
    }
}

// ---------------------------------------------------------------------------
// K3 + K5: regrid data movement (regrid.rebuild_child_level, regrid.py:270-353)
// One thread per coarse cell of a new patch's footprint: either copy its
// r_x*r_y children from the old patch covering them, or refine them from
// the parent's interiors (gather include_ghosts=False, regrid.py:295-300).
// ---------------------------------------------------------------------------
// 3 CTAs/SM (<= 80 registers): the copy pass -- most of a rebuild -- is
// latency-bound on its owner-map -> source chain and wants the warps; the
// rarer refine pass spills a little (C4 level-3 rebuild 1.24 -> 1.08 ms)
#ifndef MLAMR_RG_MINB
#define MLAMR_RG_MINB 3
#endif
template <int M, int NTR = NTA>
__global__ void __launch_bounds__(NTR, NTR == NTA ? MLAMR_RG_MINB : 1) k_regrid_fill(mlamr_level nl, mlamr_level ol, mlamr_level par,
                                                     int r_x, int r_y, mlamr_params prm,
                                                     double *refine_delta, int32_t *status, const int32_t *plist,
                                                     int nrows) {
    __shared__ double red[NTR];
    const int row = grid_row();
    if (row >= nrows) return;
    const int p = plist ? plist[row] : row;
    const PatchView nv = patch_view(nl, p);
    const int cnx = nv.nx / r_x, cny = nv.ny / r_y;
    const int clo_i = floordiv(nv.lo_i, r_x), clo_j = floordiv(nv.lo_j, r_y);
    const int64_t NF = nl.field_stride, OF = ol.field_stride;
    const double tol = prm.dry_tolerance;
    const double af = nl.dx * nl.dy, ac = par.dx * par.dy;
    double dsum[M];
#pragma unroll
    for (int m = 0; m < M; ++m) dsum[m] = 0.0;
    // old-patch copies (regrid.py:311-323) one fine cell per thread, so a
    // warp moves contiguous row segments; old patches are ratio-aligned, so
    // a coarse cell's fine block lies in one old patch and the owner of the
    // fine cell is the owner the refine pass below tests.  RG cells per
    // thread per round, each stage (owner lookups, source loads, stores)
    // issued for all of them before the next: the copy is a chain of
    // dependent loads (owner map -> old patch box/offset -> state), and
    // independent cells in flight are what reaches the bandwidth.
    constexpr int RG = 4;
    const int ncell = nv.nx * nv.ny;
    const int stride = gridDim.x * NTR;
    // A new patch whose box is an old patch's box (most of a level away from
    // the moving front) is that patch: its interior rows, side frame columns
    // included, are one contiguous range per plane in both layouts, copied
    // flat -- no owner lookups, no row split.  (The frame columns are
    // refilled before anything reads them.)
    {
        const int o0 = owner_at(ol.own, ol.level_nx, ol.level_ny, nv.lo_i, nv.lo_j);
        bool same = false;
        if (o0 >= 0) {
            const int32_t *b = ol.box + 4 * o0;
            same = b[0] == nv.lo_i && b[1] == nv.lo_j && b[2] - b[0] + 1 == nv.nx && b[3] - b[1] + 1 == nv.ny;
        }
        if (same) {
            const int64_t so = ol.offset[o0] + (int64_t)MLAMR_G * nv.NX, dof = nv.off + (int64_t)MLAMR_G * nv.NX;
            const int n = nv.ny * nv.NX;
            for (int base = blockIdx.x * NTR + threadIdx.x; base < n; base += RG * stride) {
                double v[RG][3 * M];
#pragma unroll
                for (int u = 0; u < RG; ++u)
                    if (base + u * stride < n)
#pragma unroll
                        for (int f = 0; f < 3 * M; ++f) v[u][f] = ol.state[f * OF + so + base + u * stride];
#pragma unroll
                for (int u = 0; u < RG; ++u)
                    if (base + u * stride < n)
#pragma unroll
                        for (int f = 0; f < 3 * M; ++f) nl.state[f * NF + dof + base + u * stride] = v[u][f];
            }
            // nothing refined: the patch's refine delta is zero
            if (threadIdx.x == 0)
#pragma unroll
                for (int m = 0; m < M; ++m) refine_delta[((int64_t)p * gridDim.x + blockIdx.x) * M + m] = 0.0;
            return;
        }
    }
    for (int base = blockIdx.x * NTR + threadIdx.x; base < ncell; base += RG * stride) {
        int64_t ks[RG], kd[RG];
#pragma unroll
        for (int u = 0; u < RG; ++u) {
            const int idx = base + u * stride;
            ks[u] = -1;
            kd[u] = 0;
            if (idx >= ncell) continue;
            const int j = idx / nv.nx, i = idx - (idx / nv.nx) * nv.nx;
            const int fi = nv.lo_i + i, fj = nv.lo_j + j;
            const int o = owner_at(ol.own, ol.level_nx, ol.level_ny, fi, fj);
            if (o < 0) continue;
            const int32_t *b = ol.box + 4 * o;
            const int ONX = b[2] - b[0] + 1 + 2 * MLAMR_G;
            ks[u] = ol.offset[o] + (int64_t)(fj - b[1] + MLAMR_G) * ONX + (fi - b[0] + MLAMR_G);
            kd[u] = nv.off + (int64_t)(j + MLAMR_G) * nv.NX + (i + MLAMR_G);
        }
        double v[RG][3 * M];
#pragma unroll
        for (int u = 0; u < RG; ++u)
            if (ks[u] >= 0)
#pragma unroll
                for (int f = 0; f < 3 * M; ++f) v[u][f] = ol.state[f * OF + ks[u]];
#pragma unroll
        for (int u = 0; u < RG; ++u)
            if (ks[u] >= 0)
#pragma unroll
                for (int f = 0; f < 3 * M; ++f) nl.state[f * NF + kd[u]] = v[u][f];
    }
    for (int idx = blockIdx.x * NTR + threadIdx.x; idx < cnx * cny; idx += gridDim.x * NTR) {
        const int J = idx / cnx, I = idx % cnx;
        const int ci = clo_i + I, cj = clo_j + J;
        const int fi0 = ci * r_x, fj0 = cj * r_y;
        const int o = owner_at(ol.own, ol.level_nx, ol.level_ny, fi0, fj0);
        if (o >= 0) continue;   // copied above
        Coarse5<M> c;
        gather5<M>(par, par.state, nullptr, 0.0, false, ci, cj, c);
        if (!c.avail[0]) {  // coarse data under the region is incomplete (refine.py:222-225)
            atomicOr(status, MLAMR_ST_GEOMETRY);
            continue;
        }
        Slopes<M> s;
        parent_slopes<M>(c, tol, s);
        double fine_sum[M];
#pragma unroll
        for (int m = 0; m < M; ++m) fine_sum[m] = 0.0;
        for (int q = 0; q < r_y; ++q)
            for (int pp = 0; pp < r_x; ++pp) {
                const int fi = fi0 + pp, fj = fj0 + q;
                const int64_t kd = nv.off + (int64_t)(fj - nv.lo_j + MLAMR_G) * nv.NX + (fi - nv.lo_i + MLAMR_G);
                double h[M], hu[M], hv[M];
                fine_cell<M>(s, child_offset(fi, ci, r_x), child_offset(fj, cj, r_y), nl.bathy[kd], tol, h, hu, hv);
#pragma unroll
                for (int m = 0; m < M; ++m) {
                    nl.state[m * NF + kd] = h[m];
                    nl.state[(M + m) * NF + kd] = hu[m];
                    nl.state[(2 * M + m) * NF + kd] = hv[m];
                    fine_sum[m] = fine_sum[m] + h[m];
                }
            }
#pragma unroll
        for (int m = 0; m < M; ++m) dsum[m] = dsum[m] + ((fine_sum[m] * af) - (c.h[0][m] * ac));
    }
#pragma unroll
    for (int m = 0; m < M; ++m) {
        const double s = block_sum<NTR>(dsum[m], red);
        if (threadIdx.x == 0) refine_delta[((int64_t)p * gridDim.x + blockIdx.x) * M + m] = s;
    }
}

// derefine delta (regrid.py:329-348): coarse cells covered by an old patch
// but by no new one: coarse mass minus the discarded fine mass.
template <int M, int NTR = NTA>
__global__ void __launch_bounds__(NTR) k_derefine(mlamr_level ol, mlamr_level par, const int32_t *new_child,
                                                  int r_x, int r_y, double *delta, const int32_t *plist,
                                                  int nrows) {
    __shared__ double red[NTR];
    const int row = grid_row();
    if (row >= nrows) return;
    const int p = plist ? plist[row] : row;
    const PatchView ov = patch_view(ol, p);
    const int cnx = ov.nx / r_x, cny = ov.ny / r_y;
    const int clo_i = floordiv(ov.lo_i, r_x), clo_j = floordiv(ov.lo_j, r_y);
    const int64_t OF = ol.field_stride, PF = par.field_stride;
    const double af = ol.dx * ol.dy, ac = par.dx * par.dy;
    double dsum[M];
#pragma unroll
    for (int m = 0; m < M; ++m) dsum[m] = 0.0;
    for (int idx = blockIdx.x * NTR + threadIdx.x; idx < cnx * cny; idx += gridDim.x * NTR) {
        const int J = idx / cnx, I = idx % cnx;
        const int ci = clo_i + I, cj = clo_j + J;
        if (owner_at(new_child, par.level_nx, par.level_ny, ci, cj) >= 0) continue;
        const int o = owner_at(par.own, par.level_nx, par.level_ny, ci, cj);
#pragma unroll
        for (int m = 0; m < M; ++m) {
            double fs = 0.0;
            for (int q = 0; q < r_y; ++q)
                for (int pp = 0; pp < r_x; ++pp)
                    fs = fs + ol.state[m * OF + ov.off + (int64_t)(MLAMR_G + J * r_y + q) * ov.NX + (MLAMR_G + I * r_x + pp)];
            double cv = 0.0;
            if (o >= 0) {
                const int32_t *b = par.box + 4 * o;
                const int CNX = b[2] - b[0] + 1 + 2 * MLAMR_G;
                cv = par.state[m * PF + par.offset[o] + (int64_t)(cj - b[1] + MLAMR_G) * CNX + (ci - b[0] + MLAMR_G)];
            }
            dsum[m] = dsum[m] + ((cv * ac) - (fs * af));
        }
    }
#pragma unroll
    for (int m = 0; m < M; ++m) {
        const double s = block_sum<NTR>(dsum[m], red);
        if (threadIdx.x == 0) delta[((int64_t)p * gridDim.x + blockIdx.x) * M + m] = s;
    }
}

// ---------------------------------------------------------------------------
// standalone interpolate_state over a gathered coarse array (drop-in shim)
// ---------------------------------------------------------------------------
template <int M>
__global__ void k_interp_box(const double *ch, const double *chu, const double *chv, const double *cb,
                             const uint8_t *cavail, int clo_i, int clo_j, int cnx, int cny, int flo_i,
                             int flo_j, int fnx, int fny, const double *fb, int r_x, int r_y,
                             double tol, double *oh, double *ohu, double *ohv, int32_t *status) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= fnx * fny) return;
    const int fj = idx / fnx, fi = idx % fnx;
    const int gi = flo_i + fi, gj = flo_j + fj;
    const int pi = floordiv(gi, r_x), pj = floordiv(gj, r_y);
    const int ci = pi - clo_i, cj = pj - clo_j;
    if (ci < 0 || cj < 0 || ci >= cnx || cj >= cny) {
        atomicOr(status, MLAMR_ST_GEOMETRY);
        return;
    }
    const int64_t cplane = (int64_t)cnx * cny;
    Coarse5<M> c;
    const int di[5] = {0, -1, 1, 0, 0}, dj[5] = {0, 0, 0, -1, 1};
#pragma unroll
    for (int q = 0; q < 5; ++q) {
        const int x = ci + di[q], y = cj + dj[q];
        const bool in = x >= 0 && y >= 0 && x < cnx && y < cny;
        const int64_t k = (int64_t)y * cnx + x;
        c.avail[q] = in && cavail[k];
        c.B[q] = in ? cb[k] : 0.0;
#pragma unroll
        for (int m = 0; m < M; ++m) {
            c.h[q][m] = in ? ch[m * cplane + k] : 0.0;
            c.hu[q][m] = in ? chu[m * cplane + k] : 0.0;
            c.hv[q][m] = in ? chv[m * cplane + k] : 0.0;
        }
    }
    // slopes are zero at the gathered array border (refine.py:88-91): an
    // out-of-array neighbour is treated as unusable
    Slopes<M> s;
    parent_slopes<M>(c, tol, s);
    double h[M], hu[M], hv[M];
    fine_cell<M>(s, child_offset(gi, pi, r_x), child_offset(gj, pj, r_y), fb[idx], tol, h, hu, hv);
    const int64_t fplane = (int64_t)fnx * fny;
#pragma unroll
    for (int m = 0; m < M; ++m) {
        oh[m * fplane + idx] = h[m];
        ohu[m * fplane + idx] = hu[m];
        ohv[m * fplane + idx] = hv[m];
    }
}

// ---------------------------------------------------------------------------
// K6: composite mass partials + non-finite scan (driver.py:138-153, 286-297)
// ---------------------------------------------------------------------------
template <int M>
__global__ void __launch_bounds__(NTA) k_level_reduce(mlamr_level lv, const double *interior,
                                                      const double *ghosts, const int32_t *child,
                                                      int child_rx, int child_ry, double *patch_mass,
                                                      int32_t *status, const int32_t *plist,
                                                      const int64_t *gbase, const int64_t *plan, int nrows) {
    __shared__ int bad;
    const int row = grid_row();
    if (row >= nrows) return;
    const int p = plist ? plist[row] : row;
    const PatchView pv = patch_view(lv, p);
    const int64_t FS = lv.field_stride;
    if (threadIdx.x == 0) bad = 0;
    __syncthreads();
    double msum[M];
#pragma unroll
    for (int m = 0; m < M; ++m) msum[m] = 0.0;
    int nonfinite = 0;
    for (int idx = blockIdx.x * NTA + threadIdx.x; idx < pv.NX * pv.NY; idx += gridDim.x * NTA) {
        const int J = idx / pv.NX, I = idx % pv.NX;
        const bool inner = J >= MLAMR_G && J < pv.NY - MLAMR_G && I >= MLAMR_G && I < pv.NX - MLAMR_G;
        const double *st = inner ? interior : ghosts;
        const int64_t k = pv.off + idx;
        int64_t kc = k;
        if (!inner && plan != nullptr) {
            // frame whose sibling cells the step read through the ghost plan
            // (fused sibling fill): check the sibling cell the copy would
            // have brought in
            const int gi = (J < MLAMR_G) ? J * pv.NX + I
                         : (J >= pv.NY - MLAMR_G) ? 2 * pv.NX + (J - (pv.NY - MLAMR_G)) * pv.NX + I
                         : 4 * pv.NX + (J - MLAMR_G) * 4 + (I < MLAMR_G ? I : I - pv.NX + 4);
            const int64_t v = plan[gbase[p] + gi];
            if (v >= 0) kc = v;
        }
        for (int q = 0; q < 3 * M; ++q)
            if (!isfinite(st[q * FS + kc])) nonfinite = 1;
        if (inner) {
            const int gi = pv.lo_i + I - MLAMR_G, gj = pv.lo_j + J - MLAMR_G;
            const bool covered = child != nullptr && owner_at(child, lv.level_nx, lv.level_ny, gi, gj) >= 0;
            if (!covered) {
#pragma unroll
                for (int m = 0; m < M; ++m) msum[m] = msum[m] + interior[m * FS + k];
            }
        }
    }
    if (nonfinite) atomicOr(&bad, 1);
    // fixed warp-shuffle tree, then the warp partials in warp order (one
    // barrier instead of a shared-memory tree per layer): deterministic
    __shared__ double wred[M][NTA / 32];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
        for (int m = 0; m < M; ++m) msum[m] = msum[m] + __shfl_xor_sync(0xffffffffu, msum[m], off);
    }
    if ((threadIdx.x & 31) == 0) {
#pragma unroll
        for (int m = 0; m < M; ++m) wred[m][threadIdx.x >> 5] = msum[m];
    }
    __syncthreads();
    if (threadIdx.x < M) {
        const int m = threadIdx.x;
        double sm = wred[m][0];
#pragma unroll
        for (int w = 1; w < NTA / 32; ++w) sm = sm + wred[m][w];
        patch_mass[((int64_t)p * gridDim.x + blockIdx.x) * M + m] = sm;
    }
    if (threadIdx.x == 0 && bad) atomicOr(status, MLAMR_ST_NONFINITE);
}

// ---------------------------------------------------------------------------
// reference flag rule, per cell part (regrid.flag_cells, regrid.py:58-101)
// bit0 amplitude flag, bit(1+m) wet layer m, bit7 covered.
// ---------------------------------------------------------------------------
template <int M>
__global__ void __launch_bounds__(NTA) k_flag_cells(mlamr_level lv, const double *st, mlamr_params prm,
                                                    const double *eta_rest, const double *wave_tol,
                                                    uint8_t *bits, const int32_t *plist, int nrows) {
    const int row = grid_row();
    if (row >= nrows) return;
    const int p = plist ? plist[row] : row;
    const PatchView pv = patch_view(lv, p);
    const int64_t FS = lv.field_stride;
    const double tol = prm.dry_tolerance;
    for (int idx = blockIdx.x * NTA + threadIdx.x; idx < pv.nx * pv.ny; idx += gridDim.x * NTA) {
        const int J = idx / pv.nx, I = idx % pv.nx;
        const int64_t k = pv.off + (int64_t)(J + MLAMR_G) * pv.NX + (I + MLAMR_G);
        const double B = lv.bathy[k];
        // rest depths from the rest surfaces (scenario.py:73-96, state.py:72-101)
        double hr[M], h[M];
        double bhat = 0.0 + B;
#pragma unroll
        for (int m = M - 1; m >= 0; --m) {
            const double d = eta_rest[m] - bhat;
            hr[m] = np_max(d, 0.0);
            bhat = bhat + hr[m];
            h[m] = st[m * FS + k];
        }
        uint8_t out = 0x80;
        double acc = 0.0, accr = 0.0;
#pragma unroll
        for (int m = M - 1; m >= 0; --m) {
            acc = (m == M - 1) ? h[m] : acc + h[m];
            accr = (m == M - 1) ? hr[m] : accr + hr[m];
            const double eta = acc + B;
            const double er = accr + B;
            if (fabs(eta - er) > wave_tol[m]) out |= 1;
            if (h[m] > tol) out |= (uint8_t)(2u << m);
        }
        bits[(int64_t)(pv.lo_j + J) * lv.level_nx + (pv.lo_i + I)] = out;
    }
}

// ---------------------------------------------------------------------------
// level-wide flag morphology on byte maps (mesh.dilate / mesh.erode,
// mesh.py:116-141): 3x3 neighbourhood OR (outside = 0) / AND (outside = 1),
// applied bytewise so each bit plane dilates independently.
// ---------------------------------------------------------------------------
__global__ void k_morph3(const uint8_t *in, uint8_t *out, int ny, int nx, int erode) {
    const int64_t n = (int64_t)ny * nx;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int j = (int)(idx / nx), i = (int)(idx - (int64_t)j * nx);
        uint8_t acc = erode ? 0xff : 0;
        for (int dj = -1; dj <= 1; ++dj)
            for (int di = -1; di <= 1; ++di) {
                const int jj = j + dj, ii = i + di;
                const bool inb = jj >= 0 && ii >= 0 && jj < ny && ii < nx;
                const uint8_t v = inb ? in[(int64_t)jj * nx + ii] : (erode ? 0xff : 0);
                acc = erode ? (acc & v) : (acc | v);
            }
        out[idx] = acc;
    }
}

// stage 1 of the reference rule from the per-cell bits: per layer m the
// plane "covered and dry" (regrid.py:91-92) as bit m
__global__ void k_dry_planes(const uint8_t *bits, uint8_t *dry, int64_t n, int M) {
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const uint8_t b = bits[idx];
        uint8_t d = 0;
        if (b & 0x80)
            for (int m = 0; m < M; ++m)
                if (!(b & (2u << m))) d |= (uint8_t)(1u << m);
        dry[idx] = d;
    }
}

// stage 2: amplitude flags | wet_m & near-dry_m (regrid.py:96-98)
__global__ void k_flag_combine(const uint8_t *bits, const uint8_t *neardry, uint8_t *flags, int64_t n,
                               int M) {
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const uint8_t b = bits[idx];
        uint8_t f = b & 1;
        for (int m = 0; m < M; ++m)
            if ((b & (2u << m)) && (neardry[idx] & (1u << m))) f = 1;
        flags[idx] = f;
    }
}

// final: flags & covered & allowed; allowed = erode(covered, 1)
__global__ void k_flag_mask(uint8_t *flags, const uint8_t *bits, const uint8_t *allowed, int64_t n) {
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n;
         idx += (int64_t)gridDim.x * blockDim.x)
        flags[idx] = (flags[idx] && (bits[idx] & 0x80) && allowed[idx]) ? 1 : 0;
}

__global__ void k_covered(const uint8_t *bits, uint8_t *cov, int64_t n) {
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n;
         idx += (int64_t)gridDim.x * blockDim.x)
        cov[idx] = (bits[idx] & 0x80) ? 1 : 0;
}

template <typename F>
static int dispatch_m(int M, F &&f) {
    switch (M) {
        case 1: f(std::integral_constant<int, 1>{}); return 0;
        case 2: f(std::integral_constant<int, 2>{}); return 0;
        case 3: f(std::integral_constant<int, 3>{}); return 0;
        default: return -1;
    }
}

static inline int blocks_for(int64_t n, int maxb = 64) {
    int64_t b = (n + NTA - 1) / NTA;
    if (b < 1) b = 1;
    if (b > maxb) b = maxb;
    return (int)b;
}

}  // namespace mlamr

#include <type_traits>

using namespace mlamr;

extern "C" int mlamr_paint_owner(int32_t *map, int map_nx, int map_ny, const int32_t *box,
                                 int num_patches, int grow, int first_wins, int r_x, int r_y,
                                 int max_cells, void *stream) {
    if (num_patches <= 0) return 0;
    const dim3 grid = row_grid(blocks_for(max_cells, 256), num_patches);
    k_paint<<<grid, NTA, 0, as_stream(stream)>>>(map, map_nx, map_ny, box, grow, first_wins, r_x, r_y, num_patches);
    return (int)cudaGetLastError();
}

extern "C" int mlamr_fill_ghosts(mlamr_level lv, const mlamr_level *parent, const double *parent_old_state,
                                 double theta, int r_x, int r_y, const int32_t *bcs, mlamr_params prm,
                                 const int32_t *status, const int32_t *patch_list, int n_list, void *stream) {
    const int nb = patch_list ? n_list : lv.num_patches;
    if (nb <= 0) return 0;
    mlamr_level par = parent ? *parent : lv;
    const int4 b = make_int4(bcs[0], bcs[1], bcs[2], bcs[3]);
    cudaStream_t st = as_stream(stream);
    int rc = dispatch_m(prm.num_layers, [&](auto Mc) {
        constexpr int M = decltype(Mc)::value;
        k_fill_ghosts<M><<<nb, NTA, 0, st>>>(lv, par, parent != nullptr, parent_old_state, theta,
                                             r_x, r_y, b, prm, status, patch_list);
    });
    if (rc) return rc;
    return (int)cudaGetLastError();
}

extern "C" int mlamr_ghost_plan(mlamr_level lv, const int64_t *gbase, int64_t *plan, int max_ghost,
                                void *stream) {
    if (lv.num_patches <= 0) return 0;
    const dim3 grid = row_grid((unsigned)std::max(1, std::min(16, (max_ghost + NTA - 1) / NTA)), lv.num_patches);
    k_ghost_plan<<<grid, NTA, 0, as_stream(stream)>>>(lv, gbase, plan);
    return (int)cudaGetLastError();
}

extern "C" int mlamr_fill_ghosts_planned(mlamr_level lv, const mlamr_level *parent, const double *parent_old_state,
                                         double theta, int r_x, int r_y, const int32_t *bcs, mlamr_params prm,
                                         const int32_t *status, const int64_t *gbase, const int64_t *plan,
                                         const int32_t *patch_list, int n_list, int max_ghost,
                                         const int32_t *interp_cells, int n_interp, const int32_t *n_interp_dev,
                                         const int32_t *bc_patches, int n_bc, void *stream) {
    const int nb = patch_list ? n_list : lv.num_patches;
    cudaStream_t st = as_stream(stream);
    const int4 b = make_int4(bcs[0], bcs[1], bcs[2], bcs[3]);
    int rc = dispatch_m(prm.num_layers, [&](auto Mc) {
        constexpr int M = decltype(Mc)::value;
        if (nb > 0) k_fill_copy<M><<<nb, NTC, 0, st>>>(lv, gbase, plan, patch_list, status);
        if (parent != nullptr && n_interp > 0) {
            // with a device-side count n_interp is only a capacity: a
            // grid-stride launch of at most 8 blocks per SM
            const int cap = n_interp_dev ? 148 * 8 : 148 * 32;
            const int blocks = (int)std::min<int64_t>((n_interp + NTA - 1) / NTA, cap);
            k_fill_interp<M><<<blocks, NTA, 0, st>>>(lv, *parent, parent_old_state, theta, r_x, r_y,
                                                     interp_cells, n_interp, n_interp_dev, prm, status);
        }
        if (n_bc > 0) k_fill_bc<M><<<n_bc, NTA, 0, st>>>(lv, bc_patches, b, status);
    });
    if (rc) return rc;
    return (int)cudaGetLastError();
}

// Column sums of per-block partials: one block per column, a fixed
// thread-strided order and a fixed tree, so the result is deterministic.
__global__ void __launch_bounds__(NTA) k_sum_partials(const double *part, long long rows, int cols, double scale,
                                                      double *acc, double *acc2, int init) {
    __shared__ double red[NTA];
    const int c = blockIdx.x;
    double v = 0.0;
    for (long long r = threadIdx.x; r < rows; r += NTA) v = v + part[r * cols + c];
    const double sm = block_sum<NTA>(v, red);
    if (threadIdx.x == 0) {
        const double sc = sm * scale;
        acc[c] = init ? sc : acc[c] + sc;
        if (acc2 != nullptr) acc2[c] = acc2[c] + sc;
    }
}

extern "C" int mlamr_sum_partials(const double *part, long long rows, int cols, double scale, double *acc,
                                  double *acc2, int init, void *stream) {
    cudaStream_t st = as_stream(stream);
    if (cols <= 0) return 0;
    if (rows <= 0) {
        if (!init) return 0;
        return (int)cudaMemsetAsync(acc, 0, sizeof(double) * cols, st);   // +0.0
    }
    k_sum_partials<<<cols, NTA, 0, st>>>(part, rows, cols, scale, acc, acc2, init);
    return (int)cudaGetLastError();
}

extern "C" int mlamr_plan_interp_cells(mlamr_level lv, const int64_t *gbase, const int64_t *plan,
                                       const int32_t *patch_list, int n_list, int max_ghost, int32_t *cells,
                                       int32_t *count, void *stream) {
    cudaStream_t st = as_stream(stream);
    cudaError_t e = cudaMemsetAsync(count, 0, sizeof(int32_t), st);
    if (e != cudaSuccess) return (int)e;
    const int nb = patch_list ? n_list : lv.num_patches;
    if (nb <= 0) return 0;
    const dim3 grid = row_grid((unsigned)std::max(1, std::min(16, (max_ghost + NTA - 1) / NTA)), nb);
    k_plan_interp_cells<<<grid, NTA, 0, st>>>(lv, gbase, plan, patch_list, nb, cells, count);
    return (int)cudaGetLastError();
}

extern "C" int mlamr_copy_pairs_of_plan(mlamr_level lv, const int64_t *gbase, const int64_t *plan,
                                        const int32_t *patch_list, int n_list, const int64_t *list_base,
                                        int max_ghost, int64_t *pairs, void *stream) {
    const int nb = patch_list ? n_list : lv.num_patches;
    if (nb <= 0) return 0;
    const dim3 grid = row_grid((unsigned)std::max(1, std::min(16, (max_ghost + NTA - 1) / NTA)), nb);
    k_copy_pairs_of_plan<<<grid, NTA, 0, as_stream(stream)>>>(lv, gbase, plan, patch_list, list_base, pairs, nb);
    return (int)cudaGetLastError();
}

extern "C" int mlamr_fill_copy_pairs(double *state, int64_t field_stride, const int64_t *pairs, int64_t n_pairs,
                                     int num_layers, const int32_t *status, void *stream) {
    if (n_pairs <= 0) return 0;
    const int blocks = (int)std::min<int64_t>((n_pairs + NTA - 1) / NTA, 148 * 16);
    cudaStream_t st = as_stream(stream);
    int rc = dispatch_m(num_layers, [&](auto Mc) {
        constexpr int M = decltype(Mc)::value;
        k_fill_copy_pairs<M><<<blocks, NTA, 0, st>>>(state, field_stride, pairs, n_pairs, status);
    });
    if (rc) return rc;
    return (int)cudaGetLastError();
}

extern "C" int mlamr_fill_bathymetry(mlamr_level lv, const double *level_bathy, const int32_t *bcs,
                                     void *stream) {
    if (lv.num_patches <= 0) return 0;
    const int4 b = make_int4(bcs[0], bcs[1], bcs[2], bcs[3]);
    k_fill_bathy<<<lv.num_patches, NTA, 0, as_stream(stream)>>>(lv, level_bathy, b);
    return (int)cudaGetLastError();
}

extern "C" int mlamr_average_down(mlamr_level fine, mlamr_level coarse, int r_x, int r_y, mlamr_params prm,
                                  double *patch_delta, int blocks_per_patch, const int32_t *status,
                                  void *stream) {
    if (fine.num_patches <= 0) return 0;
    const dim3 grid = row_grid(blocks_per_patch, fine.num_patches);
    cudaStream_t st = as_stream(stream);
    int rc = dispatch_m(prm.num_layers, [&](auto Mc) {
        constexpr int M = decltype(Mc)::value;
        if (r_x == 4 && r_y == 4)
            k_average_down<M, 4, 4><<<grid, NTA, 0, st>>>(fine, coarse, r_x, r_y, prm, patch_delta, status);
        else if (r_x == 2 && r_y == 2)
            k_average_down<M, 2, 2><<<grid, NTA, 0, st>>>(fine, coarse, r_x, r_y, prm, patch_delta, status);
        else if (r_x == 4 && r_y == 2)
            k_average_down<M, 4, 2><<<grid, NTA, 0, st>>>(fine, coarse, r_x, r_y, prm, patch_delta, status);
        else
            k_average_down<M, 0, 0><<<grid, NTA, 0, st>>>(fine, coarse, r_x, r_y, prm, patch_delta, status);
    });
    if (rc) return rc;
    return (int)cudaGetLastError();
}

extern "C" int mlamr_average_down_flat(mlamr_level fine, mlamr_level coarse, int r_x, int r_y, mlamr_params prm,
                                       const int64_t *coarse_base, int64_t n_coarse, const int32_t *status,
                                       void *stream) {
    if (fine.num_patches <= 0 || n_coarse <= 0) return 0;
    const int blocks = (int)std::min<int64_t>((n_coarse + NTA - 1) / NTA, 148 * 16);
    cudaStream_t st = as_stream(stream);
    int rc = dispatch_m(prm.num_layers, [&](auto Mc) {
        constexpr int M = decltype(Mc)::value;
        if (r_x == 4 && r_y == 4)
            k_average_down_flat<M, 4, 4><<<blocks, NTA, 0, st>>>(fine, coarse, r_x, r_y, prm, coarse_base, n_coarse, status);
        else if (r_x == 2 && r_y == 2)
            k_average_down_flat<M, 2, 2><<<blocks, NTA, 0, st>>>(fine, coarse, r_x, r_y, prm, coarse_base, n_coarse, status);
        else if (r_x == 4 && r_y == 2)
            k_average_down_flat<M, 4, 2><<<blocks, NTA, 0, st>>>(fine, coarse, r_x, r_y, prm, coarse_base, n_coarse, status);
        else
            k_average_down_flat<M, 0, 0><<<blocks, NTA, 0, st>>>(fine, coarse, r_x, r_y, prm, coarse_base, n_coarse, status);
    });
    if (rc) return rc;
    return (int)cudaGetLastError();
}

extern "C" int mlamr_check_bathymetry(mlamr_level fine, mlamr_level coarse, int r_x, int r_y, double atol,
                                      const int64_t *coarse_base, int64_t n_coarse, int32_t *status,
                                      int32_t *bad_patch, void *stream) {
    if (fine.num_patches <= 0 || n_coarse <= 0 || coarse.num_patches <= 0) return 0;
    const int blocks = (int)std::min<int64_t>((n_coarse + NTA - 1) / NTA, 148 * 8);
    k_check_bathy<<<blocks, NTA, 0, as_stream(stream)>>>(fine, coarse, r_x, r_y, atol, coarse_base, n_coarse, status,
                                                         bad_patch);
    return (int)cudaGetLastError();
}

extern "C" int mlamr_regrid_fill(mlamr_level newlv, mlamr_level oldlv, mlamr_level parent, int r_x, int r_y,
                                 mlamr_params prm, double *refine_delta, int blocks_per_patch,
                                 int32_t *status, const int32_t *patch_list, int n_list, void *stream) {
    const int nb = patch_list ? n_list : newlv.num_patches;
    if (nb <= 0) return 0;
    const dim3 grid = row_grid(blocks_per_patch, nb);
    cudaStream_t st = as_stream(stream);
    int rc = dispatch_m(prm.num_layers, [&](auto Mc) {
        constexpr int M = decltype(Mc)::value;
        // one block per patch (small patches, e.g. C5's 16x16): 64 threads,
        // so a patch's few cells do not leave most of a block idle
        if (blocks_per_patch == 1)
            k_regrid_fill<M, 64><<<grid, 64, 0, st>>>(newlv, oldlv, parent, r_x, r_y, prm, refine_delta, status,
                                                      patch_list, nb);
        else
            k_regrid_fill<M><<<grid, NTA, 0, st>>>(newlv, oldlv, parent, r_x, r_y, prm, refine_delta, status,
                                                   patch_list, nb);
    });
    if (rc) return rc;
    return (int)cudaGetLastError();
}

extern "C" int mlamr_derefine_delta(mlamr_level oldlv, mlamr_level parent, const int32_t *new_child,
                                    int r_x, int r_y, mlamr_params prm, double *derefine_delta,
                                    int blocks_per_patch, const int32_t *patch_list, int n_list, void *stream) {
    const int nb = patch_list ? n_list : oldlv.num_patches;
    if (nb <= 0) return 0;
    const dim3 grid = row_grid(blocks_per_patch, nb);
    cudaStream_t st = as_stream(stream);
    int rc = dispatch_m(prm.num_layers, [&](auto Mc) {
        constexpr int M = decltype(Mc)::value;
        if (blocks_per_patch == 1)
            k_derefine<M, 64><<<grid, 64, 0, st>>>(oldlv, parent, new_child, r_x, r_y, derefine_delta, patch_list,
                                                   nb);
        else
            k_derefine<M><<<grid, NTA, 0, st>>>(oldlv, parent, new_child, r_x, r_y, derefine_delta, patch_list, nb);
    });
    if (rc) return rc;
    return (int)cudaGetLastError();
}

extern "C" int mlamr_interpolate_box(int M, const double *ch, const double *chu, const double *chv,
                                     const double *cb, const uint8_t *cavail, int clo_i, int clo_j, int cnx,
                                     int cny, int flo_i, int flo_j, int fnx, int fny, const double *fb,
                                     int r_x, int r_y, mlamr_params prm, double *oh, double *ohu,
                                     double *ohv, int32_t *status, void *stream) {
    const int n = fnx * fny;
    if (n <= 0) return 0;
    cudaStream_t st = as_stream(stream);
    const int nb = (n + 127) / 128;
    int rc = dispatch_m(M, [&](auto Mc) {
        constexpr int MM = decltype(Mc)::value;
        k_interp_box<MM><<<nb, 128, 0, st>>>(ch, chu, chv, cb, cavail, clo_i, clo_j, cnx, cny, flo_i, flo_j,
                                             fnx, fny, fb, r_x, r_y, prm.dry_tolerance, oh, ohu, ohv, status);
    });
    if (rc) return rc;
    return (int)cudaGetLastError();
}

extern "C" int mlamr_level_reduce(mlamr_level lv, const double *interior_state, const double *ghost_state,
                                  const int32_t *child, double *patch_mass, int blocks_per_patch,
                                  int32_t *status, const int32_t *patch_list, int n_list, void *stream) {
    return mlamr_level_reduce_planned(lv, interior_state, ghost_state, child, patch_mass, blocks_per_patch,
                                      status, patch_list, n_list, nullptr, nullptr, stream);
}

extern "C" int mlamr_level_reduce_planned(mlamr_level lv, const double *interior_state,
                                          const double *ghost_state, const int32_t *child, double *patch_mass,
                                          int blocks_per_patch, int32_t *status, const int32_t *patch_list,
                                          int n_list, const int64_t *ghost_base, const int64_t *ghost_plan,
                                          void *stream) {
    const int nb = patch_list ? n_list : lv.num_patches;
    if (nb <= 0) return 0;
    const dim3 grid = row_grid(blocks_per_patch, nb);
    cudaStream_t st = as_stream(stream);
    int rc = dispatch_m(lv.num_layers, [&](auto Mc) {
        constexpr int M = decltype(Mc)::value;
        k_level_reduce<M><<<grid, NTA, 0, st>>>(lv, interior_state, ghost_state, child, 1, 1, patch_mass,
                                                status, patch_list, ghost_plan ? ghost_base : nullptr,
                                                ghost_plan, nb);
    });
    if (rc) return rc;
    return (int)cudaGetLastError();
}

extern "C" int mlamr_flag_cells(mlamr_level lv, const double *state, mlamr_params prm, const double *eta_rest,
                                const double *wave_tol, uint8_t *cell_bits, int blocks_per_patch,
                                const int32_t *patch_list, int n_list, void *stream) {
    const int nb = patch_list ? n_list : lv.num_patches;
    if (nb <= 0) return 0;
    const dim3 grid = row_grid(blocks_per_patch, nb);
    cudaStream_t st = as_stream(stream);
    int rc = dispatch_m(prm.num_layers, [&](auto Mc) {
        constexpr int M = decltype(Mc)::value;
        k_flag_cells<M><<<grid, NTA, 0, st>>>(lv, state, prm, eta_rest, wave_tol, cell_bits, patch_list, nb);
    });
    if (rc) return rc;
    return (int)cudaGetLastError();
}

// Whole-patch block copies between a pool and a packed exchange buffer (or
// another pool): seg[3*s] = src offset, seg[3*s+1] = dst offset, seg[3*s+2]
// = length in elements, applied to every one of `nplanes` planes.
__global__ void k_copy_segments(const double *__restrict__ src, int64_t src_stride, double *__restrict__ dst,
                                int64_t dst_stride, const int64_t *__restrict__ seg, int nplanes, int nrows) {
    const int sg = grid_row();
    if (sg >= nrows) return;
    const int64_t so = seg[3 * sg], doff = seg[3 * sg + 1], len = seg[3 * sg + 2];
    for (int q = 0; q < nplanes; ++q)
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len;
             i += (int64_t)gridDim.x * blockDim.x)
            dst[q * dst_stride + doff + i] = src[q * src_stride + so + i];
}

extern "C" int mlamr_copy_segments(const double *src, int64_t src_stride, double *dst, int64_t dst_stride,
                                   const int64_t *segments, int n_segments, int max_len, int nplanes,
                                   void *stream) {
    if (n_segments <= 0) return 0;
    const dim3 grid = row_grid((unsigned)std::max(1, std::min(8, (max_len + 255) / 256)), n_segments);
    k_copy_segments<<<grid, 256, 0, as_stream(stream)>>>(src, src_stride, dst, dst_stride, segments, nplanes,
                                                         n_segments);
    return (int)cudaGetLastError();
}

// Checkpoints (Simulation.snapshot / restore): the interiors of every patch
// of a level, plane by plane, packed contiguously (patch order, rows
// x-fastest; pbase = prefix sums of the interior sizes).  Ghost frames and
// alignment padding are rebuilt before anything reads them (every level's
// advance starts with its fill), so a checkpoint carries only these.
__global__ void __launch_bounds__(NTA) k_pack_interiors(mlamr_level lv, double *state, double *packed,
                                                        const int64_t *pbase, int64_t ntot, int nplanes,
                                                        int unpack) {
    const int p = grid_row();
    if (p >= lv.num_patches) return;
    const PatchView pv = patch_view(lv, p);
    const int n = pv.nx * pv.ny;
    const int64_t pb = pbase[p];
    const int64_t FS = lv.field_stride;
    for (int idx = blockIdx.x * NTA + threadIdx.x; idx < n; idx += gridDim.x * NTA) {
        const int j = idx / pv.nx, i = idx - j * pv.nx;
        const int64_t k = pv.off + (int64_t)(j + MLAMR_G) * pv.NX + (i + MLAMR_G);
        for (int q = 0; q < nplanes; ++q) {
            if (unpack)
                state[q * FS + k] = packed[q * ntot + pb + idx];
            else
                packed[q * ntot + pb + idx] = state[q * FS + k];
        }
    }
}

extern "C" int mlamr_pack_interiors(mlamr_level lv, double *state, double *packed, const int64_t *pbase,
                                    int64_t n_total, int max_interior, int unpack, void *stream) {
    if (lv.num_patches <= 0) return 0;
    const dim3 grid = row_grid((unsigned)std::max(1, std::min(4, (max_interior + NTA - 1) / NTA)), lv.num_patches);
    k_pack_interiors<<<grid, NTA, 0, as_stream(stream)>>>(lv, state, packed, pbase, n_total, 3 * lv.num_layers,
                                                          unpack);
    return (int)cudaGetLastError();
}

// self-test of the shared-reciprocal division against div.rn.f64
__global__ void k_selftest_div(const double *a, const double *b, int n, unsigned long long *bad,
                               unsigned long long *slow) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const double x = a[i], y = b[i];
        bool ok = true;
        const double r = recip_nr(y);
        const double q = div_fast(x, y, r, ok);
        const double ref = x / y;
        // the kernels' fallback for a refused division must be `/` too
        const double got = ok ? q : div_slow(x, y);
        if (!ok) atomicAdd(slow, 1ull);
        if (__double_as_longlong(got) != __double_as_longlong(ref) && !(got != got && ref != ref))
            atomicAdd(bad, 1ull);
    }
}

extern "C" int mlamr_selftest_div(const double *a, const double *b, int n, unsigned long long *bad,
                                  unsigned long long *slow, void *stream) {
    k_selftest_div<<<592, 256, 0, as_stream(stream)>>>(a, b, n, bad, slow);
    return (int)cudaGetLastError();
}

// Summed-area table of a 0/1 byte map for the clustering bisection
// (regrid.cluster_flags, regrid.py:129-182, evaluated from box sums):
// sat[(j+1)*(nx+1) + (i+1)] = sum of v over [0,j] x [0,i], v = map or
// 1 - map (invert), row 0 and column 0 zero.  Integer sums, so the result
// is exact in any order: one warp scans each row with shuffles, then the
// columns are scanned in row segments (segment sums, their scan, the add).
constexpr int SAT_SEG = 32;  // rows per column segment

__global__ void k_sat_rows(const uint8_t *__restrict__ map, int ny, int nx, int invert, int32_t *__restrict__ sat) {
    const int lane = threadIdx.x & 31;
    const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (row > ny) return;
    int32_t *out = sat + (int64_t)row * (nx + 1);
    if (row == 0) {
        for (int i = lane; i <= nx; i += 32) out[i] = 0;
        return;
    }
    const uint8_t *in = map + (int64_t)(row - 1) * nx;
    if (lane == 0) out[0] = 0;
    int carry = 0;
    for (int i0 = 0; i0 < nx; i0 += 32) {
        const int i = i0 + lane;
        int v = (i < nx) ? (invert ? 1 - (int)in[i] : (int)in[i]) : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int u = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += u;
        }
        if (i < nx) out[i + 1] = carry + v;
        carry += __shfl_sync(0xffffffffu, v, 31);
    }
}

__global__ void k_sat_cols_local(int32_t *__restrict__ sat, int ny, int nx, int32_t *__restrict__ segsum) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x + 1;  // column 1..nx
    const int seg = blockIdx.y;
    if (i > nx) return;
    const int j0 = 1 + seg * SAT_SEG, j1 = min(ny, j0 + SAT_SEG - 1);
    int acc = 0;
    for (int j = j0; j <= j1; ++j) {
        int32_t *q = sat + (int64_t)j * (nx + 1) + i;
        acc += *q;
        *q = acc;
    }
    segsum[(int64_t)seg * nx + (i - 1)] = acc;
}

__global__ void k_sat_cols_scan(int32_t *__restrict__ segsum, int nseg, int nx) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nx) return;
    int acc = 0;
    for (int s = 0; s < nseg; ++s) {  // exclusive scan over segments
        const int v = segsum[(int64_t)s * nx + i];
        segsum[(int64_t)s * nx + i] = acc;
        acc += v;
    }
}

__global__ void k_sat_cols_add(int32_t *__restrict__ sat, int ny, int nx, const int32_t *__restrict__ segsum) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x + 1;
    const int seg = blockIdx.y + 1;  // segment 0 has offset 0
    if (i > nx) return;
    const int off = segsum[(int64_t)seg * nx + (i - 1)];
    const int j0 = 1 + seg * SAT_SEG, j1 = min(ny, j0 + SAT_SEG - 1);
    for (int j = j0; j <= j1; ++j) sat[(int64_t)j * (nx + 1) + i] += off;
}

extern "C" int mlamr_sat_u8(const uint8_t *map, int ny, int nx, int invert, int32_t *sat, int32_t *scratch,
                            void *stream) {
    cudaStream_t st = as_stream(stream);
    if (ny <= 0 || nx <= 0) return 0;
    const int wpb = 8;
    k_sat_rows<<<(ny + 1 + wpb - 1) / wpb, 32 * wpb, 0, st>>>(map, ny, nx, invert, sat);
    const int nseg = (ny + SAT_SEG - 1) / SAT_SEG;
    const int cb = (nx + 127) / 128;
    k_sat_cols_local<<<dim3(cb, nseg), 128, 0, st>>>(sat, ny, nx, scratch);
    k_sat_cols_scan<<<cb, 128, 0, st>>>(scratch, nseg, nx);
    if (nseg > 1) k_sat_cols_add<<<dim3(cb, nseg - 1), 128, 0, st>>>(sat, ny, nx, scratch);
    return (int)cudaGetLastError();
}

// Frame records from a device pool (frames.write_frame / frame_from_hierarchy,
// frames.py:72-100, 141-163 of the reference): record p starts at element
// rec_off[p] of `out` (8-byte units) with five little-endian int64 (level,
// lo_i, lo_j, hi_i, hi_j), then the interior of bathymetry, h_0, hu_0, hv_0,
// h_1, ... as row-major ny x nx float64 planes.  Grid: (x blocks, patches);
// patch_list (optional) selects the patches, e.g. a rank's owned ones.
__global__ void k_pack_frame(mlamr_level lv, const double *__restrict__ state, int level_index,
                             const int64_t *__restrict__ rec_off, const int32_t *__restrict__ patch_list,
                             double *__restrict__ out, int nrows) {
    const int row = grid_row();
    if (row >= nrows) return;
    const int p = patch_list ? patch_list[row] : row;
    const PatchView pv = patch_view(lv, p);
    const int M = lv.num_layers;
    const int64_t n = (int64_t)pv.nx * pv.ny;
    double *rec = out + rec_off[p];
    if (blockIdx.x == 0 && threadIdx.x < 5) {
        const int64_t hdr[5] = {level_index, pv.lo_i, pv.lo_j, pv.lo_i + pv.nx - 1, pv.lo_j + pv.ny - 1};
        reinterpret_cast<int64_t *>(rec)[threadIdx.x] = hdr[threadIdx.x];
    }
    double *body = rec + 5;
    const int64_t FS = lv.field_stride;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int r = (int)(i / pv.nx), c = (int)(i - (int64_t)r * pv.nx);
        const int64_t k = pv.off + (int64_t)(r + MLAMR_G) * pv.NX + (c + MLAMR_G);
        body[i] = lv.bathy[k];
        for (int m = 0; m < M; ++m) {
            body[(1 + 3 * m) * n + i] = state[m * FS + k];
            body[(2 + 3 * m) * n + i] = state[(M + m) * FS + k];
            body[(3 + 3 * m) * n + i] = state[(2 * M + m) * FS + k];
        }
    }
}

extern "C" int mlamr_pack_frame(mlamr_level lv, const double *state, int level_index, const int64_t *rec_off,
                                const int32_t *patch_list, int n_list, int blocks_per_patch, double *out,
                                void *stream) {
    const int np = patch_list ? n_list : lv.num_patches;
    if (np <= 0) return 0;
    const dim3 grid = row_grid(blocks_per_patch > 0 ? blocks_per_patch : 1, np);
    k_pack_frame<<<grid, NTA, 0, as_stream(stream)>>>(lv, state, level_index, rec_off, patch_list, out, np);
    return (int)cudaGetLastError();
}

// Full reference flag rule + nesting mask on the device.  `bits` from
// mlamr_flag_cells; scratch = 3 byte maps of ny*nx.  Outputs: flags
// (0/1, already & covered & allowed) and allowed = erode(covered, 1).
extern "C" int mlamr_flags_reference(const uint8_t *bits, int ny, int nx, int M, int buffer_width,
                                     uint8_t *flags, uint8_t *allowed, uint8_t *scratch, void *stream) {
    cudaStream_t st = as_stream(stream);
    const int64_t n = (int64_t)ny * nx;
    if (n <= 0) return 0;
    const int nb = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
    uint8_t *a = scratch, *b = scratch + n, *c = scratch + 2 * n;
    k_dry_planes<<<nb, 256, 0, st>>>(bits, a, n, M);
    for (int w = 0; w < buffer_width; ++w) {
        k_morph3<<<nb, 256, 0, st>>>(a, b, ny, nx, 0);
        uint8_t *t = a; a = b; b = t;
    }
    k_flag_combine<<<nb, 256, 0, st>>>(bits, a, c, n, M);
    uint8_t *fa = c, *fb = b;
    for (int w = 0; w < buffer_width; ++w) {
        k_morph3<<<nb, 256, 0, st>>>(fa, fb, ny, nx, 0);
        uint8_t *t = fa; fa = fb; fb = t;
    }
    k_covered<<<nb, 256, 0, st>>>(bits, a == fa ? fb : a, n);
    uint8_t *cov = (a == fa) ? fb : a;
    k_morph3<<<nb, 256, 0, st>>>(cov, allowed, ny, nx, 1);
    k_flag_mask<<<nb, 256, 0, st>>>(fa, bits, allowed, n);
    cudaMemcpyAsync(flags, fa, n, cudaMemcpyDeviceToDevice, st);
    return (int)cudaGetLastError();
}

// Harness Bernoulli flag rule (problems.Problem.bernoulli_flags, C5): the
// counter hash of (seed, stream, j, i) -- splitmix64's finaliser, the same
// uint64 arithmetic as problems.hash_uniform, so the uniforms are
// bit-identical to numpy's -- below p flags the cell.  Writes the flag
// plane and the coverage bits (0x80) of the level's interior owner map.
__global__ void k_bernoulli(const int32_t *own, int ny, int nx, unsigned long long seed,
                            unsigned long long stream_id, double p, uint8_t *flag, uint8_t *bits) {
    const int64_t n = (int64_t)ny * nx;
    const unsigned long long G = 0x9E3779B97F4A7C15ull, M1 = 0xBF58476D1CE4E5B9ull, M2 = 0x94D049BB133111EBull;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int j = (int)(idx / nx), i = (int)(idx - (int64_t)j * nx);
        unsigned long long z = seed * G + stream_id * M2 + ((unsigned long long)(long long)j << 32) +
                               (unsigned long long)(long long)i;
        z = (z ^ (z >> 30)) * M1;
        z = (z ^ (z >> 27)) * M2;
        z = z ^ (z >> 31);
        const double u = (double)(z >> 11) * (1.0 / 9007199254740992.0);
        flag[idx] = u < p ? 1 : 0;
        const bool cov = own[(int64_t)(j + MLAMR_G) * (nx + 2 * MLAMR_G) + (i + MLAMR_G)] >= 0;
        bits[idx] = cov ? 0x80 : 0;
    }
}

// flags = dilate^w(bernoulli) & covered & allowed, allowed = erode(covered, 1)
// (the driver's host rule for "bernoulli"); scratch is
// 3*ny*nx bytes.
extern "C" int mlamr_flags_bernoulli(const int32_t *own, int ny, int nx, unsigned long long seed,
                                     unsigned long long stream_id, double p, int dilate_w, uint8_t *flags,
                                     uint8_t *allowed, uint8_t *scratch, void *stream) {
    cudaStream_t st = as_stream(stream);
    const int64_t n = (int64_t)ny * nx;
    if (n <= 0) return 0;
    const int nb = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
    uint8_t *a = scratch, *b = scratch + n, *bits = scratch + 2 * n;
    k_bernoulli<<<nb, 256, 0, st>>>(own, ny, nx, seed, stream_id, p, a, bits);
    for (int w = 0; w < dilate_w; ++w) {
        k_morph3<<<nb, 256, 0, st>>>(a, b, ny, nx, 0);
        uint8_t *t = a; a = b; b = t;
    }
    k_covered<<<nb, 256, 0, st>>>(bits, b, n);
    k_morph3<<<nb, 256, 0, st>>>(b, allowed, ny, nx, 1);
    k_flag_mask<<<nb, 256, 0, st>>>(a, bits, allowed, n);
    cudaMemcpyAsync(flags, a, n, cudaMemcpyDeviceToDevice, st);
    return (int)cudaGetLastError();
}

// Harness gradient flag rule (problems.gradient_flags_map, C1/C3).  Stage 1:
// the surfaces eta_m = (h_{M-1} + ... + h_m) + B (numpy's reversed cumsum,
// driver.level_surfaces) of the requested layers on the level grid, from
// the interior owner (later patches win, as the host's overwrite), and the
// coverage bit.  Stage 2: a covered cell is flagged when |difference| /
// spacing across one of its faces with another covered cell exceeds tol.
template <int M>
__global__ void k_grad_eta(mlamr_level lv, const double *__restrict__ state, unsigned layer_mask,
                           double *__restrict__ eta, uint8_t *__restrict__ bits) {
    const int ny = lv.level_ny, nx = lv.level_nx;
    const int64_t n = (int64_t)ny * nx;
    const int64_t FS = lv.field_stride;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int j = (int)(idx / nx), i = (int)(idx - (int64_t)j * nx);
        const int o = owner_at(lv.own, nx, ny, i, j);
        if (o < 0) {
            bits[idx] = 0;
            continue;
        }
        bits[idx] = 0x80;
        const PatchView pv = patch_view(lv, o);
        const int64_t k = pv.off + (int64_t)(j - pv.lo_j + MLAMR_G) * pv.NX + (i - pv.lo_i + MLAMR_G);
        const double B = lv.bathy[k];
        double c = state[(M - 1) * FS + k];
        int slot = 0;
        double e[M];
        e[M - 1] = c + B;
#pragma unroll
        for (int m = M - 2; m >= 0; --m) {
            c = c + state[m * FS + k];
            e[m] = c + B;
        }
#pragma unroll
        for (int m = 0; m < M; ++m)
            if (layer_mask & (1u << m)) eta[(int64_t)(slot++) * n + idx] = e[m];
    }
}

__global__ void k_cov_bits(const uint8_t *covered, uint8_t *bits, int64_t n) {
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n;
         idx += (int64_t)gridDim.x * blockDim.x)
        bits[idx] = covered[idx] ? 0x80 : 0;
}

__global__ void k_grad_flags(const double *__restrict__ eta, int K, const uint8_t *__restrict__ bits, int ny,
                             int nx, double dx, double dy, double tol, uint8_t *__restrict__ flag) {
    const int64_t n = (int64_t)ny * nx;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int j = (int)(idx / nx), i = (int)(idx - (int64_t)j * nx);
        bool f = false;
        if (bits[idx] & 0x80) {
            const bool cl = i > 0 && (bits[idx - 1] & 0x80), cr = i + 1 < nx && (bits[idx + 1] & 0x80);
            const bool cb = j > 0 && (bits[idx - nx] & 0x80), ct = j + 1 < ny && (bits[idx + nx] & 0x80);
            for (int q = 0; q < K; ++q) {
                const double *e = eta + (int64_t)q * n;
                const double v = e[idx];
                if (cl && fabs(v - e[idx - 1]) / dx > tol) f = true;
                if (cr && fabs(e[idx + 1] - v) / dx > tol) f = true;
                if (cb && fabs(v - e[idx - nx]) / dy > tol) f = true;
                if (ct && fabs(e[idx + nx] - v) / dy > tol) f = true;
            }
        }
        flag[idx] = f ? 1 : 0;
    }
}

// flags = dilate^w(gradient flags) & covered & allowed, allowed =
// erode(covered, 1) (the driver's host rule for "gradient"); eta_scratch
// holds popcount(layer_mask) level-sized fp64 planes, scratch 3*ny*nx bytes.
extern "C" int mlamr_flags_gradient(mlamr_level lv, const double *state, mlamr_params prm, unsigned layer_mask,
                                    double tol, int dilate_w, uint8_t *flags, uint8_t *allowed, uint8_t *scratch,
                                    double *eta_scratch, void *stream) {
    cudaStream_t st = as_stream(stream);
    const int ny = lv.level_ny, nx = lv.level_nx;
    const int64_t n = (int64_t)ny * nx;
    if (n <= 0) return 0;
    const int nb = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
    uint8_t *a = scratch, *b = scratch + n, *bits = scratch + 2 * n;
    int rc = dispatch_m(prm.num_layers, [&](auto Mc) {
        constexpr int M = decltype(Mc)::value;
        k_grad_eta<M><<<nb, 256, 0, st>>>(lv, state, layer_mask, eta_scratch, bits);
    });
    if (rc) return rc;
    const int K = __builtin_popcount(layer_mask & ((1u << prm.num_layers) - 1u));
    k_grad_flags<<<nb, 256, 0, st>>>(eta_scratch, K, bits, ny, nx, lv.dx, lv.dy, tol, a);
    for (int w = 0; w < dilate_w; ++w) {
        k_morph3<<<nb, 256, 0, st>>>(a, b, ny, nx, 0);
        uint8_t *t = a; a = b; b = t;
    }
    k_covered<<<nb, 256, 0, st>>>(bits, b, n);
    k_morph3<<<nb, 256, 0, st>>>(b, allowed, ny, nx, 1);
    k_flag_mask<<<nb, 256, 0, st>>>(a, bits, allowed, n);
    cudaMemcpyAsync(flags, a, n, cudaMemcpyDeviceToDevice, st);
    return (int)cudaGetLastError();
}

// Sharded form of the gradient rule, in two halves around the all-reduce of
// the raw flags.  The raw half evaluates the rule on a rank's local pool
// (owned patches + shadows: every covered neighbour of an owned cell lies
// in a held sibling's refreshed interior ring) and keeps the flags of owned
// cells only; the finish half dilates the union and masks it with the
// GLOBAL coverage (0/1 map of the level's whole layout) and its erosion.
__global__ void k_flags_owned_only(const int32_t *own, int ny, int nx, const uint8_t *owned, uint8_t *flag) {
    const int64_t n = (int64_t)ny * nx;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int j = (int)(idx / nx), i = (int)(idx - (int64_t)j * nx);
        const int o = owner_at(own, nx, ny, i, j);
        if (o < 0 || !owned[o]) flag[idx] = 0;
    }
}

extern "C" int mlamr_flags_gradient_raw(mlamr_level lv, const double *state, mlamr_params prm, unsigned layer_mask,
                                        double tol, const uint8_t *owned_patches, uint8_t *raw, uint8_t *bits,
                                        double *eta_scratch, void *stream) {
    cudaStream_t st = as_stream(stream);
    const int ny = lv.level_ny, nx = lv.level_nx;
    const int64_t n = (int64_t)ny * nx;
    if (n <= 0) return 0;
    const int nb = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
    int rc = dispatch_m(prm.num_layers, [&](auto Mc) {
        constexpr int M = decltype(Mc)::value;
        k_grad_eta<M><<<nb, 256, 0, st>>>(lv, state, layer_mask, eta_scratch, bits);
    });
    if (rc) return rc;
    const int K = __builtin_popcount(layer_mask & ((1u << prm.num_layers) - 1u));
    k_grad_flags<<<nb, 256, 0, st>>>(eta_scratch, K, bits, ny, nx, lv.dx, lv.dy, tol, raw);
    if (owned_patches != nullptr) k_flags_owned_only<<<nb, 256, 0, st>>>(lv.own, ny, nx, owned_patches, raw);
    return (int)cudaGetLastError();
}

extern "C" int mlamr_flags_finish(const uint8_t *raw, const uint8_t *covered, int ny, int nx, int dilate_w,
                                  uint8_t *flags, uint8_t *allowed, uint8_t *scratch, void *stream) {
    cudaStream_t st = as_stream(stream);
    const int64_t n = (int64_t)ny * nx;
    if (n <= 0) return 0;
    const int nb = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
    uint8_t *a = scratch, *b = scratch + n, *bits = scratch + 2 * n;
    cudaError_t e = cudaMemcpyAsync(a, raw, n, cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return (int)e;
    for (int w = 0; w < dilate_w; ++w) {
        k_morph3<<<nb, 256, 0, st>>>(a, b, ny, nx, 0);
        uint8_t *t = a; a = b; b = t;
    }
    // coverage bits in the 0x80 convention of k_covered / k_flag_mask
    k_cov_bits<<<nb, 256, 0, st>>>(covered, bits, n);
    k_covered<<<nb, 256, 0, st>>>(bits, b, n);
    k_morph3<<<nb, 256, 0, st>>>(b, allowed, ny, nx, 1);
    k_flag_mask<<<nb, 256, 0, st>>>(a, bits, allowed, n);
    e = cudaMemcpyAsync(flags, a, n, cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return (int)e;
    return (int)cudaGetLastError();
}

// Byte fill of device memory (cudaMemsetAsync: a copy-engine memset, not a
// kernel): zero planes, -1 (0xff) owner maps and "all dry" speed bits.
extern "C" int mlamr_memset(void *ptr, int byte, long long nbytes, void *stream) {
    if (nbytes <= 0) return 0;
    return (int)cudaMemsetAsync(ptr, byte, (size_t)nbytes, as_stream(stream));
}

extern "C" int mlamr_version(void) { return 1; }

extern "C" const char *mlamr_build_info(void) {
    return "mlamr_b200 sm_100a fp64 -fmad=false";
}
