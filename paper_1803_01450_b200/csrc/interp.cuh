// Coarse-data gathering and the multilayer refinement operator, per fine
// cell.  Shared by the ghost fill (K2) and the regrid refinement (K3).
//
// gather (ghost.py:29-86): a coarse cell's data comes from the parent patch
// whose interior contains it (owner map), else -- when ghosts may be used --
// from the first patch in list order whose ghost frame contains it, else it
// is unavailable (zeros, avail = false).  With a blend, values are
// (1-theta)*old + theta*new (ghost.py:68-71).
//
// interpolate_state (refine.py:158-190): bottom-up layer march of the
// minmod-limited surface interpolation; slopes need the cell and both
// neighbours along an axis to be usable (avail & h_m > tol, refine.py:82-98,
// 148-153); momenta use the same mask and are zeroed where the recovered
// depth is dry.  Only the parent and its four edge neighbours matter
// (no cross terms, refine.py:136-137), so five gathered cells suffice.
#pragma once

#include "common.cuh"

namespace mlamr {

template <int M>
struct Coarse5 {
    // cells: 0 centre, 1 left (i-1), 2 right (i+1), 3 down (j-1), 4 up (j+1)
    double h[5][M], hu[5][M], hv[5][M], B[5];
    bool avail[5];
};

template <int M>
__device__ __forceinline__ void gather_cell(const mlamr_level &par, const double *new_state,
                                            const double *old_state, double theta,
                                            bool include_ghosts, int ci, int cj,
                                            Coarse5<M> &c, int slot) {
    int o = owner_at(par.own, par.level_nx, par.level_ny, ci, cj);
    if (o < 0 && include_ghosts) o = owner_at(par.gown, par.level_nx, par.level_ny, ci, cj);
    if (o < 0) {
        c.avail[slot] = false;
        c.B[slot] = 0.0;
#pragma unroll
        for (int m = 0; m < M; ++m) {
            c.h[slot][m] = 0.0;
            c.hu[slot][m] = 0.0;
            c.hv[slot][m] = 0.0;
        }
        return;
    }
    const int32_t *b = par.box + 4 * o;
    const int NX = b[2] - b[0] + 1 + 2 * MLAMR_G;
    const int64_t k = par.offset[o] + (int64_t)(cj - b[1] + MLAMR_G) * NX + (ci - b[0] + MLAMR_G);
    const int64_t FS = par.field_stride;
    c.avail[slot] = true;
    c.B[slot] = par.bathy[k];
    if (old_state == nullptr) {
#pragma unroll
        for (int m = 0; m < M; ++m) {
            c.h[slot][m] = new_state[m * FS + k];
            c.hu[slot][m] = new_state[(M + m) * FS + k];
            c.hv[slot][m] = new_state[(2 * M + m) * FS + k];
        }
    } else {
        const double w0 = 1.0 - theta;
#pragma unroll
        for (int m = 0; m < M; ++m) {
            c.h[slot][m] = (w0 * old_state[m * FS + k]) + (theta * new_state[m * FS + k]);
            c.hu[slot][m] = (w0 * old_state[(M + m) * FS + k]) + (theta * new_state[(M + m) * FS + k]);
            c.hv[slot][m] = (w0 * old_state[(2 * M + m) * FS + k]) + (theta * new_state[(2 * M + m) * FS + k]);
        }
    }
}

template <int M>
__device__ __forceinline__ void gather5(const mlamr_level &par, const double *new_state,
                                        const double *old_state, double theta,
                                        bool include_ghosts, int ci, int cj, Coarse5<M> &c) {
    gather_cell<M>(par, new_state, old_state, theta, include_ghosts, ci, cj, c, 0);
    gather_cell<M>(par, new_state, old_state, theta, include_ghosts, ci - 1, cj, c, 1);
    gather_cell<M>(par, new_state, old_state, theta, include_ghosts, ci + 1, cj, c, 2);
    gather_cell<M>(par, new_state, old_state, theta, include_ghosts, ci, cj - 1, c, 3);
    gather_cell<M>(par, new_state, old_state, theta, include_ghosts, ci, cj + 1, c, 4);
}

// Per-layer limited slopes of the parent (refine.py:82-98) for the surface
// and both momenta; the fine cell then evaluates (v + sx*offx) + sy*offy.
template <int M>
struct Slopes {
    double base[M][3], sx[M][3], sy[M][3];
};

template <int M>
__device__ __forceinline__ void parent_slopes(const Coarse5<M> &c, double tol, Slopes<M> &s) {
    // running bottom-up cumulative depth per gathered cell (state.py:56-61)
    double acc[5];
#pragma unroll
    for (int m = M - 1; m >= 0; --m) {
        bool use[5];
        double eta[5];
#pragma unroll
        for (int q = 0; q < 5; ++q) {
            acc[q] = (m == M - 1) ? c.h[q][m] : acc[q] + c.h[q][m];
            eta[q] = acc[q] + c.B[q];
            use[q] = c.avail[q] && (c.h[q][m] > tol);
        }
        const bool okx = use[1] && use[0] && use[2];
        const bool oky = use[3] && use[0] && use[4];
#pragma unroll
        for (int f = 0; f < 3; ++f) {
            double v0, vl, vr, vd, vu;
            if (f == 0) {
                v0 = eta[0]; vl = eta[1]; vr = eta[2]; vd = eta[3]; vu = eta[4];
            } else if (f == 1) {
                v0 = c.hu[0][m]; vl = c.hu[1][m]; vr = c.hu[2][m]; vd = c.hu[3][m]; vu = c.hu[4][m];
            } else {
                v0 = c.hv[0][m]; vl = c.hv[1][m]; vr = c.hv[2][m]; vd = c.hv[3][m]; vu = c.hv[4][m];
            }
            s.base[m][f] = v0;
            s.sx[m][f] = okx ? minmod(v0 - vl, vr - v0) : 0.0;
            s.sy[m][f] = oky ? minmod(v0 - vd, vu - v0) : 0.0;
        }
    }
}

// Layer march for one fine cell (refine.py:175-189).
template <int M>
__device__ __forceinline__ void fine_cell(const Slopes<M> &s, double offx, double offy,
                                          double fine_bathy, double tol, double *h, double *hu,
                                          double *hv) {
    double bhat = fine_bathy;
#pragma unroll
    for (int m = M - 1; m >= 0; --m) {
        const double eta = (s.base[m][0] + (s.sx[m][0] * offx)) + (s.sy[m][0] * offy);
        const double hh = np_max(0.0, eta - bhat);
        double uu = (s.base[m][1] + (s.sx[m][1] * offx)) + (s.sy[m][1] * offy);
        double vv = (s.base[m][2] + (s.sx[m][2] * offx)) + (s.sy[m][2] * offy);
        if (hh <= tol) {
            uu = 0.0;
            vv = 0.0;
        }
        h[m] = hh;
        hu[m] = uu;
        hv[m] = vv;
        bhat = bhat + hh;
    }
}

// refine._parent_indexing offsets (refine.py:114-115)
__device__ __forceinline__ double child_offset(int f, int p, int r) {
    return ((double)(f - p * r) + 0.5) / (double)r - 0.5;
}

}  // namespace mlamr
