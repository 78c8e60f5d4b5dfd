// K1: batched multilayer patch step (physics.step_patch, physics.py:330-386)
// and K6 per-patch observed max wave speed (physics.py:261-278).
//
// One CTA advances one 16x32 interior tile of one patch through BOTH
// dimensionally split sweeps (physics.py:353-358).  The tile is staged in
// shared memory with a one-cell halo: the step reads ghost width 1 only
// (SURVEY.md App. C probe 3), and the first sweep is evaluated on the halo
// lines too, exactly as the reference's `full=True` first sweep covers the
// ghost rows.  Per-interface fluxes are computed once per tile; the second
// sweep consumes the first sweep's halo lines from shared memory.  The
// stepped interior is written out of place (src -> dst): neighbouring tiles
// read the pre-step halo, and the untouched src buffer doubles as the
// driver's time-interpolation stash (driver.py:260-264).
//
// Arithmetic order follows physics._sweep (physics.py:101-169) and
// _layer_inputs (physics.py:193-212) operation by operation; the library is
// compiled with -fmad=false, so results are bit-identical to the numba
// reference (which does not contract either).

#include <cstdio>

#include "common.cuh"

namespace mlamr {

constexpr int TX = 32;
constexpr int TY = 16;
constexpr int PX = TX + 2;
constexpr int PY = TY + 2;
constexpr int NPAD = PX * PY;
constexpr int NFLUX = PY * (PX - 1);  // >= PX * (PY - 1)
constexpr int NT = 256;

template <int M>
struct StepSmem {
    double S[3 * M + 1][NPAD];  // h_0..h_{M-1}, hu_.., hv_.., B
    double cw[NPAD];
    double eb[M > 1 ? M - 1 : 1][NPAD];  // eta_{m+1} = B + h_{M-1} + ... + h_{m+1}
    double src[M > 1 ? M : 1][NPAD];
    double u[NPAD];
    double v[NPAD];
    double vel[NPAD];
    double F[5][NFLUX];  // Fh, Fm, Fv, hsL, hsR of one layer
    double red[NT];
    long long redi[NT];
    unsigned char cowet[NPAD];
    unsigned char wetcol[NPAD];
};

template <int DIR>
__device__ __forceinline__ int cidx(int o, int a) {
    return DIR == 0 ? o * PX + a : a * PX + o;
}
template <int DIR>
__device__ __forceinline__ int fidx(int o, int a) {
    return DIR == 0 ? o * (PX - 1) + a : a * PX + o;
}

// One directional sweep of all layers over the staged tile
// (physics._sweep_x / _sweep_y with _layer_inputs).
// DIR 0 = x (along columns), 1 = y (along rows).  FIRST: all halo lines
// (the reference's full=True); else the interior lines only.
template <int M, int DIR, bool FIRST>
__device__ void sweep_tile(StepSmem<M> &s, int ny2, int nx2, double dt, double d,
                           const mlamr_params &prm, const double (&rr)[4][4]) {
    const int t = threadIdx.x;
    const int n_along = DIR == 0 ? nx2 : ny2;
    const int n_outer = DIR == 0 ? ny2 : nx2;
    const int o0 = FIRST ? 0 : 1;
    const int o1 = FIRST ? n_outer : n_outer - 1;
    const int no = o1 - o0;
    const double g = prm.gravity;
    const double tol = prm.dry_tolerance;
    const double lam = dt / d;
    const double *B = s.S[3 * M];

    // Phase D: per-cell layer inputs on the pre-sweep state of this direction.
    for (int idx = t; idx < no * n_along; idx += NT) {
        const int o = o0 + idx / n_along;
        const int a = idx - (idx / n_along) * n_along;
        const int k = cidx<DIR>(o, a);
        double hs = 0.0;
#pragma unroll
        for (int m = 0; m < M; ++m) hs = hs + s.S[m][k];
        s.cw[k] = sqrt(g * np_max(hs, 0.0));
        if (FIRST) s.wetcol[k] = hs > tol;
        if (M > 1) {
            bool w = true;
#pragma unroll
            for (int m = 0; m < M; ++m) w = w && (s.S[m][k] > tol);
            s.cowet[k] = w;
            double e = B[k];
#pragma unroll
            for (int m = M - 1; m >= 1; --m) {
                e = e + s.S[m][k];
                s.eb[m - 1][k] = e;
            }
        } else {
            s.cowet[k] = 1;
        }
    }
    __syncthreads();

    // Phase S: coupling sources on the updated cells (physics.py:208-211).
    if (M > 1) {
        const int nu = n_along - 2;
        for (int idx = t; idx < no * nu; idx += NT) {
            const int o = o0 + idx / nu;
            const int a = 1 + idx - (idx / nu) * nu;
            const int k = cidx<DIR>(o, a);
            const int km = cidx<DIR>(o, a - 1);
            const int kp = cidx<DIR>(o, a + 1);
            const bool wm = s.cowet[km] && s.cowet[k];
            const bool wp = s.cowet[k] && s.cowet[kp];
#pragma unroll
            for (int m = 0; m < M; ++m) {
                double acc = 0.0;
                bool has = false;
                if (m < M - 1) {
                    const double *f = s.eb[m];
                    const double dm = wm ? f[k] - f[km] : 0.0;
                    const double dp = wp ? f[kp] - f[k] : 0.0;
                    const double grad = 0.5 * (dp + dm);
                    acc = (((-g) * s.S[m][k]) * grad) / d;
                    has = true;
                }
#pragma unroll
                for (int kk = 0; kk < m; ++kk) {
                    const double *f = s.S[kk];
                    const double dm = wm ? f[k] - f[km] : 0.0;
                    const double dp = wp ? f[kp] - f[k] : 0.0;
                    const double grad = 0.5 * (dp + dm);
                    const double term = ((((-rr[kk][m]) * g) * s.S[m][k]) * grad) / d;
                    acc = has ? acc + term : term;
                    has = true;
                }
                s.src[m][k] = acc;
            }
        }
    }
    // (the syncthreads at the top of the layer loop orders Phase S)

#pragma unroll 1
    for (int m = 0; m < M; ++m) {
        double *H = s.S[m];
        double *HN = DIR == 0 ? s.S[M + m] : s.S[2 * M + m];
        double *HT = DIR == 0 ? s.S[2 * M + m] : s.S[M + m];
        const bool bottom = (m == M - 1);
        const double *Zf = bottom ? B : s.eb[m < M - 1 ? m : 0];
        __syncthreads();
        // Phase U: velocities once per cell (the reference divides twice per
        // cell, once as a left and once as a right state: same value).
        for (int idx = t; idx < no * n_along; idx += NT) {
            const int o = o0 + idx / n_along;
            const int a = idx - (idx / n_along) * n_along;
            const int k = cidx<DIR>(o, a);
            const double h = H[k];
            const bool wet = h > tol;
            const double u = wet ? HN[k] / h : 0.0;
            const double v = wet ? HT[k] / h : 0.0;
            s.u[k] = u;
            s.v[k] = v;
            if (FIRST) {
                const int r = DIR == 0 ? o : a;
                const int c = DIR == 0 ? a : o;
                if (r >= 1 && r < ny2 - 1 && c >= 1 && c < nx2 - 1) {
                    // observed_max_speed (physics.py:269-276): |hu|/h == |hu/h|
                    const double x = wet ? np_max(fabs(u), fabs(v)) : 0.0;
                    s.vel[k] = (m == 0) ? np_max(0.0, x) : np_max(s.vel[k], x);
                }
            }
        }
        __syncthreads();
        // Phase F: one HLL flux per interface (physics.py:101-161).
        const int ni = n_along - 1;
        for (int idx = t; idx < no * ni; idx += NT) {
            const int o = o0 + idx / ni;
            const int a = idx - (idx / ni) * ni;
            const int kl = cidx<DIR>(o, a);
            const int kr = cidx<DIR>(o, a + 1);
            const int fi = fidx<DIR>(o, a);
            const double hl = H[kl];
            const double hr = H[kr];
            double Zl, Zr;
            if (s.cowet[kl] && s.cowet[kr]) {
                Zl = bottom ? B[kl] : 0.0;
                Zr = bottom ? B[kr] : 0.0;
            } else {
                Zl = Zf[kl];
                Zr = Zf[kr];
            }
            const double ul = s.u[kl];
            const double ur = s.u[kr];
            const double Zs = Zl > Zr ? Zl : Zr;
            double hL = (hl + Zl) - Zs;
            if (hL < 0.0) hL = 0.0;
            double hR = (hr + Zr) - Zs;
            if (hR < 0.0) hR = 0.0;
            s.F[3][fi] = hL;
            s.F[4][fi] = hR;
            if (hL <= 0.0 && hR <= 0.0) {
                s.F[0][fi] = 0.0;
                s.F[1][fi] = 0.0;
                s.F[2][fi] = 0.0;
                continue;
            }
            const double cl = s.cw[kl];
            const double cr = s.cw[kr];
            const double sl1 = ul - cl, sl2 = ur - cr;
            const double SL = sl1 < sl2 ? sl1 : sl2;
            const double sr1 = ul + cl, sr2 = ur + cr;
            const double SR = sr1 > sr2 ? sr1 : sr2;
            const double FLh = hL * ul;
            const double FRh = hR * ur;
            const double FLm = ((hL * ul) * ul) + (((0.5 * g) * hL) * hL);
            const double FRm = ((hR * ur) * ur) + (((0.5 * g) * hR) * hR);
            double fh, fm;
            if (SL >= 0.0) {
                fh = FLh;
                fm = FLm;
            } else if (SR <= 0.0) {
                fh = FRh;
                fm = FRm;
            } else {
                const double den = SR - SL;
                double djump;
                if (hL > 0.0 && hR > 0.0) {
                    const double Bl = bottom ? B[kl] : Zf[kl];
                    const double Br = bottom ? B[kr] : Zf[kr];
                    djump = (hr + Br) - (hl + Bl);
                } else {
                    djump = hR - hL;
                }
                fh = (((SR * FLh) - (SL * FRh)) + ((SL * SR) * djump)) / den;
                fm = (((SR * FLm) - (SL * FRm)) + ((SL * SR) * ((hR * ur) - (hL * ul)))) / den;
            }
            s.F[0][fi] = fh;
            s.F[1][fi] = fm;
            double fv;
            if (fh > 0.0)
                fv = fh * s.v[kl];
            else if (fh < 0.0)
                fv = fh * s.v[kr];
            else
                fv = 0.0;
            s.F[2][fi] = fv;
        }
        __syncthreads();
        // Phase C: conservative update + pressure correction (+ source).
        const int nu = n_along - 2;
        for (int idx = t; idx < no * nu; idx += NT) {
            const int o = o0 + idx / nu;
            const int a = 1 + idx - (idx / nu) * nu;
            const int k = cidx<DIR>(o, a);
            const int fl = fidx<DIR>(o, a - 1);
            const int fr = fidx<DIR>(o, a);
            H[k] = H[k] - lam * (s.F[0][fr] - s.F[0][fl]);
            double hn = (HN[k] - lam * (s.F[1][fr] - s.F[1][fl])) -
                        (((lam * 0.5) * g) * ((s.F[4][fl] * s.F[4][fl]) - (s.F[3][fr] * s.F[3][fr])));
            if (M > 1) hn = hn + dt * s.src[m][k];
            HN[k] = hn;
            HT[k] = HT[k] - lam * (s.F[2][fr] - s.F[2][fl]);
        }
    }
    __syncthreads();
}

template <int M, bool YFIRST>
__global__ void __launch_bounds__(NT) k_step(mlamr_level lv, const double *__restrict__ src,
                                             double *__restrict__ dst,
                                             const int32_t *__restrict__ tiles, double dt,
                                             mlamr_params prm, long long *speed_bits,
                                             double *tile_acc, const int32_t *status) {
    if (status != nullptr && *status != 0) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    StepSmem<M> &s = *reinterpret_cast<StepSmem<M> *>(smem_raw);
    const int t = threadIdx.x;
    const int tile = blockIdx.x;
    const int p = tiles[3 * tile];
    const int tj0 = tiles[3 * tile + 1];
    const int ti0 = tiles[3 * tile + 2];
    const PatchView pv = patch_view(lv, p);
    const int ty = min(TY, pv.ny - tj0);
    const int tx = min(TX, pv.nx - ti0);
    const int ny2 = ty + 2, nx2 = tx + 2;
    const int64_t FS = lv.field_stride;
    const int64_t base = pv.off + (int64_t)(tj0 + 1) * pv.NX + (ti0 + 1);

    double rr[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) rr[a][b] = (a < M && b < M) ? prm.densities[a] / prm.densities[b] : 0.0;

    // stage the padded tile: 3M state planes + bathymetry
    const int npad = ny2 * nx2;
#pragma unroll 1
    for (int q = 0; q < 3 * M + 1; ++q) {
        const double *g = (q < 3 * M) ? src + q * FS : lv.bathy;
        for (int idx = t; idx < npad; idx += NT) {
            const int r = idx / nx2;
            const int c = idx - r * nx2;
            s.S[q][r * PX + c] = __ldg(g + base + (int64_t)r * pv.NX + c);
        }
    }
    __syncthreads();

    if (YFIRST)
        sweep_tile<M, 1, true>(s, ny2, nx2, dt, lv.dy, prm, rr);
    else
        sweep_tile<M, 0, true>(s, ny2, nx2, dt, lv.dx, prm, rr);

    // observed max speed of the pre-step interior (vel from the first sweep's
    // Phase U, cw/wetcol from its Phase D): speed = vel + sqrt(g*max(H,0))
    {
        double best = -1.0;
        bool any = false;
        for (int idx = t; idx < ty * tx; idx += NT) {
            const int r = 1 + idx / tx;
            const int c = 1 + idx - (idx / tx) * tx;
            const int k = r * PX + c;
            if (!s.wetcol[k]) continue;
            const double sp = s.vel[k] + s.cw[k];
            best = any ? np_max(best, sp) : sp;
            any = true;
        }
        // block max (NaN-propagating); -1 marks "no wet column"
        s.red[t] = any ? best : -1.0;
        __syncthreads();
        for (int st = NT / 2; st > 0; st >>= 1) {
            if (t < st) {
                const double a = s.red[t], b = s.red[t + st];
                s.red[t] = (a < 0.0) ? b : ((b < 0.0) ? a : np_max(a, b));
            }
            __syncthreads();
        }
        if (t == 0 && !(s.red[0] < 0.0)) {
            double v = s.red[0];
            long long bits = (v != v) ? 0x7ff8000000000000LL : __double_as_longlong(v);
            atomicMax(speed_bits + p, bits);
        }
        __syncthreads();
    }

    if (YFIRST)
        sweep_tile<M, 0, false>(s, ny2, nx2, dt, lv.dx, prm, rr);
    else
        sweep_tile<M, 1, false>(s, ny2, nx2, dt, lv.dy, prm, rr);

    // post-processing on the tile interior (physics.py:360-376)
    const double tol = prm.dry_tolerance;
    double negs[M];
#pragma unroll
    for (int m = 0; m < M; ++m) negs[m] = 0.0;
    long long fixes = 0, repairs = 0;
    const double coef = prm.gravity * (1.0 - rr[0][1]);
    for (int idx = t; idx < ty * tx; idx += NT) {
        const int r = 1 + idx / tx;
        const int c = 1 + idx - (idx / tx) * tx;
        const int k = r * PX + c;
        double h[M], hu[M], hv[M];
#pragma unroll
        for (int m = 0; m < M; ++m) {
            h[m] = s.S[m][k];
            hu[m] = s.S[M + m][k];
            hv[m] = s.S[2 * M + m][k];
            const double neg = np_min(h[m], 0.0);
            negs[m] = negs[m] + neg;
            if (neg < 0.0) h[m] = 0.0;
        }
        if (M == 2) {  // _blend_shear (physics.py:292-327)
            const double h1 = h[0], h2 = h[1 % M];
            if (h1 > tol && h2 > tol) {
                const double hu1 = hu[0], hu2 = hu[1 % M], hv1 = hv[0], hv2 = hv[1 % M];
                const double u1 = hu1 / h1, u2 = hu2 / h2, v1 = hv1 / h1, v2 = hv2 / h2;
                const double du = u1 - u2, dv = v1 - v2;
                const double shear2 = (du * du) + (dv * dv);
                const double bound = coef * (h1 + h2);
                if (shear2 > bound) {
                    ++fixes;
                    const double alpha = sqrt(bound / shear2);
                    const double htot = h1 + h2;
                    const double umean = (hu1 + hu2) / htot;
                    const double vmean = (hv1 + hv2) / htot;
                    hu[0] = h1 * (umean + alpha * (u1 - umean));
                    hu[1 % M] = h2 * (umean + alpha * (u2 - umean));
                    hv[0] = h1 * (vmean + alpha * (v1 - vmean));
                    hv[1 % M] = h2 * (vmean + alpha * (v2 - vmean));
                }
            }
        }
        // restore_wet_prefix (state.py:125-145), then zero_dry_momenta (:104-110)
#pragma unroll
        for (int m = 1; m < M; ++m) {
            if (h[m] > tol && h[m - 1] <= tol) {
                ++repairs;
                h[m - 1] = h[m - 1] + h[m];
                hu[m - 1] = hu[m - 1] + hu[m];
                hv[m - 1] = hv[m - 1] + hv[m];
                h[m] = 0.0;
                hu[m] = 0.0;
                hv[m] = 0.0;
            }
        }
        const int64_t gaddr = base + (int64_t)r * pv.NX + c;
#pragma unroll
        for (int m = 0; m < M; ++m) {
            if (h[m] <= tol) {
                hu[m] = 0.0;
                hv[m] = 0.0;
            }
            dst[m * FS + gaddr] = h[m];
            dst[(M + m) * FS + gaddr] = hu[m];
            dst[(2 * M + m) * FS + gaddr] = hv[m];
        }
    }
    // per-tile partials (fixed-order tree sums)
    double *acc = tile_acc + (int64_t)tile * (M + 2);
#pragma unroll
    for (int m = 0; m < M; ++m) {
        const double sm = block_sum<NT>(negs[m], s.red);
        if (t == 0) acc[m] = sm;
    }
    const long long fx = block_sum_ll<NT>(fixes, s.redi);
    const long long rp = block_sum_ll<NT>(repairs, s.redi);
    if (t == 0) {
        acc[M] = (double)fx;
        acc[M + 1] = (double)rp;
    }
}

// K6: observed max speed per patch without stepping (stable_dt, level 1 dt).
template <int M>
__global__ void __launch_bounds__(NT) k_max_speed(mlamr_level lv, const double *__restrict__ st,
                                                  const int32_t *__restrict__ tiles,
                                                  mlamr_params prm, long long *speed_bits) {
    __shared__ double red[NT];
    const int t = threadIdx.x;
    const int tile = blockIdx.x;
    const int p = tiles[3 * tile];
    const int tj0 = tiles[3 * tile + 1];
    const int ti0 = tiles[3 * tile + 2];
    const PatchView pv = patch_view(lv, p);
    const int ty = min(TY, pv.ny - tj0);
    const int tx = min(TX, pv.nx - ti0);
    const int64_t FS = lv.field_stride;
    const double tol = prm.dry_tolerance;
    double best = -1.0;
    bool any = false;
    for (int idx = t; idx < ty * tx; idx += NT) {
        const int r = idx / tx;
        const int c = idx - r * tx;
        const int64_t k = pv.off + (int64_t)(tj0 + MLAMR_G + r) * pv.NX + (ti0 + MLAMR_G + c);
        double hs = 0.0, vel = 0.0;
#pragma unroll
        for (int m = 0; m < M; ++m) {
            const double h = st[m * FS + k];
            hs = hs + h;
            const bool wet = h > tol;
            const double hm = wet ? h : 1.0;
            const double um = fabs(st[(M + m) * FS + k]) / hm;
            const double vm = fabs(st[(2 * M + m) * FS + k]) / hm;
            vel = np_max(vel, wet ? np_max(um, vm) : 0.0);
        }
        if (!(hs > tol)) continue;
        const double sp = vel + sqrt(prm.gravity * np_max(hs, 0.0));
        best = any ? np_max(best, sp) : sp;
        any = true;
    }
    red[t] = any ? best : -1.0;
    __syncthreads();
    for (int s2 = NT / 2; s2 > 0; s2 >>= 1) {
        if (t < s2) {
            const double a = red[t], b = red[t + s2];
            red[t] = (a < 0.0) ? b : ((b < 0.0) ? a : np_max(a, b));
        }
        __syncthreads();
    }
    if (t == 0 && !(red[0] < 0.0)) {
        const double v = red[0];
        const long long bits = (v != v) ? 0x7ff8000000000000LL : __double_as_longlong(v);
        atomicMax(speed_bits + p, bits);
    }
}

// CFL guard + deterministic reduction of the step partials.
template <int M>
__global__ void __launch_bounds__(NT) k_step_finalize(mlamr_level lv, const double *__restrict__ src,
                                                      double *__restrict__ dst,
                                                      const int32_t *__restrict__ tiles,
                                                      int n_tiles, double dt,
                                                      const long long *speed_bits,
                                                      const double *tile_acc, double *acc,
                                                      int32_t *status, int32_t *bad_patch) {
    __shared__ double red[NT];
    __shared__ int viol;
    const int t = threadIdx.x;
    if (*status != 0) return;
    const int K = M + 2;
    const double area = lv.dx * lv.dy;
    for (int q = 0; q < K; ++q) {
        double v = 0.0;
        for (int i = t; i < n_tiles; i += NT) v = v + tile_acc[(int64_t)i * K + q];
        const double sm = block_sum<NT>(v, red);
        // clipped mass = -(sum of negative depths) * cell area (physics.py:360-362)
        if (t == 0) acc[q] = acc[q] + (q < M ? (-sm) * area : sm);
    }
    const double dmin = lv.dx < lv.dy ? lv.dx : lv.dy;
    if (t == 0) viol = 0;
    __syncthreads();
    for (int p = t; p < lv.num_patches; p += NT) {
        const long long b = speed_bits[p];
        if (b < 0) continue;
        const double sp = __longlong_as_double(b);
        if ((sp * dt) / dmin > 1.0) {
            atomicOr(&viol, 1);
            atomicMin(bad_patch, p);
        }
    }
    __syncthreads();
    if (!viol) return;
    // restore every violating patch's interior (the reference raises before
    // touching it, physics.py:342-347)
    const int64_t FS = lv.field_stride;
    for (int p = 0; p < lv.num_patches; ++p) {
        const long long b = speed_bits[p];
        if (b < 0) continue;
        const double sp = __longlong_as_double(b);
        if (!((sp * dt) / dmin > 1.0)) continue;
        const PatchView pv = patch_view(lv, p);
        for (int idx = t; idx < pv.nx * pv.ny; idx += NT) {
            const int r = idx / pv.nx, c = idx - r * pv.nx;
            const int64_t k = pv.off + (int64_t)(r + MLAMR_G) * pv.NX + (c + MLAMR_G);
            for (int q = 0; q < 3 * M; ++q) dst[q * FS + k] = src[q * FS + k];
        }
    }
    if (t == 0) atomicOr(status, MLAMR_ST_CFL);
}

template <int M>
static int launch_step(const mlamr_level &lv, const double *src, double *dst,
                       const int32_t *tiles, int n_tiles, double dt, int y_first,
                       const mlamr_params &prm, long long *speed_bits, double *tile_acc,
                       const int32_t *status, cudaStream_t st) {
    const size_t smem = sizeof(StepSmem<M>);
    static bool configured[2] = {false, false};
    if (!configured[y_first ? 1 : 0]) {
        cudaError_t e;
        if (y_first)
            e = cudaFuncSetAttribute(k_step<M, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        else
            e = cudaFuncSetAttribute(k_step<M, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return (int)e;
        configured[y_first ? 1 : 0] = true;
    }
    if (n_tiles <= 0) return 0;
    if (y_first)
        k_step<M, true><<<n_tiles, NT, smem, st>>>(lv, src, dst, tiles, dt, prm, speed_bits, tile_acc, status);
    else
        k_step<M, false><<<n_tiles, NT, smem, st>>>(lv, src, dst, tiles, dt, prm, speed_bits, tile_acc, status);
    return (int)cudaGetLastError();
}

}  // namespace mlamr

using namespace mlamr;

extern "C" int mlamr_step(mlamr_level lv, const double *src_state, double *dst_state,
                          const int32_t *tiles, int n_tiles, double dt, int y_first,
                          mlamr_params prm, long long *speed_bits, double *tile_acc,
                          const int32_t *status, void *stream) {
    cudaStream_t st = as_stream(stream);
    switch (prm.num_layers) {
        case 1: return launch_step<1>(lv, src_state, dst_state, tiles, n_tiles, dt, y_first, prm, speed_bits, tile_acc, status, st);
        case 2: return launch_step<2>(lv, src_state, dst_state, tiles, n_tiles, dt, y_first, prm, speed_bits, tile_acc, status, st);
        case 3: return launch_step<3>(lv, src_state, dst_state, tiles, n_tiles, dt, y_first, prm, speed_bits, tile_acc, status, st);
        default: return -1;
    }
}

extern "C" int mlamr_step_finalize(mlamr_level lv, const double *src_state, double *dst_state,
                                   const int32_t *tiles, int n_tiles, double dt,
                                   mlamr_params prm, const long long *speed_bits,
                                   const double *tile_acc, double *acc, int32_t *status,
                                   int32_t *bad_patch, void *stream) {
    cudaStream_t st = as_stream(stream);
    switch (prm.num_layers) {
        case 1: k_step_finalize<1><<<1, NT, 0, st>>>(lv, src_state, dst_state, tiles, n_tiles, dt, speed_bits, tile_acc, acc, status, bad_patch); break;
        case 2: k_step_finalize<2><<<1, NT, 0, st>>>(lv, src_state, dst_state, tiles, n_tiles, dt, speed_bits, tile_acc, acc, status, bad_patch); break;
        case 3: k_step_finalize<3><<<1, NT, 0, st>>>(lv, src_state, dst_state, tiles, n_tiles, dt, speed_bits, tile_acc, acc, status, bad_patch); break;
        default: return -1;
    }
    return (int)cudaGetLastError();
}

extern "C" int mlamr_max_speed_tiles(mlamr_level lv, const double *state, const int32_t *tiles,
                                     int n_tiles, mlamr_params prm, long long *speed_bits,
                                     void *stream) {
    cudaStream_t st = as_stream(stream);
    if (n_tiles <= 0) return 0;
    switch (prm.num_layers) {
        case 1: k_max_speed<1><<<n_tiles, NT, 0, st>>>(lv, state, tiles, prm, speed_bits); break;
        case 2: k_max_speed<2><<<n_tiles, NT, 0, st>>>(lv, state, tiles, prm, speed_bits); break;
        case 3: k_max_speed<3><<<n_tiles, NT, 0, st>>>(lv, state, tiles, prm, speed_bits); break;
        default: return -1;
    }
    return (int)cudaGetLastError();
}
