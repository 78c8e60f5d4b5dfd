/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's per-patch numerical operators
 * (arxiv/paper_1803_01450, package `mlamr`).  Only tests/, the
 * `__graft_entry__.smoke()` checker and bench.py's cpu_baseline / reference
 * arm may load this library; the product path never does.
 *
 * Every routine restates one reference function in IEEE fp64 with the exact
 * left-to-right operation order of the Python/numba source (compiled with
 * -ffp-contract=off so no FMA contraction happens).  File:line citations are
 * relative to /root/reference/pkg/src/mlamr/.
 *
 * Array layout (same as the reference Patch, mesh.py:181-186):
 *   h, hu, hv : [M][NY][NX] row-major, x fastest, layer 0 = top
 *   bathy     : [NY][NX]
 * NY = ny + 2g, NX = nx + 2g, g = ghost width.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_CFL 3
#define ORC_GEOMETRY 4
#define ORC_ALLOC 9

/* numpy elementwise semantics (observed with numpy 2.3): ties return the
 * second operand, NaN propagates.  np.maximum(a, b), np.minimum(a, b). */
static inline double np_maximum(double a, double b) {
    if (a != a) return a;
    if (b != b) return b;
    return a > b ? a : b;
}
static inline double np_minimum(double a, double b) {
    if (a != a) return a;
    if (b != b) return b;
    return a < b ? a : b;
}

/* numpy add.reduce over the layer axis starts from +0.0
 * (physics.py:172-173 `patch.h.sum(axis=0)`). */
static inline double layer_sum(const double *h, long plane, long k, int M) {
    double s = 0.0;
    for (int m = 0; m < M; ++m) s = s + h[m * plane + k];
    return s;
}

/* ---------------------------------------------------------------------- */
/* physics._sweep (physics.py:71-169): one layer, one direction, in place.  */
/* The line being swept is addressed with strides so the y sweep needs no  */
/* transposed copies (physics.py:234-255 transposes; values are identical). */
/* ---------------------------------------------------------------------- */
static void sweep_layer(double *h, double *hn, double *ht,
                        const double *Zc, const double *Zf, const double *Bh,
                        const uint8_t *cowet, const double *cw,
                        long s_out, long s_in, int n_in, int gw,
                        double lam, double g, double dry, int j0, int j1,
                        double *scratch)
{
    double *Fh = scratch, *Fm = scratch + n_in, *Fv = scratch + 2 * n_in;
    double *hsL = scratch + 3 * n_in, *hsR = scratch + 4 * n_in;
    for (int j = j0; j < j1; ++j) {
        const long base = (long)j * s_out;
        for (int i = gw - 1; i < n_in - gw; ++i) {
            const long a = base + (long)i * s_in, b = a + s_in;
            double hl = h[a], hr = h[b];
            double Zl, Zr;
            if (cowet[a] && cowet[b]) { Zl = Zc[a]; Zr = Zc[b]; }
            else { Zl = Zf[a]; Zr = Zf[b]; }
            double ul = hl > dry ? hn[a] / hl : 0.0;
            double ur = hr > dry ? hn[b] / hr : 0.0;
            double Zs = Zl > Zr ? Zl : Zr;
            double hL = (hl + Zl) - Zs;
            if (hL < 0.0) hL = 0.0;
            double hR = (hr + Zr) - Zs;
            if (hR < 0.0) hR = 0.0;
            hsL[i] = hL;
            hsR[i] = hR;
            if (hL <= 0.0 && hR <= 0.0) {
                Fh[i] = 0.0; Fm[i] = 0.0; Fv[i] = 0.0;
                continue;
            }
            double cl = cw[a], cr = cw[b];
            double sl1 = ul - cl, sl2 = ur - cr;
            double SL = sl1 < sl2 ? sl1 : sl2;
            double sr1 = ul + cl, sr2 = ur + cr;
            double SR = sr1 > sr2 ? sr1 : sr2;
            double FLh = hL * ul, FRh = hR * ur;
            double FLm = ((hL * ul) * ul) + (((0.5 * g) * hL) * hL);
            double FRm = ((hR * ur) * ur) + (((0.5 * g) * hR) * hR);
            double fh, fm;
            if (SL >= 0.0) { fh = FLh; fm = FLm; }
            else if (SR <= 0.0) { fh = FRh; fm = FRm; }
            else {
                double den = SR - SL;
                double djump;
                if (hL > 0.0 && hR > 0.0) djump = (hr + Bh[b]) - (hl + Bh[a]);
                else djump = hR - hL;
                fh = (((SR * FLh) - (SL * FRh)) + ((SL * SR) * djump)) / den;
                fm = (((SR * FLm) - (SL * FRm)) + ((SL * SR) * ((hR * ur) - (hL * ul)))) / den;
            }
            Fh[i] = fh;
            Fm[i] = fm;
            double vl = hl > dry ? ht[a] / hl : 0.0;
            double vr = hr > dry ? ht[b] / hr : 0.0;
            if (fh > 0.0) Fv[i] = fh * vl;
            else if (fh < 0.0) Fv[i] = fh * vr;
            else Fv[i] = 0.0;
        }
        for (int i = gw; i < n_in - gw; ++i) {
            const long a = base + (long)i * s_in;
            h[a] = h[a] - lam * (Fh[i] - Fh[i - 1]);
            hn[a] = (hn[a] - lam * (Fm[i] - Fm[i - 1]))
                    - (((lam * 0.5) * g) * ((hsR[i - 1] * hsR[i - 1]) - (hsL[i] * hsL[i])));
            ht[a] = ht[a] - lam * (Fv[i] - Fv[i - 1]);
        }
    }
}

/* physics._masked_centered_grad (physics.py:176-190) along the sweep axis. */
static void masked_grad(const double *f, const uint8_t *cowet, double *grad,
                        long s_out, long s_in, int n_out, int n_in)
{
    for (int j = 0; j < n_out; ++j) {
        const long base = (long)j * s_out;
        grad[base] = 0.0;
        grad[base + (long)(n_in - 1) * s_in] = 0.0;
        for (int k = 1; k < n_in - 1; ++k) {
            long c = base + (long)k * s_in;
            double dm = (cowet[c - s_in] && cowet[c]) ? f[c] - f[c - s_in] : 0.0;
            double dp = (cowet[c] && cowet[c + s_in]) ? f[c + s_in] - f[c] : 0.0;
            grad[c] = 0.5 * (dp + dm);
        }
    }
}

typedef struct {
    int M;
    double g;
    double tol;
    const double *rho; /* densities, top to bottom */
} orc_params;

/*
 * _layer_inputs + _sweep_x/_sweep_y (physics.py:193-258) for one direction.
 * axis 1 = x (sweep along i), axis 0 = y (sweep along j).
 * M = 1 and M = 2 follow the reference exactly.  M >= 3 is this build's
 * generalisation (the reference raises IndexError, physics.py:223): layer m
 * < M-1 reconstructs against (Zc = 0, Zf = Bhat = eta_{m+1}) with source
 * -g h_m grad(eta_{m+1}); every layer m > 0 also receives
 * sum_k<m -(rho_k/rho_m) g h_m grad(h_k); cowet = all layers wet.
 */
static int sweep_dir(int axis, int NY, int NX, double *h, double *hu, double *hv,
                     const double *B, double dt, double dxdir, orc_params p,
                     int full, int gw, double *work)
{
    const int M = p.M;
    const long plane = (long)NY * NX;
    long s_out, s_in; int n_out, n_in;
    if (axis == 1) { s_out = NX; s_in = 1; n_out = NY; n_in = NX; }
    else { s_out = 1; s_in = NX; n_out = NX; n_in = NY; }
    const int j0 = full ? 0 : gw, j1 = full ? n_out : n_out - gw;
    const double lam = dt / dxdir;

    double *cw = work;                    /* plane */
    double *zeros = cw + plane;           /* plane */
    double *eta_below = zeros + plane;    /* (M-1) planes: eta_{m+1} */
    double *src = eta_below + (M > 1 ? (M - 1) : 0) * plane;   /* M planes */
    double *grad = src + (long)M * plane;                      /* plane */
    double *scratch = grad + plane;                            /* 5*max(NX,NY) */
    uint8_t *cowet = (uint8_t *)(scratch + 5 * (NX > NY ? NX : NY));

    for (long k = 0; k < plane; ++k) {
        double s = layer_sum(h, plane, k, M);
        cw[k] = sqrt(p.g * np_maximum(s, 0.0));
        zeros[k] = 0.0;
        if (M == 1) cowet[k] = 1;
        else {
            uint8_t w = 1;
            for (int m = 0; m < M; ++m) w = w && (h[m * plane + k] > p.tol);
            cowet[k] = w;
        }
    }
    /* eta_{m+1} = B + h_{M-1} + ... + h_{m+1}; M=2: eta2 = B + h[1]
     * (physics.py:207).  Built bottom-up from the bed. */
    if (M > 1) {
        for (long k = 0; k < plane; ++k) {
            double e = B[k];
            for (int m = M - 1; m >= 1; --m) {
                e = e + h[m * plane + k];
                eta_below[(m - 1) * plane + k] = e;
            }
        }
    }
    /* sources on the pre-sweep state of this direction (physics.py:208-211) */
    if (M > 1) {
        for (int m = 0; m < M; ++m) {
            double *sm = src + m * plane;
            for (long k = 0; k < plane; ++k) sm[k] = 0.0;
            int nterms = 0;
            if (m < M - 1) {
                masked_grad(eta_below + (long)m * plane, cowet, grad, s_out, s_in, n_out, n_in);
                for (long k = 0; k < plane; ++k) {
                    double t = (((-p.g) * h[m * plane + k]) * grad[k]) / dxdir;
                    sm[k] = nterms ? sm[k] + t : t;
                }
                nterms++;
            }
            for (int kk = 0; kk < m; ++kk) {
                double rr = p.rho[kk] / p.rho[m];
                masked_grad(h + (long)kk * plane, cowet, grad, s_out, s_in, n_out, n_in);
                for (long k = 0; k < plane; ++k) {
                    double t = ((((-rr) * p.g) * h[m * plane + k]) * grad[k]) / dxdir;
                    sm[k] = nterms ? sm[k] + t : t;
                }
                nterms++;
            }
        }
    }
    for (int m = 0; m < M; ++m) {
        const double *Zc, *Zf, *Bh;
        if (m == M - 1) { Zc = B; Zf = B; Bh = B; }
        else { Zc = zeros; Zf = eta_below + (long)m * plane; Bh = Zf; }
        double *hn = (axis == 1) ? hu + m * plane : hv + m * plane;
        double *ht = (axis == 1) ? hv + m * plane : hu + m * plane;
        sweep_layer(h + m * plane, hn, ht, Zc, Zf, Bh, cowet, cw, s_out, s_in, n_in,
                    gw, lam, p.g, p.tol, j0, j1, scratch);
    }
    if (M > 1) {
        for (int m = 0; m < M; ++m) {
            double *mom = (axis == 1) ? hu + m * plane : hv + m * plane;
            const double *sm = src + m * plane;
            for (int j = j0; j < j1; ++j)
                for (int i = gw; i < n_in - gw; ++i) {
                    long c = (long)j * s_out + (long)i * s_in;
                    mom[c] = mom[c] + dt * sm[c];
                }
        }
    }
    return 0;
}

static size_t sweep_work_bytes(int M, int NY, int NX) {
    long plane = (long)NY * NX;
    long nd = plane * (2 + (M > 1 ? M - 1 : 0) + M + 1) + 5L * (NX > NY ? NX : NY);
    return (size_t)nd * sizeof(double) + (size_t)plane + 64;
}

/* physics.observed_max_speed (physics.py:261-278) over the interior. */
double orc_observed_max_speed(int M, int NY, int NX, int gw, const double *h,
                              const double *hu, const double *hv, double g, double tol)
{
    const long plane = (long)NY * NX;
    int any = 0;
    double best = 0.0;
    for (int j = gw; j < NY - gw; ++j)
        for (int i = gw; i < NX - gw; ++i) {
            long k = (long)j * NX + i;
            double htot = layer_sum(h, plane, k, M);
            double vel = 0.0;
            for (int m = 0; m < M; ++m) {
                double hm = h[m * plane + k];
                int wet = hm > tol;
                double hmm = wet ? hm : 1.0;
                double um = fabs(hu[m * plane + k]) / hmm;
                double vm = fabs(hv[m * plane + k]) / hmm;
                vel = np_maximum(vel, wet ? np_maximum(um, vm) : 0.0);
            }
            double speed = vel + sqrt(g * np_maximum(htot, 0.0));
            if (htot > tol) {
                if (!any) { best = speed; any = 1; }
                else best = np_maximum(best, speed);
            }
        }
    return any ? best : 0.0;
}

typedef struct {
    double max_wave_speed;
    double mass_before[8];
    double mass_after[8];
    double clipped[8];
    int64_t cells_updated;
    int64_t fixes;
    int64_t repairs;
} orc_step_result;

/* physics._blend_shear (physics.py:292-327), interior only, M == 2. */
static int64_t blend_shear(int NY, int NX, int gw, double *h, double *hu, double *hv,
                           double g, double r, double tol)
{
    const long plane = (long)NY * NX;
    int64_t n = 0;
    const double coef = g * (1.0 - r);
    for (int j = gw; j < NY - gw; ++j)
        for (int i = gw; i < NX - gw; ++i) {
            long k = (long)j * NX + i;
            double h1 = h[k], h2 = h[plane + k];
            if (!(h1 > tol && h2 > tol)) continue;
            double hu1 = hu[k], hu2 = hu[plane + k], hv1 = hv[k], hv2 = hv[plane + k];
            double u1 = hu1 / h1, u2 = hu2 / h2, v1 = hv1 / h1, v2 = hv2 / h2;
            double du = u1 - u2, dv = v1 - v2;
            double shear2 = (du * du) + (dv * dv);
            double bound = coef * (h1 + h2);
            if (!(shear2 > bound)) continue;
            n++;
            double alpha = sqrt(bound / shear2);
            double htot = h1 + h2;
            double umean = (hu1 + hu2) / htot;
            double vmean = (hv1 + hv2) / htot;
            hu[k] = h1 * (umean + alpha * (u1 - umean));
            hu[plane + k] = h2 * (umean + alpha * (u2 - umean));
            hv[k] = h1 * (vmean + alpha * (v1 - vmean));
            hv[plane + k] = h2 * (vmean + alpha * (v2 - vmean));
        }
    return n;
}

/* physics.step_patch (physics.py:330-386).  Returns ORC_CFL (before any
 * update) when speed*dt/min(dx,dy) > 1, like CflViolationError. */
int orc_step_patch(int M, int NY, int NX, int gw, double *h, double *hu, double *hv,
                   const double *B, double dx, double dy, double dt,
                   double g, double tol, const double *rho, int y_first,
                   orc_step_result *res)
{
    orc_params p = {M, g, tol, rho};
    const long plane = (long)NY * NX;
    memset(res, 0, sizeof(*res));
    double speed = orc_observed_max_speed(M, NY, NX, gw, h, hu, hv, g, tol);
    res->max_wave_speed = speed;
    double dmin = dx < dy ? dx : dy;
    if ((speed * dt) / dmin > 1.0) return ORC_CFL;
    double area = dx * dy;
    for (int m = 0; m < M; ++m) {
        double s = 0.0;
        for (int j = gw; j < NY - gw; ++j)
            for (int i = gw; i < NX - gw; ++i) s += h[m * plane + (long)j * NX + i];
        res->mass_before[m] = s * area;
    }
    void *work = malloc(sweep_work_bytes(M, NY, NX));
    if (!work) return ORC_ALLOC;
    if (y_first) {
        sweep_dir(0, NY, NX, h, hu, hv, B, dt, dy, p, 1, gw, work);
        sweep_dir(1, NY, NX, h, hu, hv, B, dt, dx, p, 0, gw, work);
    } else {
        sweep_dir(1, NY, NX, h, hu, hv, B, dt, dx, p, 1, gw, work);
        sweep_dir(0, NY, NX, h, hu, hv, B, dt, dy, p, 0, gw, work);
    }
    free(work);
    /* clip negative depths (physics.py:360-364) */
    for (int m = 0; m < M; ++m) {
        double s = 0.0;
        for (int j = gw; j < NY - gw; ++j)
            for (int i = gw; i < NX - gw; ++i) {
                double *x = &h[m * plane + (long)j * NX + i];
                double neg = np_minimum(*x, 0.0);
                s += neg;
                if (neg < 0.0) *x = 0.0;
            }
        res->clipped[m] = -s * area;
    }
    if (M == 2) res->fixes = blend_shear(NY, NX, gw, h, hu, hv, g, rho[0] / rho[1], tol);
    /* state.restore_wet_prefix (state.py:125-145) then zero_dry_momenta (:104-110) */
    for (int m = 1; m < M; ++m)
        for (int j = gw; j < NY - gw; ++j)
            for (int i = gw; i < NX - gw; ++i) {
                long k = (long)j * NX + i;
                long a = (m - 1) * plane + k, b = m * plane + k;
                if (h[b] > tol && h[a] <= tol) {
                    res->repairs++;
                    h[a] = h[a] + h[b]; hu[a] = hu[a] + hu[b]; hv[a] = hv[a] + hv[b];
                    h[b] = 0.0; hu[b] = 0.0; hv[b] = 0.0;
                }
            }
    for (int m = 0; m < M; ++m)
        for (int j = gw; j < NY - gw; ++j)
            for (int i = gw; i < NX - gw; ++i) {
                long k = m * plane + (long)j * NX + i;
                if (h[k] <= tol) { hu[k] = 0.0; hv[k] = 0.0; }
            }
    for (int m = 0; m < M; ++m) {
        double s = 0.0;
        for (int j = gw; j < NY - gw; ++j)
            for (int i = gw; i < NX - gw; ++i) s += h[m * plane + (long)j * NX + i];
        res->mass_after[m] = s * area;
    }
    res->cells_updated = (int64_t)(NY - 2 * gw) * (NX - 2 * gw);
    return ORC_OK;
}

/* ---------------------------------------------------------------------- */
/* refine.interpolate_state (refine.py:158-190) with _limited_slopes       */
/* (:82-98), _parent_indexing (:101-116), interpolate_to_fine (:119-137),  */
/* minmod (:37-47) and state.surfaces_from_state (state.py:56-61).         */
/* ---------------------------------------------------------------------- */
static inline double minmod(double a, double b) {
    int same = (a * b) > 0.0;
    double smaller = (fabs(a) <= fabs(b)) ? a : b;
    return same ? smaller : 0.0;
}

static inline long floordiv(long a, long b) {
    long q = a / b;
    if ((a % b != 0) && ((a < 0) != (b < 0))) q--;
    return q;
}

/*
 * coarse fields cover box (clo_i, clo_j, cnx, cny): ch/chu/chv [M][cny][cnx],
 * cb [cny][cnx], cavail [cny][cnx].  Fine box (flo_i, flo_j, fnx, fny) with
 * fine bathymetry fb [fny][fnx] (row stride fb_stride).  Outputs are written
 * with row stride out_stride and layer stride out_plane.
 */
int orc_interpolate_state(int M, const double *ch, const double *chu, const double *chv,
                          const double *cb, const uint8_t *cavail,
                          int clo_i, int clo_j, int cnx, int cny,
                          int flo_i, int flo_j, int fnx, int fny,
                          const double *fb, long fb_stride,
                          int r_x, int r_y, double tol,
                          double *oh, double *ohu, double *ohv, long out_stride, long out_plane)
{
    const long cplane = (long)cnx * cny;
    for (int fj = 0; fj < fny; ++fj) {
        long pj = floordiv(flo_j + fj, r_y) - clo_j;
        if (pj < 0 || pj >= cny) return ORC_GEOMETRY;
    }
    for (int fi = 0; fi < fnx; ++fi) {
        long pi = floordiv(flo_i + fi, r_x) - clo_i;
        if (pi < 0 || pi >= cnx) return ORC_GEOMETRY;
    }
    double *eta = (double *)malloc(sizeof(double) * cplane * 2);
    uint8_t *use = (uint8_t *)malloc(cplane);
    double *bhat = (double *)malloc(sizeof(double) * (long)fnx * fny);
    if (!eta || !use || !bhat) { free(eta); free(use); free(bhat); return ORC_ALLOC; }
    double *acc = eta + cplane;
    for (int fj = 0; fj < fny; ++fj)
        for (int fi = 0; fi < fnx; ++fi) bhat[(long)fj * fnx + fi] = fb[(long)fj * fb_stride + fi];
    for (int m = M - 1; m >= 0; --m) {
        /* eta_m = cumsum over layers m..M-1 (bottom first) + B */
        for (long k = 0; k < cplane; ++k) {
            acc[k] = (m == M - 1) ? ch[m * cplane + k] : acc[k] + ch[m * cplane + k];
            eta[k] = acc[k] + cb[k];
            use[k] = cavail[k] && (ch[m * cplane + k] > tol);
        }
        for (int fj = 0; fj < fny; ++fj) {
            long gj = flo_j + fj;
            long pjg = floordiv(gj, r_y);
            int cj = (int)(pjg - clo_j);
            double offy = ((double)(gj - pjg * r_y) + 0.5) / r_y - 0.5;
            for (int fi = 0; fi < fnx; ++fi) {
                long gi = flo_i + fi;
                long pig = floordiv(gi, r_x);
                int ci = (int)(pig - clo_i);
                double offx = ((double)(gi - pig * r_x) + 0.5) / r_x - 0.5;
                long c = (long)cj * cnx + ci;
                int okx = ci >= 1 && ci <= cnx - 2 && use[c - 1] && use[c] && use[c + 1];
                int oky = cj >= 1 && cj <= cny - 2 && use[c - cnx] && use[c] && use[c + cnx];
                const double *fields[3] = {eta, chu + m * cplane, chv + m * cplane};
                double outv[3];
                for (int q = 0; q < 3; ++q) {
                    const double *v = fields[q];
                    double sx = 0.0, sy = 0.0;
                    if (ci >= 1 && ci <= cnx - 2) sx = minmod(v[c] - v[c - 1], v[c + 1] - v[c]);
                    if (cj >= 1 && cj <= cny - 2) sy = minmod(v[c] - v[c - cnx], v[c + cnx] - v[c]);
                    if (!okx) sx = 0.0;
                    if (!oky) sy = 0.0;
                    outv[q] = (v[c] + (sx * offx)) + (sy * offy);
                }
                long fk = (long)fj * fnx + fi;
                double hh = np_maximum(0.0, outv[0] - bhat[fk]);
                double uu = outv[1], vv = outv[2];
                if (hh <= tol) { uu = 0.0; vv = 0.0; }
                long o = (long)m * out_plane + (long)fj * out_stride + fi;
                oh[o] = hh; ohu[o] = uu; ohv[o] = vv;
                bhat[fk] = bhat[fk] + hh;
            }
        }
    }
    free(eta); free(use); free(bhat);
    return ORC_OK;
}

/* numpy's pairwise_sum over n contiguous doubles (numpy/_core/src/umath/
 * loops_utils.h.src): sequential from 0.0 below 8 elements, else eight
 * running accumulators combined as ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) plus
 * a sequential tail (n <= 128 here). */
static double np_pairwise(const double *a, int n)
{
    if (n < 8) {
        double res = 0.0;
        for (int i = 0; i < n; ++i) res = res + a[i];
        return res;
    }
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int i = 8;
    for (; i < n - (n % 8); i += 8)
        for (int j = 0; j < 8; ++j) r[j] = r[j] + a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res = res + a[i];
    return res;
}

/* coarsen.block_mean (coarsen.py:21-27) in numpy's evaluation order for
 * r <= 4 (SURVEY probe 2, extended): the reduction over axes (-3, -1) of
 * the (.., cny, r_y, cnx, r_x) view sums, per fine row, sequentially over p,
 * then the row sums sequentially over q -- unless the patch is ONE coarse
 * cell wide (cnx == 1): numpy then coalesces the r_y x r_x block into one
 * contiguous run of r_x*r_y elements and sums it with pairwise_sum.  One
 * divide by r_x*r_y either way.  src has row stride src_stride. */
void orc_block_mean(const double *src, long src_stride, int cnx, int cny,
                    int r_x, int r_y, double *dst, long dst_stride)
{
    double blk[64];
    for (int J = 0; J < cny; ++J)
        for (int I = 0; I < cnx; ++I) {
            double s = 0.0;
            if (cnx == 1 && r_x * r_y <= 64) {
                for (int q = 0; q < r_y; ++q)
                    for (int pp = 0; pp < r_x; ++pp)
                        blk[q * r_x + pp] = src[(long)(J * r_y + q) * src_stride + (long)I * r_x + pp];
                s = np_pairwise(blk, r_x * r_y);
            } else {
                for (int q = 0; q < r_y; ++q) {
                    const double *row = src + (long)(J * r_y + q) * src_stride + (long)I * r_x;
                    double rs = row[0];
                    for (int pp = 1; pp < r_x; ++pp) rs = rs + row[pp];
                    s = (q == 0) ? rs : s + rs;
                }
            }
            dst[(long)J * dst_stride + I] = s / (double)(r_x * r_y);
        }
}
