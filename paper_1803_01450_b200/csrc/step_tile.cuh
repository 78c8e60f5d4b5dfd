// One tile shape of the batched patch step (K1).  Included by k_step.cu
// once per shape, inside `namespace mlamr::MLAMR_STEP_NS`, with
// MLAMR_STEP_TX / _TY (interior tile columns / rows), MLAMR_STEP_NT
// (threads) and MLAMR_STEP_MINB (CTAs per SM) defined by the includer.
// Everything shape-dependent lives here: the shared tile, the sweep
// phases, the step kernel, the tile-based speed kernel and the launcher.

namespace MLAMR_STEP_NS {

constexpr int TX = MLAMR_STEP_TX;
constexpr int TY = MLAMR_STEP_TY;
constexpr int PX = TX + 2;
constexpr int PY = TY + 2;
constexpr int NPAD = PX * PY;
constexpr int NFLUX = PY * PX;  // interface (r,c) stored at the cell index of its left/lower cell
constexpr int NT = MLAMR_STEP_NT;  // threads of the step CTA

template <int M>
struct StepSmem {
    double S[3 * M + 1][NPAD];           // h_0..h_{M-1}, hu_.., hv_.., B
    double cw[NPAD];                     // sqrt(g * max(sum h, 0))
    double eb[M > 1 ? M - 1 : 1][NPAD];  // eta_{m+1} = B + h_{M-1} + ... + h_{m+1}
    double u[M][NPAD];                   // normal velocity per layer
    double v[M][NPAD];                   // transverse velocity per layer
    double F[2 * M][NFLUX];              // (Fh, Fm) per layer at interface (r,c)-(r,c)+step
    double src[M > 1 ? M - 1 : 1][NPAD]; // coupling sources of layers 1..M-1
    double red[(M + 2) * (NT / 32)];
    long long redi[NT / 32];
    unsigned char cowet[NPAD];
    unsigned char wetcol[NPAD];
};

// All shared-memory phases iterate a rectangle [r0,r1) x [c0,c1) of the
// padded tile in row-major order over the rectangle itself (compact: a
// ragged tile -- 16.5 % of C4's level-3 tile slots are outside patches --
// costs iterations in proportion to its cells, not to the full tile), with
// consecutive threads on consecutive cells of a row (no bank conflicts in
// either sweep direction).  The row split divides by the runtime width w
// with a reciprocal table, q = (idx * ceil(2^16/w)) >> 16, which is
// floor(idx/w) whenever idx/65536 < 1/w (the rounding-up error stays below
// the gap to the next integer) -- every rectangle here (idx < 612, w <= 34):
// one multiply and a shift, the cost of the compile-time pitch it replaces
// (runtime integer division costs three XU ops and saturated the XU pipe in
// the first profile).  Storage keeps the compile-time pitch PX.
// (a begin/end macro pair rather than a macro taking the body, so the
// body keeps its own source lines in the profiler's source view)
#define FOR_RECT_BEGIN(r0, r1, c0, c1)                                        \
    for (int w_ = (c1) - (c0), m_ = (int)c_div_magic[w_], idx_ = threadIdx.x; \
         idx_ < ((r1) - (r0)) * w_; idx_ += NT) {                             \
        const int q_ = (int)(((unsigned)idx_ * (unsigned)m_) >> 16);          \
        const int r = (r0) + q_;                                              \
        const int c = (c0) + idx_ - q_ * w_;
#define FOR_RECT_END }


// Reconstruction bottoms of layer m at a cell (physics.py:200-207, 105-110):
// co-wet pairs use Zc (0 for upper layers, B for the bottom layer), others
// Zf (= Bhat: eta_{m+1} for upper layers, B for the bottom layer).
template <int M>
__device__ __forceinline__ double zc_of(const StepSmem<M> &s, int m, int k) {
    return (m == M - 1) ? s.S[3 * M][k] : 0.0;
}
template <int M, bool SW = false>
__device__ __forceinline__ double zf_of(const StepSmem<M> &s, int m, int k) {
    return (m == M - 1) ? s.S[3 * M][k] : (SW ? s.src : s.eb)[m < M - 1 ? m : 0][k];
}
// The second sweep finds its eta_{m+1} planes in `src` and its co-wet flags
// in `wetcol` (SW): the first sweep's update writes them there, next to the
// planes its neighbours are still reading (see NEXT in sweep_tile), and the
// second sweep's sources go to the then free `eb` planes.
template <int M, bool SW>
__device__ __forceinline__ double *eb_pl(StepSmem<M> &s, int m) { return SW ? s.src[m] : s.eb[m]; }
template <int M, bool SW>
__device__ __forceinline__ double *src_pl(StepSmem<M> &s, int m) { return SW ? s.eb[m] : s.src[m]; }
template <int M, bool SW>
__device__ __forceinline__ unsigned char *cowet_pl(StepSmem<M> &s) { return SW ? s.wetcol : s.cowet; }

// Post-processing of one interior cell (physics.py:360-376): clip negative
// depths, the shear blend (M = 2), the wet-prefix repair and zeroing dry
// momenta, then the store to the destination state.  Runs inside the last
// sweep's update, on the values that update produced.
struct PostCtx {
    double *dst;
    int64_t base, FS;
    int NX;
    double tol, coef;
    double negs[MLAMR_MAX_LAYERS];
    long long fixes, repairs;
};

template <int M>
__device__ __forceinline__ void post_cell(double (&h)[M], double (&hu)[M], double (&hv)[M], PostCtx &pc, int r,
                                          int c) {
    const double tol = pc.tol, coef = pc.coef;
#pragma unroll
    for (int m = 0; m < M; ++m) {
        const double neg = np_min(h[m], 0.0);
        pc.negs[m] = pc.negs[m] + neg;
        if (neg < 0.0) h[m] = 0.0;
    }
    if (M == 2) {  // _blend_shear (physics.py:292-327)
        const double h1 = h[0], h2 = h[1 % M];
        // Screen: U >= shear2 / (1 + 2^-18) is built from approximate
        // reciprocals (rcp.approx, relative error far below 1/8), so
        // U * 1.125 < bound proves the reference's `shear2 > bound` false
        // and the blend a no-op -- almost every co-wet cell, whose shear is
        // orders of magnitude below g(1-r)(h1+h2).  Only cells the screen
        // cannot clear take the exact divisions below.  NaN/inf operands
        // fail the screen's comparison; h >= 1e300 (reciprocal below the
        // normal range, flushed by .ftz) and coef <= 0 skip it.
        bool maybe = true;
        if (h1 > tol && h2 > tol && coef > 0.0 && h1 < 1e300 && h2 < 1e300) {
            double a1, a2;
            asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(a1) : "d"(h1));
            asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(a2) : "d"(h2));
            const double su = fabs(hu[0]) * a1 + fabs(hu[1 % M]) * a2;
            const double sv = fabs(hv[0]) * a1 + fabs(hv[1 % M]) * a2;
            maybe = !((su * su + sv * sv) * 1.125 < coef * (h1 + h2));
        }
        if (maybe && h1 > tol && h2 > tol) {
            const double hu1 = hu[0], hu2 = hu[1 % M], hv1 = hv[0], hv2 = hv[1 % M];
            bool ok = true;
            const double y1 = recip_nr(h1), y2 = recip_nr(h2);
            double u1 = div_fast(hu1, h1, y1, ok), v1 = div_fast(hv1, h1, y1, ok);
            double u2 = div_fast(hu2, h2, y2, ok), v2 = div_fast(hv2, h2, y2, ok);
            if (!ok) {
                u1 = div_slow(hu1, h1);
                u2 = div_slow(hu2, h2);
                v1 = div_slow(hv1, h1);
                v2 = div_slow(hv2, h2);
            }
            const double du = u1 - u2, dv = v1 - v2;
            const double shear2 = (du * du) + (dv * dv);
            const double bound = coef * (h1 + h2);
            if (shear2 > bound) {
                ++pc.fixes;
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
            ++pc.repairs;
            h[m - 1] = h[m - 1] + h[m];
            hu[m - 1] = hu[m - 1] + hu[m];
            hv[m - 1] = hv[m - 1] + hv[m];
            h[m] = 0.0;
            hu[m] = 0.0;
            hv[m] = 0.0;
        }
    }
    const int64_t gaddr = pc.base + (int64_t)r * pc.NX + c;
#pragma unroll
    for (int m = 0; m < M; ++m) {
        if (h[m] <= tol) {
            hu[m] = 0.0;
            hv[m] = 0.0;
        }
        pc.dst[m * pc.FS + gaddr] = h[m];
        pc.dst[(M + m) * pc.FS + gaddr] = hu[m];
        pc.dst[(2 * M + m) * pc.FS + gaddr] = hv[m];
    }
}

// One directional sweep of all layers over the staged tile
// (physics._sweep_x / _sweep_y with _layer_inputs), three phases:
//   A  per cell:      layer inputs (cw, cowet, eta_{m+1}) and velocities
//   B  per interface: HLL fluxes of every layer, coupling sources
//   C  per cell:      conservative update + pressure correction + source
// DIR 0 = x (interfaces between columns c, c+1), 1 = y (rows r, r+1).
// FIRST: all halo lines (the reference's full=True); else interior lines.
// AW: every cell the sweep reads is wet in every layer (tol < h < 1e150), so
// every pair is co-wet and the predicates below are known: the upper
// layers' reconstruction is the identity (Zl = Zr = 0 and h > 0 give
// (h + 0) - 0 = h exactly), their pressure correction is exactly +0
// (C * (h0^2 - h0^2) with finite h0), and the wet/co-wet selects go.  The
// arithmetic that remains is operation for operation the general path's.
//
// One call runs phase A (RUN_A, all-wet path AWA) and/or phases B-C
// (RUN_BC, all-wet path AW) and returns, block-wide, whether every cell
// phase A read (RUN_A only) or every cell phase C updated is wet in every
// layer -- the all-wet decision for what follows.
template <int M, int DIR, bool FIRST, bool AWA, bool AW, bool RUN_A, bool RUN_BC, bool LAST = false,
          bool SW = false, bool NEXT = false>
__device__ bool sweep_tile(StepSmem<M> &s, int ny2, int nx2, double dt, double d, double lam, double yd,
                           const mlamr_params &prm, const double (&rr)[4][4], double &best,
                           double &nacc, PostCtx *post = nullptr) {
    // lam = dt / d and yd = recip_nr(d) come from the kernel prologue, where
    // their latency overlaps the tile's in-flight loads
    const double g = prm.gravity;
    const double tol = prm.dry_tolerance;
    const double *B = s.S[3 * M];
    constexpr int STEP = DIR == 0 ? 1 : PX;  // neighbour offset along the sweep
    const int n_along = DIR == 0 ? nx2 : ny2;
    // lines: DIR 0 sweeps rows (lines = rows), DIR 1 sweeps columns
    const int lr0 = (DIR == 0 && !FIRST) ? 1 : 0, lr1 = (DIR == 0 && !FIRST) ? ny2 - 1 : ny2;
    const int lc0 = (DIR == 1 && !FIRST) ? 1 : 0, lc1 = (DIR == 1 && !FIRST) ? nx2 - 1 : nx2;
    // updated cells exclude the first/last cell along the sweep
    const int ur0 = DIR == 1 ? 1 : lr0, ur1 = DIR == 1 ? ny2 - 1 : lr1;
    const int uc0 = DIR == 0 ? 1 : lc0, uc1 = DIR == 0 ? nx2 - 1 : lc1;
    // interfaces: (r,c)-(r,c+1) for DIR 0, (r,c)-(r+1,c) for DIR 1
    const int fr1 = DIR == 1 ? ny2 - 1 : lr1;
    const int fc1 = DIR == 0 ? nx2 - 1 : lc1;

    if (RUN_A) {
        bool wet_in = true;
        // ---- Phase A: per-cell inputs on the pre-sweep state of this direction
        FOR_RECT_BEGIN(lr0, lr1, lc0, lc1)
            const int k = r * PX + c;
            double h[M];
            double hs = 0.0;
            bool w = true;
#pragma unroll
            for (int m = 0; m < M; ++m) {
                h[m] = s.S[m][k];
                hs = hs + h[m];
                w = w && (h[m] > tol);
                wet_in = wet_in & (h[m] > tol) & (h[m] < 1e150);
            }
            // AW: hs > tol > 0, so numpy's maximum(hs, 0) is hs
            const double cw = sqrt(g * (AWA ? hs : np_max(hs, 0.0)));
            s.cw[k] = cw;
            if (!AWA) s.cowet[k] = (M == 1) ? 1 : w;
            if (M > 1) {
                double e = B[k];
#pragma unroll
                for (int m = M - 1; m >= 1; --m) {
                    e = e + h[m];
                    s.eb[m - 1][k] = e;
                }
            }
            const bool interior = FIRST && r >= 1 && r < ny2 - 1 && c >= 1 && c < nx2 - 1 && (AWA || hs > tol);
#pragma unroll
            for (int m = 0; m < M; ++m) {
                const bool wet = AWA || h[m] > tol;
                const double hn = s.S[(DIR == 0 ? M : 2 * M) + m][k];
                const double ht = s.S[(DIR == 0 ? 2 * M : M) + m][k];
                double u = 0.0, v = 0.0;
                if (wet) {
                    bool ok = true;
                    const double y = recip_nr(h[m]);
                    u = div_fast(hn, h[m], y, ok);
                    v = div_fast(ht, h[m], y, ok);
                    if (!ok) {
                        u = div_slow(hn, h[m]);
                        v = div_slow(ht, h[m]);
                    }
                }
                s.u[m][k] = u;
                s.v[m][k] = v;
                if (interior) {
                    // observed_max_speed (physics.py:261-278): speed = max(0, x_0,
                    // .., x_{M-1}) + cw with x_m = wet ? max(|hu|/h, |hv|/h) : 0 and
                    // |hu|/h == |hu/h|.  Dry layers have u = v = 0 here, x_m >= 0,
                    // and rounding is monotone, so max_m(x_m) + cw ==
                    // max_m(x_m + cw) and max(cw, x_0 + cw) == x_0 + cw: the
                    // running max is bit-identical to the reference's for
                    // non-NaN operands.  fmax ignores NaN, so NaN-ness (numpy's
                    // maximum propagates it) travels in `nacc`: |u| + |v| is NaN
                    // iff either is (cw is finite or inf: hs > tol here), and the
                    // tile maximum is replaced by NaN at the end.
                    const double au = fabs(u), av = fabs(v);
                    best = fmax(best, fmax(au, av) + cw);
                    nacc = nacc + (au + av);
                }
            }
        FOR_RECT_END
        const bool all_in = __syncthreads_and(wet_in) != 0;
        if (!RUN_BC) return all_in;
    }

    // ---- Phase B: HLL fluxes per interface (physics.py:101-161) + sources
    FOR_RECT_BEGIN(lr0, fr1, lc0, fc1)
        const int kl = r * PX + c;
        const int kr = kl + STEP;
        const unsigned char *CW = cowet_pl<M, SW>(s);
        const bool cop = AW || (CW[kl] && CW[kr]);
        const double cl = s.cw[kl];
        const double cr = s.cw[kr];
#pragma unroll
        for (int m = 0; m < M; ++m) {
            const double hl = s.S[m][kl];
            const double hr = s.S[m][kr];
            const double ul = s.u[m][kl];
            const double ur = s.u[m][kr];
            double hL, hR;
            if (AW && m < M - 1) {
                hL = hl;
                hR = hr;
            } else {
                const double Zl = cop ? zc_of<M>(s, m, kl) : zf_of<M, SW>(s, m, kl);
                const double Zr = cop ? zc_of<M>(s, m, kr) : zf_of<M, SW>(s, m, kr);
                const double Zs = Zl > Zr ? Zl : Zr;
                hL = (hl + Zl) - Zs;
                if (hL < 0.0) hL = 0.0;
                hR = (hr + Zr) - Zs;
                if (hR < 0.0) hR = 0.0;
            }
            double fh = 0.0, fm = 0.0;
            if ((AW && m < M - 1) || !(hL <= 0.0 && hR <= 0.0)) {
                const double sl1 = ul - cl, sl2 = ur - cr;
                const double SL = sl1 < sl2 ? sl1 : sl2;
                const double sr1 = ul + cl, sr2 = ur + cr;
                const double SR = sr1 > sr2 ? sr1 : sr2;
                const double FLh = hL * ul;
                const double FRh = hR * ur;
                const double FLm = ((hL * ul) * ul) + (((0.5 * g) * hL) * hL);
                const double FRm = ((hR * ur) * ur) + (((0.5 * g) * hR) * hR);
                // the subsonic case first (nearly every interface): written as
                // if / else-if / else, the compiler copied the left and the
                // right state into the flux registers in front of each test
                // (8 moves per layer on the common path).  NaN speeds fail
                // both tests and take the HLL branch, as in the reference.
                if (SL >= 0.0 || SR <= 0.0) {
                    const bool left = SL >= 0.0;
                    fh = left ? FLh : FRh;
                    fm = left ? FLm : FRm;
                } else {
                    const double den = SR - SL;
                    double djump;
                    if ((AW && m < M - 1) || (hL > 0.0 && hR > 0.0))
                        djump = (hr + zf_of<M, SW>(s, m, kr)) - (hl + zf_of<M, SW>(s, m, kl));
                    else
                        djump = hR - hL;
                    const double nh = ((SR * FLh) - (SL * FRh)) + ((SL * SR) * djump);
                    const double nm = ((SR * FLm) - (SL * FRm)) + ((SL * SR) * ((hR * ur) - (hL * ul)));
                    bool ok = true;
                    const double y = recip_nr(den);
                    fh = div_fast(nh, den, y, ok);
                    fm = div_fast(nm, den, y, ok);
                    if (!ok) {
                        fh = div_slow(nh, den);
                        fm = div_slow(nm, den);
                    }
                }
            }
            s.F[2 * m][kl] = fh;
            s.F[2 * m + 1][kl] = fm;

        }
        // coupling sources of layers >= 1 for the interface's upper cell
        // (physics.py:208-211), on the pre-sweep state
        const int a = DIR == 0 ? c : r;
        if (M > 1 && a + 1 < n_along - 1) {
            const int k = kr, km = kl, kp = kr + STEP;
            const bool wm = AW || (CW[km] && CW[k]);
            const bool wp = AW || (CW[k] && CW[kp]);
#pragma unroll
            for (int m = 1; m < M; ++m) {
                double acc = 0.0;
                bool has = false;
                bool ok = true;
                if (m < M - 1) {
                    const double *f = eb_pl<M, SW>(s, m < M - 1 ? m : 0);
                    const double dm = wm ? f[k] - f[km] : 0.0;
                    const double dp = wp ? f[kp] - f[k] : 0.0;
                    const double num = ((-g) * s.S[m][k]) * (0.5 * (dp + dm));
                    double q = div_fast(num, d, yd, ok);
                    if (!ok) q = div_slow(num, d);
                    acc = q;
                    has = true;
                }
#pragma unroll
                for (int kk = 0; kk < m; ++kk) {
                    const double *f = s.S[kk];
                    const double dm = wm ? f[k] - f[km] : 0.0;
                    const double dp = wp ? f[kp] - f[k] : 0.0;
                    const double num = (((-rr[kk][m]) * g) * s.S[m][k]) * (0.5 * (dp + dm));
                    ok = true;
                    double q = div_fast(num, d, yd, ok);
                    if (!ok) q = div_slow(num, d);
                    acc = has ? acc + q : q;
                    has = true;
                }
                src_pl<M, SW>(s, m - 1)[k] = acc;
            }
        }
    FOR_RECT_END
    __syncthreads();

    // ---- Phase C: conservative update + pressure correction + source.
    // The updated cells are exactly the cells the other sweep reads, so
    // their wetness decides (block-wide, with the closing barrier) whether
    // that sweep can take the all-wet path.
    bool wet_out = true;
    // NEXT: this update also computes the other sweep's per-cell inputs
    // (its phase A) from the registers -- the updated cells are exactly the
    // cells that phase reads.  cw and u are not read by this phase and are
    // stored at once; eta_{m+1} and the co-wet flags go to the planes the
    // other sweep reads with SW; v, which this phase reads at neighbours,
    // waits in registers for the closing barrier.
    constexpr int MAXIT = (NPAD + NT - 1) / NT;
    double v2s[NEXT ? MAXIT : 1][M];
    int k2s[NEXT ? MAXIT : 1];
#pragma unroll
    for (int it = 0; it < (NEXT ? MAXIT : 1); ++it) k2s[it] = -1;
    const unsigned char *CWc = cowet_pl<M, SW>(s);
    const int uw = uc1 - uc0;
    const unsigned um = c_div_magic[uw];
#pragma unroll
    for (int it = 0; it < MAXIT; ++it) {
        const int idx_ = threadIdx.x + it * NT;
        if (idx_ >= (ur1 - ur0) * uw) break;
        const int q_ = (int)(((unsigned)idx_ * um) >> 16);
        const int r = ur0 + q_;
        const int c = uc0 + idx_ - q_ * uw;
        const int k = r * PX + c;
        const int km = k - STEP, kp = k + STEP;
        const bool copl = AW || (CWc[km] && CWc[k]);
        const bool copr = AW || (CWc[k] && CWc[kp]);
        double nh[M], nn[M], nt[M];   // LAST: the updated cell stays in registers
#pragma unroll
        for (int m = 0; m < M; ++m) {
            double *H = s.S[m];
            double *HN = s.S[(DIR == 0 ? M : 2 * M) + m];
            double *HT = s.S[(DIR == 0 ? 2 * M : M) + m];
            const double h0 = H[k];
            const double fhl = s.F[2 * m][km], fhr = s.F[2 * m][k];
            const double fml = s.F[2 * m + 1][km], fmr = s.F[2 * m + 1][k];
            // upwinded transverse flux (physics.py:155-161):
            // f > 0 ? f * v_left : (f < 0 ? f * v_right : 0), branch-free
            // (both neighbours' v loaded; f == +-0 or NaN gives +0)
            const double vkm = s.v[m][km], vk = s.v[m][k], vkp = s.v[m][kp];
            const double fvl = fabs(fhl) > 0.0 ? fhl * (fhl > 0.0 ? vkm : vk) : 0.0;
            const double fvr = fabs(fhr) > 0.0 ? fhr * (fhr > 0.0 ? vk : vkp) : 0.0;
            const double hnew = h0 - lam * (fhr - fhl);
            if (!LAST) H[k] = hnew;
            nh[m] = hnew;
            wet_out = wet_out & (hnew > tol) & (hnew < 1e150);
            double hn;
            if (AW && m < M - 1) {
                // both faces reconstruct to h0: the correction is exactly +0
                hn = HN[k] - lam * (fmr - fml);
            } else {
                // this cell's reconstructed depths at its two faces: hsR of the
                // left interface and hsL of the right one (physics.py:113-121)
                const double Zl_l = copl ? zc_of<M>(s, m, km) : zf_of<M, SW>(s, m, km);
                const double Zk_l = copl ? zc_of<M>(s, m, k) : zf_of<M, SW>(s, m, k);
                const double Zk_r = copr ? zc_of<M>(s, m, k) : zf_of<M, SW>(s, m, k);
                const double Zr_r = copr ? zc_of<M>(s, m, kp) : zf_of<M, SW>(s, m, kp);
                const double Zs_l = Zl_l > Zk_l ? Zl_l : Zk_l;
                const double Zs_r = Zk_r > Zr_r ? Zk_r : Zr_r;
                double hsR_l = (h0 + Zk_l) - Zs_l;
                if (hsR_l < 0.0) hsR_l = 0.0;
                double hsL_r = (h0 + Zk_r) - Zs_r;
                if (hsL_r < 0.0) hsL_r = 0.0;
                hn = (HN[k] - lam * (fmr - fml)) - (((lam * 0.5) * g) * ((hsR_l * hsR_l) - (hsL_r * hsL_r)));
            }
            if (M > 1) {
                double sm;
                if (m == 0) {  // physics.py:210, from the pre-sweep eta_1 and own h_0
                    const double *f = eb_pl<M, SW>(s, 0);
                    const double dm = copl ? f[k] - f[km] : 0.0;
                    const double dp = copr ? f[kp] - f[k] : 0.0;
                    const double num = ((-g) * h0) * (0.5 * (dp + dm));
                    bool ok = true;
                    sm = div_fast(num, d, yd, ok);
                    if (!ok) sm = div_slow(num, d);
                } else {
                    sm = src_pl<M, SW>(s, m - 1)[k];
                }
                hn = hn + dt * sm;
            }
            const double htn = HT[k] - lam * (fvr - fvl);
            if (!LAST) {
                HN[k] = hn;
                HT[k] = htn;
            }
            nn[m] = hn;
            nt[m] = htn;
        }
        if (LAST) {
            // hu/hv from the normal/transverse momenta of this direction
            if (DIR == 0) post_cell<M>(nh, nn, nt, *post, r, c);
            else post_cell<M>(nh, nt, nn, *post, r, c);
        }
        if (NEXT) {
            // the other sweep's phase A (general path) on the updated cell:
            // its normal momentum is this sweep's transverse one (nt)
            double hs = 0.0;
            bool w = true;
#pragma unroll
            for (int m = 0; m < M; ++m) {
                hs = hs + nh[m];
                w = w && (nh[m] > tol);
            }
            s.cw[k] = sqrt(g * np_max(hs, 0.0));
            cowet_pl<M, !SW>(s)[k] = (M == 1) ? 1 : w;
            if (M > 1) {
                double e = B[k];
#pragma unroll
                for (int m = M - 1; m >= 1; --m) {
                    e = e + nh[m];
                    eb_pl<M, !SW>(s, m - 1)[k] = e;
                }
            }
#pragma unroll
            for (int m = 0; m < M; ++m) {
                double u = 0.0, v = 0.0;
                if (nh[m] > tol) {
                    bool ok = true;
                    const double y = recip_nr(nh[m]);
                    u = div_fast(nt[m], nh[m], y, ok);
                    v = div_fast(nn[m], nh[m], y, ok);
                    if (!ok) {
                        u = div_slow(nt[m], nh[m]);
                        v = div_slow(nn[m], nh[m]);
                    }
                }
                s.u[m][k] = u;
                v2s[NEXT ? it : 0][m] = v;
            }
            k2s[NEXT ? it : 0] = k;
        }
    }
    // the last sweep's wetness is not used and nothing reads its shared
    // planes afterwards (the tile's reductions have their own barrier)
    const bool all_wet = LAST ? true : (__syncthreads_and(wet_out) != 0);
    if (NEXT) {
#pragma unroll
        for (int it = 0; it < MAXIT; ++it) {
            if (k2s[it] < 0) continue;
#pragma unroll
            for (int m = 0; m < M; ++m) s.v[m][k2s[it]] = v2s[it][m];
        }
    }
    return all_wet;
}


template <int M, bool YFIRST>
__global__ void __launch_bounds__(NT, MLAMR_STEP_MINB) k_step(mlamr_level lv, const double *__restrict__ src,
                                             double *__restrict__ dst,
                                             const TileDesc *__restrict__ desc, double dt,
                                             mlamr_params prm, StepConst kc, long long *speed_bits,
                                             double *tile_acc, const int32_t *status,
                                             const int64_t *__restrict__ gplan) {
    // the status word is read now but tested only once this tile's staging
    // is in flight: testing it first put a dependent global load in front
    // of every CTA's loads
    const int32_t st0 = status != nullptr ? *status : 0;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    StepSmem<M> &s = *reinterpret_cast<StepSmem<M> *>(smem_raw);
    const int t = threadIdx.x;
    const int tile = blockIdx.x;
    // one 32-byte descriptor (k_make_desc) instead of the chain tile list ->
    // box/offset -> ghost base: one L2 round trip in front of the staging
    const int4 dq0 = __ldg(reinterpret_cast<const int4 *>(desc + tile));
    const int4 dq1 = __ldg(reinterpret_cast<const int4 *>(desc + tile) + 1);
    const int p = dq0.x, tj0 = dq0.y, ti0 = dq0.z;
    PatchView pv;
    pv.nx = dq0.w & 0xffff;
    pv.ny = (int)((unsigned)dq0.w >> 16);
    pv.NX = pv.nx + 2 * MLAMR_G;
    pv.NY = pv.ny + 2 * MLAMR_G;
    pv.off = (int64_t)(((unsigned long long)(unsigned)dq1.y << 32) | (unsigned)dq1.x);
    const int64_t gb = (int64_t)(((unsigned long long)(unsigned)dq1.w << 32) | (unsigned)dq1.z);
    const int ty = min(TY, pv.ny - tj0);
    const int tx = min(TX, pv.nx - ti0);
    const int ny2 = ty + 2, nx2 = tx + 2;
    const int64_t FS = lv.field_stride;
    const int64_t base = pv.off + (int64_t)(tj0 + 1) * pv.NX + (ti0 + 1);

    // stage the padded tile with asynchronous 8-byte copies (LDGSTS): every
    // thread keeps ~NITEM*(3M+1) global loads in flight instead of
    // serialising load -> shared store pairs.  The (row, column) split of a
    // thread's items is done once; each plane then costs one address add and
    // one LDGSTS per item.
    {
        constexpr int NITEM = (NPAD + NT - 1) / NT;
        unsigned sa[NITEM];
        const double *ga[NITEM];
        bool in[NITEM], fr[NITEM];
        int64_t gv[NITEM];
        const unsigned sm_ = c_div_magic[nx2];
#pragma unroll
        for (int i = 0; i < NITEM; ++i) {
            // the compact mapping of FOR_RECT over the padded tile: the
            // first sweep's phase A reads exactly the cells its thread staged
            const int idx = t + i * NT;
            const int r = (int)(((unsigned)idx * sm_) >> 16), c = idx - r * nx2;
            in[i] = idx < ny2 * nx2;
            sa[i] = (unsigned)__cvta_generic_to_shared(&s.S[0][0]) + (r * PX + c) * 8;
            ga[i] = src + base + (int64_t)r * pv.NX + c;
            fr[i] = false;
            gv[i] = -1;
            if (gplan != nullptr && in[i]) {
                // halo cell in the patch's ghost frame: with a ghost plan the
                // sibling copy is fused into this staging -- read the covering
                // sibling's interior cell directly (ghost.py:186-196); cells
                // without a sibling (coarse interpolation, physical BC) come
                // from the frame the fill kernels wrote
                const int J = tj0 + 1 + r, I = ti0 + 1 + c;  // patch-array coordinates
                if (J < MLAMR_G || J >= pv.NY - MLAMR_G || I < MLAMR_G || I >= pv.NX - MLAMR_G) {
                    int gi;
                    if (J < MLAMR_G)
                        gi = J * pv.NX + I;
                    else if (J >= pv.NY - MLAMR_G)
                        gi = 2 * pv.NX + (J - (pv.NY - MLAMR_G)) * pv.NX + I;
                    else
                        gi = 4 * pv.NX + (J - MLAMR_G) * 4 + (I < MLAMR_G ? I : I - pv.NX + 4);
                    fr[i] = true;
                    gv[i] = gplan[gb + gi];
                }
            }
        }
        const int64_t boff = lv.bathy - src;  // same patch layout, one plane
        // cells whose address is known go first; the frame cells' plan
        // lookups (dependent loads) complete behind them
#pragma unroll
        for (int q = 0; q < 3 * M + 1; ++q) {
            const int64_t po = (q < 3 * M) ? q * FS : boff;
#pragma unroll
            for (int i = 0; i < NITEM; ++i)
                if (in[i] && !fr[i])
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa[i] + q * NPAD * 8),
                                 "l"(ga[i] + po));
        }
        if (gplan != nullptr) {
#pragma unroll
            for (int i = 0; i < NITEM; ++i) {
                if (!fr[i]) continue;
                const double *gs = gv[i] >= 0 ? src + gv[i] : ga[i];
#pragma unroll
                for (int q = 0; q < 3 * M + 1; ++q) {
                    // bathymetry always from the patch's own frame
                    const double *a = (q < 3 * M) ? gs + q * FS : ga[i] + boff;
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa[i] + q * NPAD * 8), "l"(a));
                }
            }
        }
    }
    asm volatile("cp.async.commit_group;\n" ::);
    if (st0 != 0) {  // an earlier kernel raised an error: nothing to do
        asm volatile("cp.async.wait_group 0;\n" ::);
        return;
    }
    const double(&rr)[4][4] = kc.rr;
    const double lam_x = kc.lam_x, lam_y = kc.lam_y;
    const double y_x = recip_nr(lv.dx), y_y = recip_nr(lv.dy);
    asm volatile("cp.async.wait_group 0;\n" ::);
    // no barrier here: the first sweep's phase A walks the padded tile with
    // the staging's own thread -> cell mapping (idx = t + i*NT), so every
    // thread reads only cells whose copies it issued and has waited for;
    // phase A's closing barrier publishes the tile to the other threads
    double best = -1.0;  // running observed speed over this thread's cells
    double nacc = 0.0;   // NaN iff a speed operand was NaN
    // each sweep takes the all-wet path when every cell it reads is wet in
    // every layer (~90 % of C4's level-3 tiles)
    // phase A of the first sweep runs the general path and finds out
    // whether the rest of that sweep can take the all-wet path; the
    // first sweep's update does the same for the second sweep
    constexpr int D1 = YFIRST ? 1 : 0, D2 = YFIRST ? 0 : 1;
    const double d1 = YFIRST ? lv.dy : lv.dx, d2 = YFIRST ? lv.dx : lv.dy;
    const double l1 = YFIRST ? lam_y : lam_x, l2 = YFIRST ? lam_x : lam_y;
    const double q1 = YFIRST ? y_y : y_x, q2 = YFIRST ? y_x : y_y;
    const bool aw1 = sweep_tile<M, D1, true, false, false, true, false>(s, ny2, nx2, dt, d1, l1, q1, prm, rr, best, nacc);
    // the first sweep's update also prepares the second sweep's inputs (NEXT)
    const bool aw2 = aw1 ? sweep_tile<M, D1, true, false, true, false, true, false, false, true>(
                               s, ny2, nx2, dt, d1, l1, q1, prm, rr, best, nacc)
                         : sweep_tile<M, D1, true, false, false, false, true, false, false, true>(
                               s, ny2, nx2, dt, d1, l1, q1, prm, rr, best, nacc);
    // post-processing on the tile interior (physics.py:360-376), fused into
    // the second sweep's update of exactly those cells
    PostCtx pc;
    pc.dst = dst;
    pc.base = base;
    pc.FS = FS;
    pc.NX = pv.NX;
    pc.tol = prm.dry_tolerance;
    pc.coef = kc.coef;
#pragma unroll
    for (int m = 0; m < MLAMR_MAX_LAYERS; ++m) pc.negs[m] = 0.0;
    pc.fixes = pc.repairs = 0;
    if (aw2)
        sweep_tile<M, D2, false, true, true, false, true, true, true>(s, ny2, nx2, dt, d2, l2, q2, prm, rr, best, nacc, &pc);
    else
        sweep_tile<M, D2, false, false, false, false, true, true, true>(s, ny2, nx2, dt, d2, l2, q2, prm, rr, best, nacc, &pc);

    // per-tile partials in one fused pass: warp shuffles (fixed xor tree),
    // then warp 0 combines the NT/32 warp values in warp order -- the same
    // order on every run, so the sums are deterministic
    constexpr int NW = NT / 32;
    const int lane = t & 31, warp = t >> 5;
    double v[M + 2];
#pragma unroll
    for (int m = 0; m < M; ++m) v[m] = pc.negs[m];
    v[M] = (double)pc.fixes;
    v[M + 1] = (double)pc.repairs;
    // negative-depth sums and counters are zero in almost every warp: the
    // shuffle tree runs only where one is not
    bool any = false;
#pragma unroll
    for (int q = 0; q < M + 2; ++q) any = any || (v[q] != 0.0);
    if (__any_sync(0xffffffffu, any)) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
            for (int q = 0; q < M + 2; ++q) v[q] = v[q] + __shfl_xor_sync(0xffffffffu, v[q], off);
        }
    } else {
#pragma unroll
        for (int q = 0; q < M + 2; ++q) v[q] = 0.0;
    }
    // speed max on the bit patterns: speeds are >= 0 (or NaN, canonicalised
    // above every finite value), and "no wet column" is -1, so the ordering
    // of the signed 64-bit patterns is the numpy maximum the reference takes
    if (nacc != nacc) best = nacc;
    const long long mybits = (best < 0.0) ? -1LL
                           : ((best != best) ? 0x7ff8000000000000LL : __double_as_longlong(best));
    const int hi = __reduce_max_sync(0xffffffffu, (int)(mybits >> 32));
    const unsigned lo = __reduce_max_sync(0xffffffffu, ((int)(mybits >> 32) == hi) ? (unsigned)mybits : 0u);
    if (lane == 0) {
#pragma unroll
        for (int q = 0; q < M + 2; ++q) s.red[q * NW + warp] = v[q];
        s.redi[warp] = (hi < 0) ? -1LL : (long long)(((unsigned long long)(unsigned)hi << 32) | lo);
    }
    __syncthreads();
    // one lane per quantity (each sums its warp values in warp order, so
    // the result is the serial sum's), the speed maximum on another warp:
    // the CTA's tail is one short chain instead of M+3 serial ones
    if (t < M + 2) {
        double a = s.red[t * NW];
#pragma unroll
        for (int w = 1; w < NW; ++w) a = a + s.red[t * NW + w];
        tile_acc[(int64_t)tile * (M + 2) + t] = a;
    } else if (t == 32) {
        long long b = s.redi[0];
#pragma unroll
        for (int w = 1; w < NW; ++w) b = max(b, s.redi[w]);
        if (b >= 0) atomicMax(speed_bits + p, b);
    }
}

// K6: observed max speed per patch without stepping (stable_dt, level 1 dt).
template <int M>
__global__ void __launch_bounds__(NTF) k_max_speed(mlamr_level lv, const double *__restrict__ st,
                                                  const int32_t *__restrict__ tiles,
                                                  mlamr_params prm, long long *speed_bits) {
    __shared__ double red[NTF];
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
    for (int idx = t; idx < ty * tx; idx += NTF) {
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
    for (int s2 = NTF / 2; s2 > 0; s2 >>= 1) {
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

template <int M>
static int launch_step(const mlamr_level &lv, const double *src, double *dst,
                       const TileDesc *desc, int n_tiles, double dt, int y_first,
                       const mlamr_params &prm, long long *speed_bits, double *tile_acc,
                       const int32_t *status, const int64_t *gplan, cudaStream_t st) {
    const size_t smem = sizeof(StepSmem<M>);
    // the shared-memory opt-in is a per-device function attribute
    constexpr int kMaxDev = 64;
    static bool configured[kMaxDev][2] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= kMaxDev) return -4;
    if (!configured[dev][y_first ? 1 : 0]) {
        cudaError_t e;
        if (y_first)
            e = cudaFuncSetAttribute(k_step<M, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        else
            e = cudaFuncSetAttribute(k_step<M, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return (int)e;
#ifdef MLAMR_STEP_CARVEOUT
        if (y_first)
            e = cudaFuncSetAttribute(k_step<M, true>, cudaFuncAttributePreferredSharedMemoryCarveout, MLAMR_STEP_CARVEOUT);
        else
            e = cudaFuncSetAttribute(k_step<M, false>, cudaFuncAttributePreferredSharedMemoryCarveout, MLAMR_STEP_CARVEOUT);
        if (e != cudaSuccess) return (int)e;
#endif
        configured[dev][y_first ? 1 : 0] = true;
    }
    if (n_tiles <= 0) return 0;
    StepConst kc;
    kc.lam_x = dt / lv.dx;
    kc.lam_y = dt / lv.dy;
    for (int a = 0; a < 4; ++a)
        for (int b = 0; b < 4; ++b)
            kc.rr[a][b] = (a < b && b < M) ? prm.densities[a] / prm.densities[b] : 0.0;
    kc.coef = (M > 1) ? prm.gravity * (1.0 - kc.rr[0][1]) : 0.0;
    if (y_first)
        k_step<M, true><<<n_tiles, NT, smem, st>>>(lv, src, dst, desc, dt, prm, kc, speed_bits, tile_acc, status,
                                                   gplan);
    else
        k_step<M, false><<<n_tiles, NT, smem, st>>>(lv, src, dst, desc, dt, prm, kc, speed_bits, tile_acc, status,
                                                    gplan);
    return (int)cudaGetLastError();
}

#undef FOR_RECT_BEGIN
#undef FOR_RECT_END

}  // namespace MLAMR_STEP_NS
