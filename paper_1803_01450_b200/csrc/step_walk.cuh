// K1, line-walker form: the batched patch step (physics.step_patch,
// physics.py:330-386) with each directional sweep done by threads that walk
// a short segment of one grid line through registers.  Included by
// k_step.cu inside `namespace mlamr` (StepConst, recip_nr, div_fast, ...).
//
// Why: the phase-per-cell form (step_tile.cuh) publishes every per-cell and
// per-interface intermediate (velocities, wave speeds, fluxes, sources,
// co-wet flags) through shared memory between block barriers, recomputes
// each cell's reconstructed face depths and transverse fluxes twice, and
// spends most of its instruction stream on index math, shared loads/stores
// and selects around ~35 % FP64 work.  A walker keeps a three-cell window
// in registers: per step it loads one cell, derives its layer inputs
// (_layer_inputs, physics.py:193-212), computes the flux of the interface
// it shares with the previous cell once (_sweep's interface loop,
// physics.py:101-161: HLL flux, reconstructed depths hsL/hsR, upwinded
// transverse flux) and updates the previous cell from its two interfaces
// (physics.py:162-169 plus the coupling source added afterwards,
// physics.py:235-237/256-258).  Only the state travels through shared
// memory: the staged tile (S) and the first sweep's output (T).
//
// Geometry: the same 16x32 interior tiles (and tile list) as the wide
// phase kernel, staged with a one-cell halo (the step reads ghost width 1,
// SURVEY.md App. C probe 3).  The first sweep runs on every line of the
// padded tile (the reference's full=True sweep over the ghost rows), the
// second on the interior lines.  A line of n cells has n-2 updated cells,
// cut into segments of K; a segment's walker reads cells a-1 .. a+K, so
// segment ends are recomputed by both neighbours (idempotent: same inputs,
// same IEEE operations).
//
// Arithmetic is operation for operation the phase kernel's (and so the
// reference's), compiled with -fmad=false; the all-wet specialisation
// (every cell a sweep reads wet in every layer, tol < h < 1e150) is the
// same proof as step_tile.cuh's AW path.

namespace walk {

using wide::PostCtx;
using wide::post_cell;

constexpr int TX = 32;            // interior tile columns (= wide::TX, same tile list)
constexpr int TY = 16;            // interior tile rows
constexpr int PX = TX + 2;        // padded row length
constexpr int PY = TY + 2;        // padded rows
constexpr int PXS = PX + 1;       // shared row pitch (odd: column walks are conflict-free)
constexpr int NPAD = PY * PXS;
#ifndef MLAMR_WALK_K
#define MLAMR_WALK_K 4
#endif
constexpr int K = MLAMR_WALK_K;   // updated cells per walker segment
#ifndef MLAMR_WALK_NT
#define MLAMR_WALK_NT 160
#endif
#ifndef MLAMR_WALK_MINB
#define MLAMR_WALK_MINB 3
#endif
constexpr int NT = MLAMR_WALK_NT;
constexpr int NW = NT / 32;
static_assert(PY * ((TX + K - 1) / K) <= NT, "first x sweep must fit one segment per thread");
static_assert(PX * ((TY + K - 1) / K) <= NT, "first y sweep must fit one segment per thread");

template <int M>
struct Smem {
    double S[3 * M + 1][NPAD];  // staged state h_0.., hu_0.., hv_0.., B
    double T[3 * M][NPAD];      // state after the first sweep
    double red[(M + 2) * NW];
    long long redi[NW];
};

// One cell's layer inputs for one sweep direction (_layer_inputs,
// physics.py:193-212, and the velocities of _sweep, physics.py:104-105, 153-154).
template <int M>
struct Cell {
    double h[M], hn[M], ht[M];        // depth, normal and transverse momentum
    double B;
    double cw;                        // sqrt(g * max(sum h, 0))
    double eb[M > 1 ? M - 1 : 1];     // eta_{m+1} = B + h_{M-1} + ... + h_{m+1}
    double u[M], v[M];                // normal / transverse velocity (0 where dry)
    bool cowet;                       // every layer wet (M = 1: always)
};

// Bottoms of layer m (physics.py:200-207): co-wet pairs use Zc (0 for upper
// layers, B for the bottom one), others Zf = Bhat (eta_{m+1}, or B).
template <int M>
__device__ __forceinline__ double zc(const Cell<M> &c, int m) { return (m == M - 1) ? c.B : 0.0; }
template <int M>
__device__ __forceinline__ double zf(const Cell<M> &c, int m) { return (m == M - 1) ? c.B : c.eb[m < M - 1 ? m : 0]; }

// Interface quantities of layer m kept for the two cells that share it.
struct Face {
    double fh, fm, fv;   // mass, normal-momentum and upwinded transverse flux
    double hL, hR;       // reconstructed depths (hsL, hsR of _sweep)
};

// Load one cell from plane set P (h, hu, hv per layer) and B from S, and
// derive its layer inputs.  SPEED: observed_max_speed's running maximum
// over this cell (first sweep, tile-interior cells; physics.py:261-278):
// max_m(max(|u_m|,|v_m|)) + cw, bit-identical to the reference by monotone
// rounding (see step_tile.cuh phase A); NaN-ness travels in nacc.
template <int M, int DIR, bool AW>
__device__ __forceinline__ void load_cell(Cell<M> &c, const double (*P)[NPAD], const double *Bp, int k,
                                          double g, double tol, bool speed, double &best, double &nacc) {
    double hs = 0.0;
    bool w = true;
#pragma unroll
    for (int m = 0; m < M; ++m) {
        c.h[m] = P[m][k];
        c.hn[m] = P[(DIR == 0 ? M : 2 * M) + m][k];
        c.ht[m] = P[(DIR == 0 ? 2 * M : M) + m][k];
        hs = hs + c.h[m];
        w = w && (c.h[m] > tol);
    }
    c.B = Bp[k];
    // AW: hs > tol > 0, so numpy's maximum(hs, 0) is hs
    c.cw = sqrt(g * (AW ? hs : np_max(hs, 0.0)));
    c.cowet = (M == 1) ? true : (AW ? true : w);
    if (M > 1) {
        double e = c.B;
#pragma unroll
        for (int m = M - 1; m >= 1; --m) {
            e = e + c.h[m];
            c.eb[m - 1] = e;
        }
    }
    const bool sp = speed && (AW || hs > tol);
#pragma unroll
    for (int m = 0; m < M; ++m) {
        double u = 0.0, v = 0.0;
        if (AW || c.h[m] > tol) {
            bool ok = true;
            const double y = recip_nr(c.h[m]);
            u = div_fast(c.hn[m], c.h[m], y, ok);
            v = div_fast(c.ht[m], c.h[m], y, ok);
            if (!ok) {
                u = c.hn[m] / c.h[m];
                v = c.ht[m] / c.h[m];
            }
        }
        c.u[m] = u;
        c.v[m] = v;
        if (sp) {
            const double au = fabs(u), av = fabs(v);
            best = fmax(best, fmax(au, av) + c.cw);
            nacc = nacc + (au + av);
        }
    }
}

// The interface between cells l and r, layer m (physics.py:101-161).
template <int M, bool AW>
__device__ __forceinline__ void face(Face &f, const Cell<M> &l, const Cell<M> &r, int m, double g) {
    const bool cop = AW || (l.cowet && r.cowet);
    const double hl = l.h[m], hr = r.h[m];
    const double ul = l.u[m], ur = r.u[m];
    double hL, hR;
    if (AW && m < M - 1) {
        hL = hl;
        hR = hr;
    } else {
        const double Zl = cop ? zc<M>(l, m) : zf<M>(l, m);
        const double Zr = cop ? zc<M>(r, m) : zf<M>(r, m);
        const double Zs = Zl > Zr ? Zl : Zr;
        hL = (hl + Zl) - Zs;
        if (hL < 0.0) hL = 0.0;
        hR = (hr + Zr) - Zs;
        if (hR < 0.0) hR = 0.0;
    }
    f.hL = hL;
    f.hR = hR;
    double fh = 0.0, fm = 0.0;
    if ((AW && m < M - 1) || !(hL <= 0.0 && hR <= 0.0)) {
        const double cl = l.cw, cr = r.cw;
        const double sl1 = ul - cl, sl2 = ur - cr;
        const double SL = sl1 < sl2 ? sl1 : sl2;
        const double sr1 = ul + cl, sr2 = ur + cr;
        const double SR = sr1 > sr2 ? sr1 : sr2;
        const double FLh = hL * ul;
        const double FRh = hR * ur;
        const double FLm = ((hL * ul) * ul) + (((0.5 * g) * hL) * hL);
        const double FRm = ((hR * ur) * ur) + (((0.5 * g) * hR) * hR);
        if (SL >= 0.0) {
            fh = FLh;
            fm = FLm;
        } else if (SR <= 0.0) {
            fh = FRh;
            fm = FRm;
        } else {
            const double den = SR - SL;
            double djump;
            if ((AW && m < M - 1) || (hL > 0.0 && hR > 0.0))
                djump = (hr + zf<M>(r, m)) - (hl + zf<M>(l, m));
            else
                djump = hR - hL;
            const double nh = ((SR * FLh) - (SL * FRh)) + ((SL * SR) * djump);
            const double nm = ((SR * FLm) - (SL * FRm)) + ((SL * SR) * ((hR * ur) - (hL * ul)));
            bool ok = true;
            const double y = recip_nr(den);
            fh = div_fast(nh, den, y, ok);
            fm = div_fast(nm, den, y, ok);
            if (!ok) {
                fh = nh / den;
                fm = nm / den;
            }
        }
    }
    f.fh = fh;
    f.fm = fm;
    // upwinded transverse flux (physics.py:153-161); fh == +-0 or NaN gives +0
    f.fv = fabs(fh) > 0.0 ? fh * (fh > 0.0 ? l.v[m] : r.v[m]) : 0.0;
}

// Masked centred gradient of a field at cell c (physics.py:172-186) times
// 0.5, from its two neighbours; pairs that are not co-wet contribute 0.
__device__ __forceinline__ double half_grad(double fm1, double f0, double fp1, bool wm, bool wp) {
    const double dm = wm ? f0 - fm1 : 0.0;
    const double dp = wp ? fp1 - f0 : 0.0;
    return 0.5 * (dp + dm);
}

// Update of the middle cell c from its faces (physics.py:162-169), plus the
// coupling source of this direction (physics.py:208-211; M >= 2 generalised
// as in step_tile.cuh): results into nh/nn/nt (depth, normal, transverse).
template <int M, bool AW>
__device__ __forceinline__ void update(const Cell<M> &a, const Cell<M> &c, const Cell<M> &b,
                                       const Face (&fl)[M], const Face (&fr)[M], double lam, double dt,
                                       double g, double d, double yd, const double (&rr)[4][4],
                                       double (&nh)[M], double (&nn)[M], double (&nt)[M]) {
    const bool wm = AW || (a.cowet && c.cowet);
    const bool wp = AW || (c.cowet && b.cowet);
#pragma unroll
    for (int m = 0; m < M; ++m) {
        const double h0 = c.h[m];
        nh[m] = h0 - lam * (fr[m].fh - fl[m].fh);
        double hn;
        if (AW && m < M - 1) {
            // both faces reconstruct to h0: the pressure correction is exactly +0
            hn = c.hn[m] - lam * (fr[m].fm - fl[m].fm);
        } else {
            hn = (c.hn[m] - lam * (fr[m].fm - fl[m].fm)) -
                 (((lam * 0.5) * g) * ((fl[m].hR * fl[m].hR) - (fr[m].hL * fr[m].hL)));
        }
        if (M > 1) {
            double acc = 0.0;
            bool has = false;
            if (m < M - 1) {
                const int e = m < M - 1 ? m : 0;
                const double num = ((-g) * h0) * half_grad(a.eb[e], c.eb[e], b.eb[e], wm, wp);
                bool ok = true;
                double q = div_fast(num, d, yd, ok);
                if (!ok) q = num / d;
                acc = q;
                has = true;
            }
#pragma unroll
            for (int kk = 0; kk < m; ++kk) {
                const double num = (((-rr[kk][m]) * g) * h0) * half_grad(a.h[kk], c.h[kk], b.h[kk], wm, wp);
                bool ok = true;
                double q = div_fast(num, d, yd, ok);
                if (!ok) q = num / d;
                acc = has ? acc + q : q;
                has = true;
            }
            hn = hn + dt * acc;
        }
        nn[m] = hn;
        nt[m] = c.ht[m] - lam * (fr[m].fv - fl[m].fv);
    }
}

// One sweep over the lines of the tile.  DIR 0 = x (lines are rows), 1 = y.
// FIRST: all lines of the padded tile, output into T; else interior lines,
// post-processed and stored to global memory (LAST).  Returns whether
// every updated cell is wet in every layer (FIRST only; block-wide).
template <int M, int DIR, bool FIRST, bool AW>
__device__ __forceinline__ bool sweep(Smem<M> &s, int ny2, int nx2, double dt, double d, double lam, double yd,
                                      const mlamr_params &prm, const double (&rr)[4][4], double &best,
                                      double &nacc, PostCtx *post) {
    const double g = prm.gravity, tol = prm.dry_tolerance;
    const double (*P)[NPAD] = FIRST ? s.S : s.T;
    const double *Bp = s.S[3 * M];
    const int n_along = DIR == 0 ? nx2 : ny2;
    const int nlines = FIRST ? (DIR == 0 ? ny2 : nx2) : (DIR == 0 ? ny2 - 2 : nx2 - 2);
    const int line0 = FIRST ? 0 : 1;
    const int nseg = (n_along - 2 + K - 1) / K;
    const int t = threadIdx.x;
    bool wet_out = true;
    if (t < nlines * nseg) {
        // lines vary fastest across threads: x walks then touch one cell per
        // row (odd pitch: conflict-free), y walks consecutive columns
        const int seg = t / nlines;
        const int line = line0 + (t - seg * nlines);
        const int a = 1 + seg * K;                 // first updated cell
        const int kv = min(K, n_along - 1 - a);    // updated cells in this segment
        const int kstep = DIR == 0 ? 1 : PXS;
        const int k0 = DIR == 0 ? line * PXS + (a - 1) : (a - 1) * PXS + line;
        const bool sp_line = FIRST && line >= 1 && line < (DIR == 0 ? ny2 : nx2) - 1;
        Cell<M> c0, c1, c2;
        Face fl[M], fr[M];
        // one rolled loop (the step body is large: unrolled walks overflowed
        // the instruction cache); step j loads cell j, forms the face
        // (j-1, j) and updates cell j-1
#pragma unroll 1
        for (int j = 0; j <= kv + 1; ++j) {
            const int kj = k0 + j * kstep;
            const int cj = a - 1 + j;                 // along-line index of cell j
            load_cell<M, DIR, AW>(c2, P, Bp, kj, g, tol, sp_line && cj >= 1 && cj < n_along - 1, best, nacc);
            if (j >= 1) {
#pragma unroll
                for (int m = 0; m < M; ++m) face<M, AW>(fr[m], c1, c2, m, g);
            }
            if (j >= 2) {
                double nh[M], nn[M], nt[M];
                update<M, AW>(c0, c1, c2, fl, fr, lam, dt, g, d, yd, rr, nh, nn, nt);
                const int kc = kj - kstep;            // the updated cell
                if (FIRST) {
#pragma unroll
                    for (int m = 0; m < M; ++m) {
                        s.T[m][kc] = nh[m];
                        s.T[(DIR == 0 ? M : 2 * M) + m][kc] = nn[m];
                        s.T[(DIR == 0 ? 2 * M : M) + m][kc] = nt[m];
                        wet_out = wet_out & (nh[m] > tol) & (nh[m] < 1e150);
                    }
                } else {
                    const int r = DIR == 0 ? line : cj - 1;
                    const int c = DIR == 0 ? cj - 1 : line;
                    if (DIR == 0) post_cell<M>(nh, nn, nt, *post, r, c);
                    else post_cell<M>(nh, nt, nn, *post, r, c);
                }
            }
            c0 = c1;
            c1 = c2;
#pragma unroll
            for (int m = 0; m < M; ++m) fl[m] = fr[m];
        }
    }
    if (!FIRST) return true;
    return __syncthreads_and(wet_out) != 0;
}

template <int M, bool YFIRST>
__global__ void __launch_bounds__(NT, MLAMR_WALK_MINB) k_step(mlamr_level lv, const double *__restrict__ src,
                                                              double *__restrict__ dst,
                                                              const int32_t *__restrict__ tiles, double dt,
                                                              mlamr_params prm, StepConst kc, long long *speed_bits,
                                                              double *tile_acc, const int32_t *status,
                                                              const int64_t *__restrict__ gbase,
                                                              const int64_t *__restrict__ gplan) {
    const int32_t st0 = status != nullptr ? *status : 0;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem<M> &s = *reinterpret_cast<Smem<M> *>(smem_raw);
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
    const double tol = prm.dry_tolerance;

    // stage the padded tile with asynchronous 8-byte copies (as the phase
    // kernel, with the sibling ghost copy fused through the ghost plan)
    constexpr int NITEM = (PY * PX + NT - 1) / NT;
    bool in[NITEM];
    unsigned sa[NITEM];
    {
        const double *ga[NITEM];
        bool fr[NITEM];
        int64_t gv[NITEM];
#pragma unroll
        for (int i = 0; i < NITEM; ++i) {
            const int idx = t + i * NT;
            const int r = idx / PX, c = idx - (idx / PX) * PX;
            in[i] = idx < ny2 * PX && c < nx2;
            sa[i] = (unsigned)__cvta_generic_to_shared(&s.S[0][0]) + (r * PXS + c) * 8;
            ga[i] = src + base + (int64_t)r * pv.NX + c;
            fr[i] = false;
            gv[i] = -1;
            if (gplan != nullptr && in[i]) {
                const int J = tj0 + 1 + r, I = ti0 + 1 + c;
                if (J < MLAMR_G || J >= pv.NY - MLAMR_G || I < MLAMR_G || I >= pv.NX - MLAMR_G) {
                    int gi;
                    if (J < MLAMR_G)
                        gi = J * pv.NX + I;
                    else if (J >= pv.NY - MLAMR_G)
                        gi = 2 * pv.NX + (J - (pv.NY - MLAMR_G)) * pv.NX + I;
                    else
                        gi = 4 * pv.NX + (J - MLAMR_G) * 4 + (I < MLAMR_G ? I : I - pv.NX + 4);
                    fr[i] = true;
                    gv[i] = gplan[gbase[p] + gi];
                }
            }
        }
        const int64_t boff = lv.bathy - src;
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
                    const double *a = (q < 3 * M) ? gs + q * FS : ga[i] + boff;
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa[i] + q * NPAD * 8), "l"(a));
                }
            }
        }
    }
    asm volatile("cp.async.commit_group;\n" ::);
    if (st0 != 0) {
        asm volatile("cp.async.wait_group 0;\n" ::);
        return;
    }
    const double(&rr)[4][4] = kc.rr;
    const double y_x = recip_nr(lv.dx), y_y = recip_nr(lv.dy);
    asm volatile("cp.async.wait_group 0;\n" ::);
    // all-wet test of the first sweep over the cells this thread staged;
    // the block-wide vote is also the barrier that publishes the tile
    bool wet_in = true;
#pragma unroll
    for (int i = 0; i < NITEM; ++i) {
        if (!in[i]) continue;
        const int off = (int)((sa[i] - (unsigned)__cvta_generic_to_shared(&s.S[0][0])) / 8);
#pragma unroll
        for (int m = 0; m < M; ++m) {
            const double h = s.S[m][off];
            wet_in = wet_in & (h > tol) & (h < 1e150);
        }
    }
    const bool aw1 = __syncthreads_and(wet_in) != 0;

    double best = -1.0, nacc = 0.0;
    constexpr int D1 = YFIRST ? 1 : 0, D2 = YFIRST ? 0 : 1;
    const double d1 = YFIRST ? lv.dy : lv.dx, d2 = YFIRST ? lv.dx : lv.dy;
    const double l1 = YFIRST ? kc.lam_y : kc.lam_x, l2 = YFIRST ? kc.lam_x : kc.lam_y;
    const double q1 = YFIRST ? y_y : y_x, q2 = YFIRST ? y_x : y_y;
    const bool aw2 = aw1 ? sweep<M, D1, true, true>(s, ny2, nx2, dt, d1, l1, q1, prm, rr, best, nacc, nullptr)
                         : sweep<M, D1, true, false>(s, ny2, nx2, dt, d1, l1, q1, prm, rr, best, nacc, nullptr);
    PostCtx pc;
    pc.dst = dst;
    pc.base = base;
    pc.FS = FS;
    pc.NX = pv.NX;
    pc.tol = tol;
    pc.coef = kc.coef;
#pragma unroll
    for (int m = 0; m < MLAMR_MAX_LAYERS; ++m) pc.negs[m] = 0.0;
    pc.fixes = pc.repairs = 0;
    if (aw2)
        sweep<M, D2, false, true>(s, ny2, nx2, dt, d2, l2, q2, prm, rr, best, nacc, &pc);
    else
        sweep<M, D2, false, false>(s, ny2, nx2, dt, d2, l2, q2, prm, rr, best, nacc, &pc);

    // per-tile partials (same reduction as the phase kernel)
    const int lane = t & 31, warp = t >> 5;
    double v[M + 2];
#pragma unroll
    for (int m = 0; m < M; ++m) v[m] = pc.negs[m];
    v[M] = (double)pc.fixes;
    v[M + 1] = (double)pc.repairs;
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

template <int M>
static int launch_step(const mlamr_level &lv, const double *src, double *dst, const int32_t *tiles, int n_tiles,
                       double dt, int y_first, const mlamr_params &prm, long long *speed_bits, double *tile_acc,
                       const int32_t *status, const int64_t *gbase, const int64_t *gplan, cudaStream_t st) {
    const size_t smem = sizeof(Smem<M>);
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
        k_step<M, true><<<n_tiles, NT, smem, st>>>(lv, src, dst, tiles, dt, prm, kc, speed_bits, tile_acc, status,
                                                   gbase, gplan);
    else
        k_step<M, false><<<n_tiles, NT, smem, st>>>(lv, src, dst, tiles, dt, prm, kc, speed_bits, tile_acc, status,
                                                    gbase, gplan);
    return (int)cudaGetLastError();
}

}  // namespace walk
