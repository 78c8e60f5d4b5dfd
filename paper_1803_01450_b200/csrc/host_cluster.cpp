// Host-side clustering of refinement flags (regrid.cluster_flags,
// regrid.py:129-182 of /root/reference/pkg/src/mlamr), native C++.
//
// Same recursive bisection and cut preference (hole > inflection >
// midpoint, regrid._signature_cut, regrid.py:104-126) and the same output
// order, but every signature, bounding box, flag count and "all allowed"
// test is answered from prefix sums in O(width + height) instead of
// re-scanning the sub-array, so a 2048^2 flag map clusters in milliseconds.

#include <algorithm>
#include <array>
#include <cstdint>
#include <cstdlib>
#include <vector>

namespace {

struct Cut {
    int index;
    int quality;
    bool valid;
};

Cut signature_cut(const std::vector<int64_t> &sig) {
    const int n = (int)sig.size();
    if (n < 2) return {0, 0, false};
    // widest interior run of zeros (first of the widest on ties)
    int best_lo = -1, best_len = 0;
    int k = 0;
    while (k < n) {
        if (sig[k] != 0) {
            ++k;
            continue;
        }
        int e = k;
        while (e + 1 < n && sig[e + 1] == 0) ++e;
        if (k > 0 && e < n - 1) {
            const int len = e - k + 1;
            if (len > best_len) {
                best_len = len;
                best_lo = k;
            }
        }
        k = e + 1;
    }
    if (best_len > 0) return {best_lo + best_len / 2, 2, true};
    if (n >= 4) {
        int64_t best = 0;
        int arg = -1;
        int64_t prev = sig[2] - 2 * sig[1] + sig[0];
        for (int q = 1; q + 2 < n; ++q) {
            const int64_t d2 = sig[q + 2] - 2 * sig[q + 1] + sig[q];
            const int64_t jump = std::llabs(d2 - prev);
            if (jump > best) {
                best = jump;
                arg = q - 1;
            }
            prev = d2;
        }
        if (arg >= 0 && best > 0) return {arg + 2, 1, true};
    }
    return {n / 2, 0, true};
}

// One int32 summed-area table answers every query: box counts in O(1) and
// row/column signatures in O(1) per entry.  The table lives in a reusable
// buffer so repeated regrids do not pay for fresh pages.
struct Prefix {
    int ny = 0, nx = 0;
    std::vector<int32_t> *sat = nullptr;  // (ny+1) x (nx+1)
    const int32_t *ext = nullptr;         // external table (device-built), same layout
    void wrap(const int32_t *table, int ny_, int nx_) {
        ny = ny_;
        nx = nx_;
        ext = table;
    }
    void build(const uint8_t *m, int ny_, int nx_, std::vector<int32_t> &store) {
        ny = ny_;
        nx = nx_;
        sat = &store;
        const size_t W = (size_t)nx + 1;
        if (store.size() < (size_t)(ny + 1) * W) store.resize((size_t)(ny + 1) * W);
        int32_t *S = store.data();
        // row prefix sums (independent rows), then a column scan in blocks of
        // 256 columns (each thread walks its block down the rows)
#pragma omp parallel for schedule(static)
        for (int j = -1; j < ny; ++j) {
            int32_t *cur = S + (size_t)(j + 1) * W;
            cur[0] = 0;
            if (j < 0) {
                for (int i = 0; i < nx; ++i) cur[i + 1] = 0;
                continue;
            }
            const uint8_t *row = m + (size_t)j * nx;
            int32_t rs = 0;
            for (int i = 0; i < nx; ++i) {
                rs += row[i] ? 1 : 0;
                cur[i + 1] = rs;
            }
        }
        const int nblk = (nx + 255) / 256;
#pragma omp parallel for schedule(static)
        for (int bk = 0; bk < nblk; ++bk) {
            const int i0 = 1 + bk * 256, i1 = std::min(nx, bk * 256 + 256);
            for (int j = 1; j < ny; ++j) {
                const int32_t *up = S + (size_t)j * W;
                int32_t *cur = S + (size_t)(j + 1) * W;
                for (int i = i0; i <= i1; ++i) cur[i] += up[i];
            }
        }
    }
    inline int64_t box(int i0, int j0, int i1, int j1) const {
        const size_t W = (size_t)nx + 1;
        const int32_t *S = ext ? ext : sat->data();
        return (int64_t)S[(size_t)(j1 + 1) * W + i1 + 1] - S[(size_t)j0 * W + i1 + 1] -
               S[(size_t)(j1 + 1) * W + i0] + S[(size_t)j0 * W + i0];
    }
    inline int64_t colsum(int i, int j0, int j1) const { return box(i, j0, i, j1); }
    inline int64_t rowsum(int j, int i0, int i1) const { return box(i0, j, i1, j); }
};

}  // namespace

// One node of the bisection: trim to the flags' bounding box, accept it
// (efficiency, or a single cell, or no valid cut) or split it in two.
// Returns 0 (dropped: no flags), 1 (accepted into `out`), 2 (split into
// l and r).
struct Node { int i0, j0, i1, j1; };

static int cluster_node(const Prefix &F, const Prefix *BADp, double eff, const Node &nd, std::array<int, 4> &out,
                        Node &l, Node &r, std::vector<int64_t> &sx, std::vector<int64_t> &sy) {
    if (F.box(nd.i0, nd.j0, nd.i1, nd.j1) == 0) return 0;
    int a_j = nd.j0, b_j = nd.j1, a_i = nd.i0, b_i = nd.i1;
    while (F.rowsum(a_j, nd.i0, nd.i1) == 0) ++a_j;
    while (F.rowsum(b_j, nd.i0, nd.i1) == 0) --b_j;
    while (F.colsum(a_i, nd.j0, nd.j1) == 0) ++a_i;
    while (F.colsum(b_i, nd.j0, nd.j1) == 0) --b_i;
    const int64_t nflag = F.box(a_i, a_j, b_i, b_j);
    const int w = b_i - a_i + 1, h = b_j - a_j + 1;
    const int64_t area = (int64_t)w * h;
    const bool ok = BADp == nullptr || BADp->box(a_i, a_j, b_i, b_j) == 0;
    out = {a_i, a_j, b_i, b_j};
    if (area == 1 || (ok && (double)nflag >= eff * (double)area)) return 1;
    sx.resize(w);
    sy.resize(h);
    for (int i = 0; i < w; ++i) sx[i] = F.colsum(a_i + i, a_j, b_j);
    for (int j = 0; j < h; ++j) sy[j] = F.rowsum(a_j + j, a_i, b_i);
    const Cut cx = signature_cut(sx);
    const Cut cy = signature_cut(sy);
    if (!cx.valid && !cy.valid) return 1;
    const int qx = cx.valid ? cx.quality : -1, nxs = cx.valid ? w : 0;
    const int qy = cy.valid ? cy.quality : -1, nys = cy.valid ? h : 0;
    const bool cut_x = (qx > qy) || (qx == qy && nxs >= nys);
    if (cut_x) {
        l = {a_i, a_j, a_i + cx.index - 1, b_j};
        r = {a_i + cx.index, a_j, b_i, b_j};
    } else {
        l = {a_i, a_j, b_i, a_j + cy.index - 1};
        r = {a_i, a_j + cy.index, b_i, b_j};
    }
    return 2;
}

// Sub-trees below this many cells are bisected by the task that reached them.
constexpr int64_t kTaskCells = 1 << 14;

static void cluster_subtree(const Prefix &F, const Prefix *BADp, double eff, Node root,
                            std::vector<std::array<int, 4>> &boxes) {
    std::vector<Node> stack{root};
    std::vector<int64_t> sx, sy;
    while (!stack.empty()) {
        const Node nd = stack.back();
        stack.pop_back();
        std::array<int, 4> bx;
        Node l, r;
        const int k = cluster_node(F, BADp, eff, nd, bx, l, r, sx, sy);
        if (k == 1) boxes.push_back(bx);
        if (k == 2) {
            stack.push_back(r);
            stack.push_back(l);
        }
    }
}

// The bisection tree is walked by OpenMP tasks down to kTaskCells-sized
// nodes, each finishing its sub-tree serially into its own list.  The
// accepted boxes are disjoint, so the final (lo_j, lo_i) sort fixes one
// order whatever the traversal -- the reference's order (regrid.py:182).
static void cluster_task(const Prefix &F, const Prefix *BADp, double eff, Node nd,
                         std::vector<std::vector<std::array<int, 4>>> &lists) {
    if ((int64_t)(nd.i1 - nd.i0 + 1) * (nd.j1 - nd.j0 + 1) <= kTaskCells) {
        std::vector<std::array<int, 4>> mine;
        cluster_subtree(F, BADp, eff, nd, mine);
#pragma omp critical(mlamr_cluster_lists)
        lists.push_back(std::move(mine));
        return;
    }
    std::vector<int64_t> sx, sy;
    std::array<int, 4> bx;
    Node l, r;
    const int k = cluster_node(F, BADp, eff, nd, bx, l, r, sx, sy);
    if (k == 1) {
#pragma omp critical(mlamr_cluster_lists)
        lists.push_back({bx});
    } else if (k == 2) {
#pragma omp task default(none) firstprivate(l, eff, BADp) shared(F, lists)
        cluster_task(F, BADp, eff, l, lists);
#pragma omp task default(none) firstprivate(r, eff, BADp) shared(F, lists)
        cluster_task(F, BADp, eff, r, lists);
    }
}

static int cluster_recursion(const Prefix &F, const Prefix *BADp, int ny, int nx, double eff,
                             int32_t *out_boxes, int max_boxes) {
    std::vector<std::vector<std::array<int, 4>>> lists;
    if (ny > 0 && nx > 0) {
        const Node root{0, 0, nx - 1, ny - 1};
#pragma omp parallel default(none) shared(F, BADp, eff, root, lists)
#pragma omp single
        cluster_task(F, BADp, eff, root, lists);
    }
    std::vector<std::array<int, 4>> boxes;
    for (auto &v : lists) boxes.insert(boxes.end(), v.begin(), v.end());
    std::sort(boxes.begin(), boxes.end(), [](const std::array<int, 4> &a, const std::array<int, 4> &b) {
        return a[1] != b[1] ? a[1] < b[1] : a[0] < b[0];
    });
    if ((int)boxes.size() > max_boxes) return -1;
    for (size_t k = 0; k < boxes.size(); ++k)
        for (int q = 0; q < 4; ++q) out_boxes[4 * k + q] = boxes[k][q];
    return (int)boxes.size();
}

// Returns the number of boxes written to out_boxes [n*4] as (lo_i, lo_j,
// hi_i, hi_j) sorted by (lo_j, lo_i); -1 if more than max_boxes; -2 if a
// flag lies outside `allowed` (the reference raises ValueError).
extern "C" int mlamr_cluster_flags(const uint8_t *flags, int ny, int nx, double eff,
                                   const uint8_t *allowed, int32_t *out_boxes, int max_boxes) {
    static thread_local std::vector<int32_t> store_f, store_b;
    static thread_local std::vector<uint8_t> bad;
    Prefix F;
    F.build(flags, ny, nx, store_f);
    Prefix BAD;
    if (allowed != nullptr) {
        bad.resize((size_t)ny * nx);
        uint8_t *badp = bad.data();  // thread_local storage: hand the pointer to the team
        int outside = 0;
        const int64_t n = (int64_t)ny * nx;
#pragma omp parallel for schedule(static) reduction(|| : outside)
        for (int64_t k = 0; k < n; ++k) {
            badp[k] = allowed[k] ? 0 : 1;
            outside = outside || (flags[k] && !allowed[k]);
        }
        if (outside) return -2;
        BAD.build(bad.data(), ny, nx, store_b);
    }
    return cluster_recursion(F, allowed != nullptr ? &BAD : nullptr, ny, nx, eff, out_boxes, max_boxes);
}

// Same clustering from summed-area tables built elsewhere (the device):
// sat_flags / sat_bad are int32 (ny+1) x (nx+1), zero first row/column;
// sat_bad counts cells outside `allowed` (NULL = everything allowed).
extern "C" int mlamr_cluster_sat(const int32_t *sat_flags, const int32_t *sat_bad, int ny, int nx, double eff,
                                 int32_t *out_boxes, int max_boxes) {
    Prefix F, BAD;
    F.wrap(sat_flags, ny, nx);
    if (sat_bad != nullptr) BAD.wrap(sat_bad, ny, nx);
    return cluster_recursion(F, sat_bad != nullptr ? &BAD : nullptr, ny, nx, eff, out_boxes, max_boxes);
}

// Harness max-patch-size chop of clustered boxes: each
// box is cut into tiles of at most max_nx x max_ny cells, from the box
// corner or (aligned) at global multiples of the tile size; output sorted by
// (lo_j, lo_i).  Returns the count, or -1 if it exceeds cap.
extern "C" int mlamr_chop_boxes(const int32_t *boxes, int n, int max_nx, int max_ny, int aligned,
                                int32_t *out, int cap) {
    std::vector<std::array<int, 4>> res;
    for (int k = 0; k < n; ++k) {
        const int lo_i = boxes[4 * k], lo_j = boxes[4 * k + 1], hi_i = boxes[4 * k + 2], hi_j = boxes[4 * k + 3];
        for (int j = lo_j; j <= hi_j;) {
            const int nj = aligned ? (j / max_ny + 1) * max_ny : j + max_ny;
            const int j1 = std::min(nj - 1, hi_j);
            for (int i = lo_i; i <= hi_i;) {
                const int ni = aligned ? (i / max_nx + 1) * max_nx : i + max_nx;
                res.push_back({i, j, std::min(ni - 1, hi_i), j1});
                i = ni;
            }
            j = nj;
        }
    }
    std::stable_sort(res.begin(), res.end(), [](const std::array<int, 4> &a, const std::array<int, 4> &b) {
        return a[1] != b[1] ? a[1] < b[1] : a[0] < b[0];
    });
    if ((int)res.size() > cap) return -1;
    for (size_t k = 0; k < res.size(); ++k)
        for (int q = 0; q < 4; ++q) out[4 * k + q] = res[k][q];
    return (int)res.size();
}

// Step tile list (device.tile_list): (patch, j0, i0) for every tile_y x
// tile_x interior tile of every box, patch-major, rows of tiles in order.
// Returns the count; out may be NULL to count only.
extern "C" long long mlamr_tile_list(const int64_t *boxes, int n, int tile_y, int tile_x, int32_t *out) {
    long long t = 0;
    for (int p = 0; p < n; ++p) {
        const int64_t nx = boxes[4 * p + 2] - boxes[4 * p] + 1, ny = boxes[4 * p + 3] - boxes[4 * p + 1] + 1;
        const int tx = (int)((nx + tile_x - 1) / tile_x), ty = (int)((ny + tile_y - 1) / tile_y);
        if (out != nullptr)
            for (int a = 0; a < ty; ++a)
                for (int b = 0; b < tx; ++b) {
                    out[3 * t] = p;
                    out[3 * t + 1] = a * tile_y;
                    out[3 * t + 2] = b * tile_x;
                    ++t;
                }
        else
            t += (long long)tx * ty;
    }
    return t;
}

// For each box of `a` (int64 [na][4], inclusive), does it intersect any box
// of `b`?  Bucket grid over b's extent (cell `bucket`), CSR of box ids per
// bucket, exact tests on candidates.  Host-side planning for multi-GPU
// shadow sets (distributed.py).
extern "C" int mlamr_boxes_meet_any(const int64_t *a, int na, const int64_t *b, int nb, int bucket,
                                    uint8_t *out) {
    for (int k = 0; k < na; ++k) out[k] = 0;
    if (na == 0 || nb == 0) return 0;
    int64_t x0 = b[0], y0 = b[1], x1 = b[2], y1 = b[3];
    for (int k = 1; k < nb; ++k) {
        x0 = std::min(x0, b[4 * k]);
        y0 = std::min(y0, b[4 * k + 1]);
        x1 = std::max(x1, b[4 * k + 2]);
        y1 = std::max(y1, b[4 * k + 3]);
    }
    const int64_t S = bucket > 0 ? bucket : 64;
    const int64_t gx = (x1 - x0) / S + 1, gy = (y1 - y0) / S + 1;
    if (gx * gy > (int64_t)1 << 26) return -1;
    auto bx = [&](int64_t x) { return std::min<int64_t>(gx - 1, std::max<int64_t>(0, (x - x0) / S)); };
    auto by = [&](int64_t y) { return std::min<int64_t>(gy - 1, std::max<int64_t>(0, (y - y0) / S)); };
    std::vector<int64_t> cnt(gx * gy + 1, 0);
    for (int k = 0; k < nb; ++k)
        for (int64_t j = by(b[4 * k + 1]); j <= by(b[4 * k + 3]); ++j)
            for (int64_t i = bx(b[4 * k]); i <= bx(b[4 * k + 2]); ++i) cnt[j * gx + i + 1]++;
    for (int64_t q = 0; q < gx * gy; ++q) cnt[q + 1] += cnt[q];
    std::vector<int32_t> ids(cnt[gx * gy]);
    std::vector<int64_t> fill(cnt.begin(), cnt.end() - 1);
    for (int k = 0; k < nb; ++k)
        for (int64_t j = by(b[4 * k + 1]); j <= by(b[4 * k + 3]); ++j)
            for (int64_t i = bx(b[4 * k]); i <= bx(b[4 * k + 2]); ++i) ids[fill[j * gx + i]++] = k;
#pragma omp parallel for schedule(dynamic, 256)
    for (int k = 0; k < na; ++k) {
        const int64_t *A = a + 4 * k;
        if (A[2] < x0 || A[0] > x1 || A[3] < y0 || A[1] > y1) continue;
        bool hit = false;
        for (int64_t j = by(A[1]); j <= by(A[3]) && !hit; ++j)
            for (int64_t i = bx(A[0]); i <= bx(A[2]) && !hit; ++i)
                for (int64_t q = cnt[j * gx + i]; q < cnt[j * gx + i + 1]; ++q) {
                    const int64_t *Bq = b + 4 * ids[q];
                    if (A[0] <= Bq[2] && Bq[0] <= A[2] && A[1] <= Bq[3] && Bq[1] <= A[3]) {
                        hit = true;
                        break;
                    }
                }
        out[k] = hit ? 1 : 0;
    }
    return 0;
}
