// Stateful patch-table runtime over the K1-K6 kernels: the handle-based
// C-ABI of SURVEY.md §8(b) (pt_create / pt_set_level / pt_upload_patches /
// pt_download / step / stash / fill / regrid / average_down / mass /
// finite).  A caller that holds the reference's host `Patch` arrays
// (numpy, mesh.py:158-232) drives the GPU through plain host pointers and
// sizes -- no torch, no device pointers.  Device pools use the same SoA
// layout as the Python driver (device.py): per level, 3M state planes and
// one bathymetry plane of `field_stride` elements, patch p a
// (ny+4)x(nx+4) block at offset[p]; two state buffers (the step is out of
// place, and the pre-step buffer is the time-interpolation stash).
//
// Host work per layout (tile list, ghost-plan compaction) happens once, at
// upload / regrid; every per-step call is a few kernel launches on the
// handle's stream plus the scalar read-backs the reference's driver needs.

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <map>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/mlamr_b200.h"

namespace {

constexpr int G = 2;          // ghost width
constexpr int64_t ALIGN = 32; // elements: patch blocks on 256-byte boundaries
constexpr int NTHR = 256;     // blocks-per-patch unit of the helper kernels

template <typename T>
struct DevBuf {
    T *p = nullptr;
    size_t n = 0;
    void ensure(size_t want) {
        if (want <= n && p) return;
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
        if (want == 0) want = 1;
        if (cudaMalloc(&p, want * sizeof(T)) == cudaSuccess) n = want;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
};

struct Level {
    int level = 0, nx = 0, ny = 0, r_x = 1, r_y = 1, r_t = 1;
    double dx = 0.0, dy = 0.0;
    bool configured = false;
    // layout
    int P = 0;
    std::vector<int32_t> boxes;
    std::vector<int64_t> offsets;
    int64_t FS = 0;
    int max_cells = 0, max_interior = 0, max_ghost = 0, max_nx = 0;
    // device
    DevBuf<int32_t> box, own, gown, child, tiles, interp, bcp;
    DevBuf<int64_t> off, gbase, plan;
    DevBuf<double> state[2], bathy, level_bathy, tile_acc, part;
    DevBuf<long long> speed;
    int cur = 0, n_tiles = 0, tile_tx = 32, n_interp = 0, n_bc = 0;
    bool has_level_bathy = false;
    // stash: the pre-step buffer at (t0, dt) for the children's time blend
    bool has_stash = false;
    int stash_buf = 0;
    double stash_t0 = 0.0, stash_dt = 0.0;

    // layout-dependent buffers (the level-wide bathymetry stays)
    void release() {
        box.release(); own.release(); gown.release(); child.release(); tiles.release();
        interp.release(); bcp.release(); off.release(); gbase.release(); plan.release();
        state[0].release(); state[1].release(); bathy.release();
        tile_acc.release(); part.release(); speed.release();
        P = 0;
    }
    void release_all() {
        release();
        level_bathy.release();
        has_level_bathy = false;
    }
};

}  // namespace

struct mlamr_pt {
    mlamr_params prm;
    int32_t bcs[4];
    cudaStream_t st;
    int device = 0;
    std::map<int, Level> levels;
    DevBuf<int32_t> status, bad;
    DevBuf<double> acc;
};

namespace {

int check(cudaError_t e) { return e == cudaSuccess ? 0 : (int)e; }

mlamr_level level_struct(const Level &L, int M, const double *state) {
    mlamr_level lv;
    std::memset(&lv, 0, sizeof(lv));
    lv.num_patches = L.P;
    lv.num_layers = M;
    lv.level_nx = L.nx;
    lv.level_ny = L.ny;
    lv.dx = L.dx;
    lv.dy = L.dy;
    lv.field_stride = L.FS;
    lv.box = L.box.p;
    lv.offset = L.off.p;
    lv.state = const_cast<double *>(state);
    lv.bathy = L.bathy.p;
    lv.own = L.own.p;
    lv.gown = L.gown.n ? L.gown.p : nullptr;
    return lv;
}

int blocks_per_patch(int cells) { return std::max(1, std::min(64, (cells + NTHR - 1) / NTHR)); }

// the level's layout-dependent tables: owner maps, tiles, ghost plan
int build_layout(mlamr_pt *pt, Level &L) {
    const int M = pt->prm.num_layers;
    const int P = L.P;
    L.offsets.assign(P, 0);
    int64_t acc = 0;
    L.max_cells = L.max_interior = L.max_ghost = L.max_nx = 0;
    for (int p = 0; p < P; ++p) {
        const int nx = L.boxes[4 * p + 2] - L.boxes[4 * p] + 1, ny = L.boxes[4 * p + 3] - L.boxes[4 * p + 1] + 1;
        const int64_t size = (int64_t)(nx + 2 * G) * (ny + 2 * G);
        L.offsets[p] = acc;
        acc += (size + ALIGN - 1) / ALIGN * ALIGN;
        L.max_cells = std::max<int>(L.max_cells, (int)size);
        L.max_interior = std::max(L.max_interior, nx * ny);
        L.max_ghost = std::max(L.max_ghost, 4 * (nx + 2 * G) + 4 * ny);
        L.max_nx = std::max(L.max_nx, nx);
    }
    L.FS = std::max<int64_t>(acc, ALIGN);
    L.box.ensure(std::max(1, 4 * P));
    L.off.ensure(std::max(1, P));
    for (int b = 0; b < 2; ++b) L.state[b].ensure((size_t)3 * M * L.FS);
    L.bathy.ensure(L.FS);
    const size_t mapn = (size_t)(L.nx + 2 * G) * (L.ny + 2 * G);
    L.own.ensure(mapn);
    L.gown.ensure(mapn);
    if (!L.box.p || !L.off.p || !L.state[0].p || !L.state[1].p || !L.bathy.p || !L.own.p || !L.gown.p) return -2;
    cudaStream_t st = pt->st;
    int rc = 0;
    rc |= check(cudaMemsetAsync(L.state[0].p, 0, sizeof(double) * 3 * M * L.FS, st));
    rc |= check(cudaMemsetAsync(L.state[1].p, 0, sizeof(double) * 3 * M * L.FS, st));
    rc |= check(cudaMemsetAsync(L.bathy.p, 0, sizeof(double) * L.FS, st));
    if (P) {
        rc |= check(cudaMemcpyAsync(L.box.p, L.boxes.data(), sizeof(int32_t) * 4 * P, cudaMemcpyHostToDevice, st));
        rc |= check(cudaMemcpyAsync(L.off.p, L.offsets.data(), sizeof(int64_t) * P, cudaMemcpyHostToDevice, st));
    }
    rc |= check(cudaMemsetAsync(L.own.p, 0xff, sizeof(int32_t) * mapn, st));
    rc |= check(cudaMemsetAsync(L.gown.p, 0xff, sizeof(int32_t) * mapn, st));
    if (rc) return rc;
    if (P) {
        if ((rc = mlamr_paint_owner(L.own.p, L.nx, L.ny, L.box.p, P, 0, 0, 1, 1, L.max_interior, st))) return rc;
        if ((rc = mlamr_paint_owner(L.gown.p, L.nx, L.ny, L.box.p, P, G, 1, 1, 1, L.max_cells, st))) return rc;
    }
    // step tiles
    int ty = 16, tx = 32;
    mlamr_step_tile(L.max_nx, M, &ty, &tx);
    L.tile_tx = tx;
    std::vector<int32_t> tl;
    for (int p = 0; p < P; ++p) {
        const int nx = L.boxes[4 * p + 2] - L.boxes[4 * p] + 1, ny = L.boxes[4 * p + 3] - L.boxes[4 * p + 1] + 1;
        for (int j0 = 0; j0 < ny; j0 += ty)
            for (int i0 = 0; i0 < nx; i0 += tx) {
                tl.push_back(p);
                tl.push_back(j0);
                tl.push_back(i0);
            }
    }
    L.n_tiles = (int)(tl.size() / 3);
    L.tiles.ensure(std::max<size_t>(3, tl.size()));
    if (!tl.empty())
        rc |= check(cudaMemcpyAsync(L.tiles.p, tl.data(), sizeof(int32_t) * tl.size(), cudaMemcpyHostToDevice, st));
    L.tile_acc.ensure((size_t)std::max(1, L.n_tiles) * (M + 2));
    L.speed.ensure(std::max(1, P));
    // ghost plan, compacted on the host once per layout
    std::vector<int64_t> gb(P + 1, 0);
    for (int p = 0; p < P; ++p) {
        const int nx = L.boxes[4 * p + 2] - L.boxes[4 * p] + 1, ny = L.boxes[4 * p + 3] - L.boxes[4 * p + 1] + 1;
        gb[p + 1] = gb[p] + 4 * (nx + 2 * G) + 4 * ny;
    }
    L.gbase.ensure(std::max(1, P));
    L.plan.ensure(std::max<int64_t>(1, gb[P]));
    if (P) {
        rc |= check(cudaMemcpyAsync(L.gbase.p, gb.data(), sizeof(int64_t) * P, cudaMemcpyHostToDevice, st));
        mlamr_level lv = level_struct(L, M, L.state[L.cur].p);
        if ((rc |= mlamr_ghost_plan(lv, L.gbase.p, L.plan.p, L.max_ghost, st))) return rc;
    }
    std::vector<int64_t> plan(gb[P]);
    if (gb[P]) {
        rc |= check(cudaMemcpyAsync(plan.data(), L.plan.p, sizeof(int64_t) * gb[P], cudaMemcpyDeviceToHost, st));
        rc |= check(cudaStreamSynchronize(st));
    }
    std::vector<int32_t> cells;
    for (int p = 0; p < P; ++p)
        for (int64_t g = gb[p]; g < gb[p + 1]; ++g)
            if (plan[g] == -1) {
                cells.push_back(p);
                cells.push_back((int32_t)(g - gb[p]));
            }
    L.n_interp = (int)(cells.size() / 2);
    L.interp.ensure(std::max<size_t>(2, cells.size()));
    if (!cells.empty())
        rc |= check(cudaMemcpyAsync(L.interp.p, cells.data(), sizeof(int32_t) * cells.size(), cudaMemcpyHostToDevice,
                                    st));
    std::vector<int32_t> bcl;
    for (int p = 0; p < P; ++p)
        if (L.boxes[4 * p] == 0 || L.boxes[4 * p + 1] == 0 || L.boxes[4 * p + 2] == L.nx - 1 ||
            L.boxes[4 * p + 3] == L.ny - 1)
            bcl.push_back(p);
    L.n_bc = (int)bcl.size();
    L.bcp.ensure(std::max<size_t>(1, bcl.size()));
    if (!bcl.empty())
        rc |= check(cudaMemcpyAsync(L.bcp.p, bcl.data(), sizeof(int32_t) * bcl.size(), cudaMemcpyHostToDevice, st));
    rc |= check(cudaStreamSynchronize(st));   // host vectors above go out of scope
    return rc;
}

// coarsened owner map of level+1's boxes in this level's index space
int paint_child(mlamr_pt *pt, Level &par, const Level &fine) {
    const size_t mapn = (size_t)(par.nx + 2 * G) * (par.ny + 2 * G);
    par.child.ensure(mapn);
    int rc = check(cudaMemsetAsync(par.child.p, 0xff, sizeof(int32_t) * mapn, pt->st));
    if (rc || fine.P == 0) return rc;
    int mc = 1;
    for (int p = 0; p < fine.P; ++p) {
        const int nx = fine.boxes[4 * p + 2] - fine.boxes[4 * p] + 1, ny = fine.boxes[4 * p + 3] - fine.boxes[4 * p + 1] + 1;
        mc = std::max(mc, (nx / par.r_x) * (ny / par.r_y));
    }
    return mlamr_paint_owner(par.child.p, par.nx, par.ny, fine.box.p, fine.P, 0, 0, par.r_x, par.r_y, mc, pt->st);
}

Level *get(mlamr_pt *pt, int level) {
    auto it = pt->levels.find(level);
    return (it == pt->levels.end() || !it->second.configured) ? nullptr : &it->second;
}

int read_status(mlamr_pt *pt) {
    int32_t st = 0;
    cudaMemcpyAsync(&st, pt->status.p, sizeof(int32_t), cudaMemcpyDeviceToHost, pt->st);
    cudaStreamSynchronize(pt->st);
    return st;
}

}  // namespace

extern "C" {

mlamr_pt *mlamr_pt_create(mlamr_params prm, const int32_t *bcs, void *stream) {
    if (prm.num_layers < 1 || prm.num_layers > 3) return nullptr;
    mlamr_pt *pt = new mlamr_pt();
    pt->prm = prm;
    for (int i = 0; i < 4; ++i) pt->bcs[i] = bcs ? bcs[i] : MLAMR_BC_WALL;
    pt->st = reinterpret_cast<cudaStream_t>(stream);
    cudaGetDevice(&pt->device);
    pt->status.ensure(1);
    pt->bad.ensure(1);
    pt->acc.ensure(prm.num_layers + 2);
    cudaMemsetAsync(pt->status.p, 0, sizeof(int32_t), pt->st);
    cudaMemsetAsync(pt->acc.p, 0, sizeof(double) * (prm.num_layers + 2), pt->st);
    return pt;
}

void mlamr_pt_destroy(mlamr_pt *pt) {
    if (!pt) return;
    cudaStreamSynchronize(pt->st);
    for (auto &kv : pt->levels) kv.second.release_all();
    pt->status.release();
    pt->bad.release();
    pt->acc.release();
    delete pt;
}

int mlamr_pt_set_level(mlamr_pt *pt, int level, int nx, int ny, double dx, double dy, int r_x, int r_y, int r_t) {
    if (!pt || level < 1 || nx <= 0 || ny <= 0) return -1;
    Level &L = pt->levels[level];
    L.level = level;
    L.nx = nx;
    L.ny = ny;
    L.dx = dx;
    L.dy = dy;
    L.r_x = r_x;
    L.r_y = r_y;
    L.r_t = r_t;
    L.configured = true;
    return 0;
}

int mlamr_pt_set_level_bathymetry(mlamr_pt *pt, int level, const double *h_bathy) {
    Level *L = get(pt, level);
    if (!L || !h_bathy) return -1;
    L->level_bathy.ensure((size_t)L->nx * L->ny);
    L->has_level_bathy = true;
    return check(cudaMemcpy(L->level_bathy.p, h_bathy, sizeof(double) * L->nx * L->ny, cudaMemcpyHostToDevice));
}

int mlamr_pt_upload_patches(mlamr_pt *pt, int level, int n, const int32_t *h_boxes, const double *const *h,
                            const double *const *hu, const double *const *hv, const double *const *h_bathy) {
    Level *L = get(pt, level);
    if (!L || n < 0) return -1;
    const int M = pt->prm.num_layers;
    cudaStreamSynchronize(pt->st);
    L->release();
    L->P = n;
    L->boxes.assign(h_boxes, h_boxes + 4 * n);
    L->cur = 0;
    L->has_stash = false;
    int rc = build_layout(pt, *L);
    if (rc) return rc;
    // pack the patches into the pool layout in pinned memory, one copy up
    double *stage = nullptr;
    if (cudaMallocHost(&stage, sizeof(double) * (3 * M + 1) * L->FS) != cudaSuccess) return -2;
    std::memset(stage, 0, sizeof(double) * (3 * M + 1) * L->FS);
    for (int p = 0; p < n; ++p) {
        const int nx = L->boxes[4 * p + 2] - L->boxes[4 * p] + 1, ny = L->boxes[4 * p + 3] - L->boxes[4 * p + 1] + 1;
        const size_t cells = (size_t)(nx + 2 * G) * (ny + 2 * G);
        for (int m = 0; m < M; ++m) {
            std::memcpy(stage + (size_t)m * L->FS + L->offsets[p], h[p] + m * cells, sizeof(double) * cells);
            std::memcpy(stage + (size_t)(M + m) * L->FS + L->offsets[p], hu[p] + m * cells, sizeof(double) * cells);
            std::memcpy(stage + (size_t)(2 * M + m) * L->FS + L->offsets[p], hv[p] + m * cells, sizeof(double) * cells);
        }
        if (h_bathy) std::memcpy(stage + (size_t)3 * M * L->FS + L->offsets[p], h_bathy[p], sizeof(double) * cells);
    }
    rc |= check(cudaMemcpyAsync(L->state[0].p, stage, sizeof(double) * 3 * M * L->FS, cudaMemcpyHostToDevice, pt->st));
    if (h_bathy)
        rc |= check(cudaMemcpyAsync(L->bathy.p, stage + (size_t)3 * M * L->FS, sizeof(double) * L->FS,
                                    cudaMemcpyHostToDevice, pt->st));
    rc |= check(cudaStreamSynchronize(pt->st));
    cudaFreeHost(stage);
    if (!h_bathy && L->has_level_bathy) {
        mlamr_level lv = level_struct(*L, M, L->state[0].p);
        rc |= mlamr_fill_bathymetry(lv, L->level_bathy.p, pt->bcs, pt->st);
    }
    // child maps: this level as a parent, and the level below for this one
    Level *fine = get(pt, level + 1);
    if (fine && fine->P) rc |= paint_child(pt, *L, *fine);
    Level *par = get(pt, level - 1);
    if (par && par->P) rc |= paint_child(pt, *par, *L);
    return rc;
}

int mlamr_pt_num_patches(mlamr_pt *pt, int level) {
    Level *L = get(pt, level);
    return L ? L->P : -1;
}

int mlamr_pt_download(mlamr_pt *pt, int level, double *const *h, double *const *hu, double *const *hv) {
    Level *L = get(pt, level);
    if (!L) return -1;
    const int M = pt->prm.num_layers;
    double *stage = nullptr;
    if (cudaMallocHost(&stage, sizeof(double) * 3 * M * L->FS) != cudaSuccess) return -2;
    int rc = check(cudaMemcpyAsync(stage, L->state[L->cur].p, sizeof(double) * 3 * M * L->FS,
                                   cudaMemcpyDeviceToHost, pt->st));
    rc |= check(cudaStreamSynchronize(pt->st));
    for (int p = 0; p < L->P && !rc; ++p) {
        const int nx = L->boxes[4 * p + 2] - L->boxes[4 * p] + 1, ny = L->boxes[4 * p + 3] - L->boxes[4 * p + 1] + 1;
        const size_t cells = (size_t)(nx + 2 * G) * (ny + 2 * G);
        for (int m = 0; m < M; ++m) {
            if (h) std::memcpy(h[p] + m * cells, stage + (size_t)m * L->FS + L->offsets[p], sizeof(double) * cells);
            if (hu) std::memcpy(hu[p] + m * cells, stage + (size_t)(M + m) * L->FS + L->offsets[p], sizeof(double) * cells);
            if (hv) std::memcpy(hv[p] + m * cells, stage + (size_t)(2 * M + m) * L->FS + L->offsets[p], sizeof(double) * cells);
        }
    }
    cudaFreeHost(stage);
    return rc;
}

int mlamr_pt_max_speed(mlamr_pt *pt, int level, double *out_speed) {
    Level *L = get(pt, level);
    if (!L) return -1;
    if (L->P == 0) return 0;
    const int M = pt->prm.num_layers;
    int rc = check(cudaMemsetAsync(L->speed.p, 0xff, sizeof(long long) * L->P, pt->st));
    mlamr_level lv = level_struct(*L, M, L->state[L->cur].p);
    rc |= mlamr_max_speed_tiles(lv, L->state[L->cur].p, L->tiles.p, L->n_tiles, L->tile_tx, pt->prm, L->speed.p, pt->st);
    std::vector<long long> bits(L->P);
    rc |= check(cudaMemcpyAsync(bits.data(), L->speed.p, sizeof(long long) * L->P, cudaMemcpyDeviceToHost, pt->st));
    rc |= check(cudaStreamSynchronize(pt->st));
    for (int p = 0; p < L->P; ++p) {
        double v = 0.0;
        if (bits[p] >= 0) std::memcpy(&v, &bits[p], sizeof(double));
        out_speed[p] = v;
    }
    return rc;
}

int mlamr_pt_stash(mlamr_pt *pt, int level, double t0, double dt) {
    Level *L = get(pt, level);
    if (!L) return -1;
    L->has_stash = true;
    L->stash_buf = L->cur;   // the step leaves its source buffer untouched
    L->stash_t0 = t0;
    L->stash_dt = dt;
    return 0;
}

int mlamr_pt_clear_stash(mlamr_pt *pt, int level) {
    Level *L = get(pt, level);
    if (!L) return -1;
    L->has_stash = false;
    return 0;
}

int mlamr_pt_fill_ghosts(mlamr_pt *pt, int level, double t) {
    Level *L = get(pt, level);
    if (!L) return -1;
    if (L->P == 0) return 0;
    const int M = pt->prm.num_layers;
    mlamr_level lv = level_struct(*L, M, L->state[L->cur].p);
    Level *par = get(pt, level - 1);
    mlamr_level plv;
    const mlamr_level *pp = nullptr;
    const double *old = nullptr;
    double theta = 0.0;
    int rx = 1, ry = 1;
    if (par && par->P) {
        plv = level_struct(*par, M, par->state[par->cur].p);
        pp = &plv;
        rx = par->r_x;
        ry = par->r_y;
        if (par->has_stash) {
            old = par->state[par->stash_buf].p;
            theta = par->stash_dt > 0.0 ? std::min(1.0, std::max(0.0, (t - par->stash_t0) / par->stash_dt)) : 1.0;
        }
    }
    return mlamr_fill_ghosts_planned(lv, pp, old, theta, rx, ry, pt->bcs, pt->prm, pt->status.p, L->gbase.p,
                                     L->plan.p, nullptr, 0, L->max_ghost, L->interp.p, pp ? L->n_interp : 0, nullptr,
                                     L->bcp.p, L->n_bc, pt->st);
}

int mlamr_pt_step_level(mlamr_pt *pt, int level, double dt, int y_first, double *out_counters, int *bad_patch) {
    Level *L = get(pt, level);
    if (!L) return -1;
    if (L->P == 0) return 0;
    const int M = pt->prm.num_layers;
    double *src = L->state[L->cur].p, *dst = L->state[1 - L->cur].p;
    int rc = check(cudaMemsetAsync(L->speed.p, 0xff, sizeof(long long) * L->P, pt->st));
    const int32_t big = 0x7fffffff;
    rc |= check(cudaMemcpyAsync(pt->bad.p, &big, sizeof(int32_t), cudaMemcpyHostToDevice, pt->st));
    rc |= check(cudaMemsetAsync(pt->acc.p, 0, sizeof(double) * (M + 2), pt->st));
    mlamr_level lv = level_struct(*L, M, src);
    rc |= mlamr_step(lv, src, dst, L->tiles.p, L->n_tiles, L->tile_tx, dt, y_first, pt->prm, L->speed.p,
                     L->tile_acc.p, pt->status.p, nullptr, nullptr, pt->st);
    rc |= mlamr_step_finalize(lv, src, dst, L->tiles.p, L->n_tiles, dt, pt->prm, L->speed.p, L->tile_acc.p,
                              pt->acc.p, pt->status.p, pt->bad.p, 0, pt->st);
    if (rc) return rc;
    double acc[MLAMR_MAX_LAYERS + 2];
    int32_t bad = 0;
    cudaMemcpyAsync(acc, pt->acc.p, sizeof(double) * (M + 2), cudaMemcpyDeviceToHost, pt->st);
    cudaMemcpyAsync(&bad, pt->bad.p, sizeof(int32_t), cudaMemcpyDeviceToHost, pt->st);
    const int st = read_status(pt);
    if (out_counters) std::memcpy(out_counters, acc, sizeof(double) * (M + 2));
    if (bad_patch) *bad_patch = (bad == big) ? -1 : bad;
    if (st & MLAMR_ST_CFL) {   // the reference raises before touching the patch: nothing was written
        const int32_t zero = 0;
        cudaMemcpyAsync(pt->status.p, &zero, sizeof(int32_t), cudaMemcpyHostToDevice, pt->st);
        cudaStreamSynchronize(pt->st);
        return MLAMR_ST_CFL;
    }
    if (st) return st;
    L->cur = 1 - L->cur;
    return 0;
}

int mlamr_pt_average_down(mlamr_pt *pt, int fine_level) {
    Level *F = get(pt, fine_level), *C = get(pt, fine_level - 1);
    if (!F || !C) return -1;
    if (F->P == 0 || C->P == 0) return 0;
    const int M = pt->prm.num_layers;
    std::vector<int64_t> base(F->P + 1, 0);
    for (int p = 0; p < F->P; ++p) {
        const int nx = F->boxes[4 * p + 2] - F->boxes[4 * p] + 1, ny = F->boxes[4 * p + 3] - F->boxes[4 * p + 1] + 1;
        base[p + 1] = base[p] + (int64_t)(nx / C->r_x) * (ny / C->r_y);
    }
    DevBuf<int64_t> bd;
    bd.ensure(F->P + 1);
    int rc = check(cudaMemcpyAsync(bd.p, base.data(), sizeof(int64_t) * (F->P + 1), cudaMemcpyHostToDevice, pt->st));
    mlamr_level fl = level_struct(*F, M, F->state[F->cur].p), cl = level_struct(*C, M, C->state[C->cur].p);
    rc |= mlamr_average_down_flat(fl, cl, C->r_x, C->r_y, pt->prm, bd.p, base[F->P], pt->status.p, pt->st);
    rc |= check(cudaStreamSynchronize(pt->st));
    bd.release();
    return rc;
}

int mlamr_pt_regrid(mlamr_pt *pt, int level, int n, const int32_t *h_new_boxes, double *out_refine,
                    double *out_derefine) {
    Level *par = get(pt, level - 1);
    Level *L = get(pt, level);
    if (!par || !L || !L->has_level_bathy) return -1;
    const int M = pt->prm.num_layers;
    // the old pool moves aside; the new one takes its place
    Level old = std::move(*L);
    Level &N = pt->levels[level];
    N = Level();
    N.level = old.level; N.nx = old.nx; N.ny = old.ny; N.dx = old.dx; N.dy = old.dy;
    N.r_x = old.r_x; N.r_y = old.r_y; N.r_t = old.r_t; N.configured = true;
    N.level_bathy = old.level_bathy;   // shared ownership: moved below
    old.level_bathy = DevBuf<double>();
    N.has_level_bathy = true;
    N.P = n;
    N.boxes.assign(h_new_boxes, h_new_boxes + 4 * n);
    int rc = build_layout(pt, N);
    if (rc) return rc;
    mlamr_level nl = level_struct(N, M, N.state[0].p), pl = level_struct(*par, M, par->state[par->cur].p);
    rc |= mlamr_fill_bathymetry(nl, N.level_bathy.p, pt->bcs, pt->st);
    mlamr_level ol = level_struct(old, M, old.P ? old.state[old.cur].p : nullptr);
    if (old.P == 0) {
        std::memset(&ol, 0, sizeof(ol));
        ol.num_layers = M;
        ol.level_nx = N.nx;
        ol.level_ny = N.ny;
        ol.dx = N.dx;
        ol.dy = N.dy;
    }
    double ref[MLAMR_MAX_LAYERS] = {0}, der[MLAMR_MAX_LAYERS] = {0};
    if (n) {
        const int bpp = blocks_per_patch(N.max_interior / (par->r_x * par->r_y));
        N.part.ensure((size_t)n * bpp * M);
        rc |= check(cudaMemsetAsync(N.part.p, 0, sizeof(double) * n * bpp * M, pt->st));
        rc |= mlamr_regrid_fill(nl, ol, pl, par->r_x, par->r_y, pt->prm, N.part.p, bpp, pt->status.p, nullptr, 0,
                                pt->st);
        std::vector<double> part((size_t)n * bpp * M);
        rc |= check(cudaMemcpyAsync(part.data(), N.part.p, sizeof(double) * part.size(), cudaMemcpyDeviceToHost, pt->st));
        rc |= check(cudaStreamSynchronize(pt->st));
        for (size_t i = 0; i < part.size(); ++i) ref[i % M] += part[i];
    }
    rc |= paint_child(pt, *par, N);
    if (old.P) {
        const int bpp = blocks_per_patch(old.max_interior / (par->r_x * par->r_y));
        DevBuf<double> dp;
        dp.ensure((size_t)old.P * bpp * M);
        rc |= check(cudaMemsetAsync(dp.p, 0, sizeof(double) * old.P * bpp * M, pt->st));
        rc |= mlamr_derefine_delta(ol, pl, par->child.p, par->r_x, par->r_y, pt->prm, dp.p, bpp, nullptr, 0, pt->st);
        std::vector<double> part((size_t)old.P * bpp * M);
        rc |= check(cudaMemcpyAsync(part.data(), dp.p, sizeof(double) * part.size(), cudaMemcpyDeviceToHost, pt->st));
        rc |= check(cudaStreamSynchronize(pt->st));
        for (size_t i = 0; i < part.size(); ++i) der[i % M] += part[i];
        dp.release();
    }
    Level *fine = get(pt, level + 1);
    if (fine && fine->P) rc |= paint_child(pt, N, *fine);
    cudaStreamSynchronize(pt->st);
    old.release();
    if (out_refine) std::memcpy(out_refine, ref, sizeof(double) * M);
    if (out_derefine) std::memcpy(out_derefine, der, sizeof(double) * M);
    const int st = read_status(pt);
    return rc ? rc : st;
}

int mlamr_pt_composite_mass(mlamr_pt *pt, double *out) {
    if (!pt) return -1;
    const int M = pt->prm.num_layers;
    std::vector<double> tot(M, 0.0);
    int rc = 0;
    for (auto &kv : pt->levels) {
        Level &L = kv.second;
        if (!L.configured || L.P == 0) continue;
        const int bpp = blocks_per_patch(L.max_cells);
        L.part.ensure((size_t)L.P * bpp * M);
        rc |= check(cudaMemsetAsync(L.part.p, 0, sizeof(double) * L.P * bpp * M, pt->st));
        Level *fine = get(pt, kv.first + 1);
        const int32_t *child = (fine && fine->P && L.child.n) ? L.child.p : nullptr;
        mlamr_level lv = level_struct(L, M, L.state[L.cur].p);
        rc |= mlamr_level_reduce(lv, L.state[L.cur].p, L.state[L.cur].p, child, L.part.p, bpp, pt->status.p, nullptr,
                                 0, pt->st);
        std::vector<double> part((size_t)L.P * bpp * M);
        rc |= check(cudaMemcpyAsync(part.data(), L.part.p, sizeof(double) * part.size(), cudaMemcpyDeviceToHost, pt->st));
        rc |= check(cudaStreamSynchronize(pt->st));
        std::vector<double> lev(M, 0.0);
        for (size_t i = 0; i < part.size(); ++i) lev[i % M] += part[i];
        for (int m = 0; m < M; ++m) tot[m] += lev[m] * (L.dx * L.dy);
    }
    std::memcpy(out, tot.data(), sizeof(double) * M);
    return rc;
}

int mlamr_pt_check_finite(mlamr_pt *pt) {
    if (!pt) return -1;
    double tmp[MLAMR_MAX_LAYERS];
    int rc = mlamr_pt_composite_mass(pt, tmp);
    if (rc) return rc;
    const int st = read_status(pt);
    return st & MLAMR_ST_NONFINITE;
}

int mlamr_pt_status(mlamr_pt *pt) { return pt ? read_status(pt) : -1; }

}  // extern "C"
