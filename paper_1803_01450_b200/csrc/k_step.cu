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

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>

#include "common.cuh"

namespace mlamr {

constexpr int NTF = 256;  // threads of the helper kernels (power of two)

// Per-launch constants, divided on the host (IEEE division, so the values
// are the ones the device's `/` would give).
struct StepConst {
    double lam_x, lam_y;  // dt / dx, dt / dy
    double rr[4][4];      // rho_k / rho_m for k < m
    double coef;          // g * (1 - rho_0 / rho_1), the shear bound (physics.py:306)
};

// One tile of the step's work list as the kernel wants it: everything the
// tile header would otherwise read through the chain tile list ->
// box/offset -> ghost base (two dependent L2 round trips in front of every
// CTA's staging; 4.5 % of the kernel's warp-stall samples).  Written by
// k_make_desc in front of each step launch (~2 us).
struct __align__(16) TileDesc {
    int32_t p, tj0, ti0;  // patch, tile origin in the patch interior
    int32_t nxy;          // patch interior nx | ny << 16 (a patch side stays below 65,536 cells)
    int64_t off;          // patch offset in a field plane
    int64_t gb;           // ghost plan base of the patch (0 without a plan)
};

__global__ void k_make_desc(mlamr_level lv, const int32_t *__restrict__ tiles, int n_tiles,
                            const int64_t *__restrict__ gbase, TileDesc *__restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_tiles) return;
    TileDesc d;
    d.p = tiles[3 * i];
    d.tj0 = tiles[3 * i + 1];
    d.ti0 = tiles[3 * i + 2];
    const int32_t *b = lv.box + 4 * d.p;
    d.nxy = (b[2] - b[0] + 1) | ((b[3] - b[1] + 1) << 16);
    d.off = lv.offset[d.p];
    d.gb = gbase != nullptr ? gbase[d.p] : 0;
    out[i] = d;
}

// ceil(2^16 / w) for the step's compact rectangle iteration (step_tile.cuh):
// q = (idx * c_div_magic[w]) >> 16 == idx / w for every idx < 65536 / w.
__constant__ unsigned c_div_magic[64] = {
    0u,
#define MLAMR_MAGIC(w) (65536u + (w) - 1u) / (w)
    MLAMR_MAGIC(1), MLAMR_MAGIC(2), MLAMR_MAGIC(3), MLAMR_MAGIC(4), MLAMR_MAGIC(5), MLAMR_MAGIC(6),
    MLAMR_MAGIC(7), MLAMR_MAGIC(8), MLAMR_MAGIC(9), MLAMR_MAGIC(10), MLAMR_MAGIC(11), MLAMR_MAGIC(12),
    MLAMR_MAGIC(13), MLAMR_MAGIC(14), MLAMR_MAGIC(15), MLAMR_MAGIC(16), MLAMR_MAGIC(17), MLAMR_MAGIC(18),
    MLAMR_MAGIC(19), MLAMR_MAGIC(20), MLAMR_MAGIC(21), MLAMR_MAGIC(22), MLAMR_MAGIC(23), MLAMR_MAGIC(24),
    MLAMR_MAGIC(25), MLAMR_MAGIC(26), MLAMR_MAGIC(27), MLAMR_MAGIC(28), MLAMR_MAGIC(29), MLAMR_MAGIC(30),
    MLAMR_MAGIC(31), MLAMR_MAGIC(32), MLAMR_MAGIC(33), MLAMR_MAGIC(34), MLAMR_MAGIC(35), MLAMR_MAGIC(36),
    MLAMR_MAGIC(37), MLAMR_MAGIC(38), MLAMR_MAGIC(39), MLAMR_MAGIC(40), MLAMR_MAGIC(41), MLAMR_MAGIC(42),
    MLAMR_MAGIC(43), MLAMR_MAGIC(44), MLAMR_MAGIC(45), MLAMR_MAGIC(46), MLAMR_MAGIC(47), MLAMR_MAGIC(48),
    MLAMR_MAGIC(49), MLAMR_MAGIC(50), MLAMR_MAGIC(51), MLAMR_MAGIC(52), MLAMR_MAGIC(53), MLAMR_MAGIC(54),
    MLAMR_MAGIC(55), MLAMR_MAGIC(56), MLAMR_MAGIC(57), MLAMR_MAGIC(58), MLAMR_MAGIC(59), MLAMR_MAGIC(60),
    MLAMR_MAGIC(61), MLAMR_MAGIC(62), MLAMR_MAGIC(63)
#undef MLAMR_MAGIC
};

// K1 in two tile shapes: 16x32 interior tiles (320 threads, 2 CTAs/SM) for
// levels whose patches are wider than 16 cells, 16x16 tiles (192 threads,
// 4 CTAs/SM) for narrow-patch levels (C5's 16x16 patches would leave half
// of a 32-wide tile idle).  mlamr_step_tile() tells the host which shape
// to build a level's tile list with.
#ifndef MLAMR_W_TY
#define MLAMR_W_TY 16
#endif
#ifndef MLAMR_W_NT
#define MLAMR_W_NT 320
#endif
#ifndef MLAMR_W_MINB
#define MLAMR_W_MINB 2
#endif
#define MLAMR_STEP_NS wide
#define MLAMR_STEP_TX 32
#define MLAMR_STEP_TY MLAMR_W_TY
#define MLAMR_STEP_NT MLAMR_W_NT
#define MLAMR_STEP_MINB MLAMR_W_MINB
#include "step_tile.cuh"
#undef MLAMR_STEP_NS
#undef MLAMR_STEP_TX
#undef MLAMR_STEP_TY
#undef MLAMR_STEP_NT
#undef MLAMR_STEP_MINB

#ifndef MLAMR_N_NT
#define MLAMR_N_NT 192
#endif
#ifndef MLAMR_N_MINB
#define MLAMR_N_MINB 4
#endif
#define MLAMR_STEP_NS narrow
#define MLAMR_STEP_TX 16
#define MLAMR_STEP_TY 16
#define MLAMR_STEP_NT MLAMR_N_NT
#define MLAMR_STEP_MINB MLAMR_N_MINB
#include "step_tile.cuh"
#undef MLAMR_STEP_NS
#undef MLAMR_STEP_TX
#undef MLAMR_STEP_TY
#undef MLAMR_STEP_NT
#undef MLAMR_STEP_MINB

// K1 line-walker form for the wide tiles (M <= 2): step_walk.cuh
#include "step_walk.cuh"

// Which K1 form runs the wide tiles.  The phase form is the default: the
// walker is bit-identical but measured slower on C4 (3.74 vs 3.07 ms per
// level-3 launch; profiles/r02/README.md).  MLAMR_STEP=walk or
// mlamr_set_step_form(1) selects the walker.
static int step_form_init() {
    const char *e = getenv("MLAMR_STEP");
    return (e && strcmp(e, "walk") == 0) ? 1 : 0;
}
static std::atomic<int> g_step_form{step_form_init()};
static bool use_walker() { return g_step_form.load(std::memory_order_relaxed) == 1; }

// Descriptor scratch, one per (device, stream), grown on demand: launches
// on one stream are ordered, so reuse is safe -- provided a descriptor
// build and the step launch that reads it enter the stream back to back.
// The reference calls step_patch from a thread pool (driver.py:231-232), so
// callers hold g_desc_mu from desc_scratch() until the step is launched.
static std::mutex g_desc_mu;
static TileDesc *desc_scratch(cudaStream_t st, int n_tiles) {
    struct Buf { TileDesc *p; int cap; };
    static std::map<std::pair<int, cudaStream_t>, Buf> pool;
    int dev = 0;
    cudaGetDevice(&dev);
    Buf &b = pool[{dev, st}];
    if (b.cap < n_tiles) {
        // the old buffer may still be read by a launch in flight on `st`:
        // stream-ordered free
        if (b.p != nullptr) cudaFreeAsync(b.p, st);
        b.p = nullptr;
        b.cap = 0;
        const int cap = n_tiles + n_tiles / 4 + 1024;
        if (cudaMallocAsync(&b.p, sizeof(TileDesc) * (size_t)cap, st) != cudaSuccess) return nullptr;
        b.cap = cap;
    }
    return b.p;
}

// with g_desc_mu held
static const TileDesc *make_desc(const mlamr_level &lv, const int32_t *tiles, int n_tiles, const int64_t *gbase,
                                 cudaStream_t st) {
    TileDesc *desc = desc_scratch(st, n_tiles);
    if (desc != nullptr)
        k_make_desc<<<(n_tiles + 255) / 256, 256, 0, st>>>(lv, tiles, n_tiles, gbase, desc);
    return desc;
}

// CFL guard + deterministic reduction of the step partials.  FIN_BLOCKS
// CTAs each reduce a fixed contiguous chunk of tiles into chunk[b][q]; the
// last CTA to finish (atomic ticket) sums the chunks in order and applies
// the CFL guard, so the result is independent of scheduling.
constexpr int FIN_BLOCKS = 148;

template <int M>
__global__ void __launch_bounds__(NTF) k_step_finalize(mlamr_level lv, const double *__restrict__ src,
                                                      double *__restrict__ dst,
                                                      const int32_t *__restrict__ tiles,
                                                      int n_tiles, double dt,
                                                      long long *speed_bits,
                                                      const double *tile_acc, double *acc,
                                                      int32_t *status, int32_t *bad_patch,
                                                      double *chunk, unsigned int *ticket, int reset_speeds) {
    __shared__ double red[NTF];
    __shared__ int viol;
    __shared__ bool last;
    const int t = threadIdx.x;
    if (*status != 0) return;
    // CFL guard (physics.py:342-347) spread over all blocks: a single block
    // walking every patch was a chain of dependent loads (most of the
    // launch); violations meet in ticket[1], reset by the last block
    const double dmin = lv.dx < lv.dy ? lv.dx : lv.dy;
    {
        bool v = false;
        for (int p = blockIdx.x * NTF + t; p < lv.num_patches; p += gridDim.x * NTF) {
            const long long b = speed_bits[p];
            if (b < 0) continue;
            const double sp = __longlong_as_double(b);
            if ((sp * dt) / dmin > 1.0) {
                v = true;
                atomicMin(bad_patch, p);
            }
        }
        if (__any_sync(0xffffffffu, v) && (t & 31) == 0) atomicOr(ticket + 1, 1u);
    }
    const int K = M + 2;
    const int per = (n_tiles + FIN_BLOCKS - 1) / FIN_BLOCKS;
    const int t0 = blockIdx.x * per, t1 = min(n_tiles, t0 + per);
    for (int q = 0; q < K; ++q) {
        double v = 0.0;
        for (int i = t0 + t; i < t1; i += NTF) v = v + tile_acc[(int64_t)i * K + q];
        const double sm = block_sum<NTF>(v, red);
        if (t == 0) chunk[blockIdx.x * K + q] = sm;
    }
    __threadfence();
    __syncthreads();
    if (t == 0) last = (atomicAdd(ticket, 1u) == gridDim.x - 1);
    __syncthreads();
    if (!last) return;
    __threadfence();
    const double area = lv.dx * lv.dy;
    if (t < K) {
        double sm = 0.0;
        for (int b2 = 0; b2 < (int)gridDim.x; ++b2) sm = sm + ((volatile double *)chunk)[b2 * K + t];
        // clipped mass = -(sum of negative depths) * cell area (physics.py:360-362)
        acc[t] = acc[t] + (t < M ? (-sm) * area : sm);
    }
    if (t == 0) {
        viol = (int)((volatile unsigned int *)ticket)[1];
        ticket[0] = 0u;
        ticket[1] = 0u;
    }
    __syncthreads();
    if (!viol) {
        // every block has read the speeds (ticket): leave them at "all dry"
        // for the next step's atomicMax (replaces a fill before each step)
        if (reset_speeds)
            for (int p = t; p < lv.num_patches; p += NTF) speed_bits[p] = -1LL;
        return;
    }
    // restore every violating patch's interior (the reference raises before
    // touching it, physics.py:342-347)
    const int64_t FS = lv.field_stride;
    for (int p = 0; p < lv.num_patches; ++p) {
        const long long b = speed_bits[p];
        if (b < 0) continue;
        const double sp = __longlong_as_double(b);
        if (!((sp * dt) / dmin > 1.0)) continue;
        const PatchView pv = patch_view(lv, p);
        for (int idx = t; idx < pv.nx * pv.ny; idx += NTF) {
            const int r = idx / pv.nx, c = idx - r * pv.nx;
            const int64_t k = pv.off + (int64_t)(r + MLAMR_G) * pv.NX + (c + MLAMR_G);
            for (int q = 0; q < 3 * M; ++q) dst[q * FS + k] = src[q * FS + k];
        }
    }
    if (t == 0) atomicOr(status, MLAMR_ST_CFL);
}

}  // namespace mlamr

using namespace mlamr;

extern "C" int mlamr_step_tile(int max_patch_nx, int num_layers, int *ty, int *tx) {
    // narrow tiles for narrow patches, and for M >= 3, whose 3M+1 state
    // planes and per-layer scratch make a wide tile's shared memory
    // (~132 KB) allow one CTA per SM (narrow: ~70 KB, 3 CTAs)
#ifdef MLAMR_FORCE_NARROW
    max_patch_nx = 1;
#endif
    if ((max_patch_nx > 0 && max_patch_nx <= narrow::TX) || num_layers >= 3) {
        *ty = narrow::TY;
        *tx = narrow::TX;
    } else {
        *ty = wide::TY;
        *tx = wide::TX;
    }
    return 0;
}

template <int M>
static int launch_step_shape(int tile_tx, const mlamr_level &lv, const double *src, double *dst,
                             const int32_t *tiles, int n_tiles, double dt, int y_first,
                             const mlamr_params &prm, long long *speed_bits, double *tile_acc,
                             const int32_t *status, const int64_t *gbase, const int64_t *gplan,
                             cudaStream_t st) {
    if (n_tiles <= 0) return 0;
    if (tile_tx == narrow::TX) {
        std::lock_guard<std::mutex> lk(g_desc_mu);
        const TileDesc *desc = make_desc(lv, tiles, n_tiles, gbase, st);
        if (desc == nullptr) return -2;
        return narrow::launch_step<M>(lv, src, dst, desc, n_tiles, dt, y_first, prm, speed_bits, tile_acc, status,
                                      gplan, st);
    }
    if constexpr (M <= 2) {
        if (tile_tx == wide::TX && use_walker())
            return walk::launch_step<M>(lv, src, dst, tiles, n_tiles, dt, y_first, prm, speed_bits, tile_acc,
                                        status, gbase, gplan, st);
    }
    if (tile_tx == wide::TX) {
        std::lock_guard<std::mutex> lk(g_desc_mu);
        const TileDesc *desc = make_desc(lv, tiles, n_tiles, gbase, st);
        if (desc == nullptr) return -2;
        return wide::launch_step<M>(lv, src, dst, desc, n_tiles, dt, y_first, prm, speed_bits, tile_acc, status,
                                    gplan, st);
    }
    return -3;
}

extern "C" int mlamr_set_step_form(int form) {
    if (form != 0 && form != 1) return -1;
    return g_step_form.exchange(form);
}

extern "C" int mlamr_step(mlamr_level lv, const double *src_state, double *dst_state,
                          const int32_t *tiles, int n_tiles, int tile_tx, double dt, int y_first,
                          mlamr_params prm, long long *speed_bits, double *tile_acc,
                          const int32_t *status, const int64_t *ghost_base, const int64_t *ghost_plan,
                          void *stream) {
    cudaStream_t st = as_stream(stream);
    const int64_t *gb = ghost_plan ? ghost_base : nullptr;
    switch (prm.num_layers) {
        case 1: return launch_step_shape<1>(tile_tx, lv, src_state, dst_state, tiles, n_tiles, dt, y_first, prm, speed_bits, tile_acc, status, gb, ghost_plan, st);
        case 2: return launch_step_shape<2>(tile_tx, lv, src_state, dst_state, tiles, n_tiles, dt, y_first, prm, speed_bits, tile_acc, status, gb, ghost_plan, st);
        case 3: return launch_step_shape<3>(tile_tx, lv, src_state, dst_state, tiles, n_tiles, dt, y_first, prm, speed_bits, tile_acc, status, gb, ghost_plan, st);
        default: return -1;
    }
}

extern "C" int mlamr_step_finalize(mlamr_level lv, const double *src_state, double *dst_state,
                                   const int32_t *tiles, int n_tiles, double dt,
                                   mlamr_params prm, long long *speed_bits,
                                   const double *tile_acc, double *acc, int32_t *status,
                                   int32_t *bad_patch, int reset_speeds, void *stream) {
    cudaStream_t st = as_stream(stream);
    // scratch for the chunk sums and the completion ticket, one per
    // (device, stream): launches on one stream are ordered, so reuse is safe
    struct Scratch { double *chunk; unsigned int *ticket; };
    static std::mutex mu;
    static std::map<std::pair<int, cudaStream_t>, Scratch> pool;
    int dev = 0;
    cudaGetDevice(&dev);
    Scratch sc;
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = pool.find({dev, st});
        if (it == pool.end()) {
            if (cudaMalloc(&sc.chunk, sizeof(double) * FIN_BLOCKS * (MLAMR_MAX_LAYERS + 2)) != cudaSuccess) return -2;
            if (cudaMalloc(&sc.ticket, 2 * sizeof(unsigned int)) != cudaSuccess) return -2;
            cudaMemsetAsync(sc.ticket, 0, 2 * sizeof(unsigned int), st);
            pool[{dev, st}] = sc;
        } else {
            sc = it->second;
        }
    }
    double *chunk = sc.chunk;
    unsigned int *ticket = sc.ticket;
    switch (prm.num_layers) {
        case 1: k_step_finalize<1><<<FIN_BLOCKS, NTF, 0, st>>>(lv, src_state, dst_state, tiles, n_tiles, dt, speed_bits, tile_acc, acc, status, bad_patch, chunk, ticket, reset_speeds); break;
        case 2: k_step_finalize<2><<<FIN_BLOCKS, NTF, 0, st>>>(lv, src_state, dst_state, tiles, n_tiles, dt, speed_bits, tile_acc, acc, status, bad_patch, chunk, ticket, reset_speeds); break;
        case 3: k_step_finalize<3><<<FIN_BLOCKS, NTF, 0, st>>>(lv, src_state, dst_state, tiles, n_tiles, dt, speed_bits, tile_acc, acc, status, bad_patch, chunk, ticket, reset_speeds); break;
        default: return -1;
    }
    return (int)cudaGetLastError();
}

extern "C" int mlamr_max_speed_tiles(mlamr_level lv, const double *state, const int32_t *tiles,
                                     int n_tiles, int tile_tx, mlamr_params prm, long long *speed_bits,
                                     void *stream) {
    cudaStream_t st = as_stream(stream);
    if (n_tiles <= 0) return 0;
    if (tile_tx != narrow::TX && tile_tx != wide::TX) return -3;
    const bool nar = tile_tx == narrow::TX;
    switch (prm.num_layers) {
        case 1:
            if (nar) narrow::k_max_speed<1><<<n_tiles, NTF, 0, st>>>(lv, state, tiles, prm, speed_bits);
            else wide::k_max_speed<1><<<n_tiles, NTF, 0, st>>>(lv, state, tiles, prm, speed_bits);
            break;
        case 2:
            if (nar) narrow::k_max_speed<2><<<n_tiles, NTF, 0, st>>>(lv, state, tiles, prm, speed_bits);
            else wide::k_max_speed<2><<<n_tiles, NTF, 0, st>>>(lv, state, tiles, prm, speed_bits);
            break;
        case 3:
            if (nar) narrow::k_max_speed<3><<<n_tiles, NTF, 0, st>>>(lv, state, tiles, prm, speed_bits);
            else wide::k_max_speed<3><<<n_tiles, NTF, 0, st>>>(lv, state, tiles, prm, speed_bits);
            break;
        default: return -1;
    }
    return (int)cudaGetLastError();
}
