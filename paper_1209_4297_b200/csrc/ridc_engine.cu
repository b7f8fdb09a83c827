// ridc_engine.cu -- kernels + host runtime behind include/ridc_b200.h (sm_100a).
//
// Single-device engine: every tick of the lagged pipeline is ONE kernel launch
// covering all active levels (levels are independent within a tick:
// level j at tick k computes step k - j(j+1)/2, reading only data published
// in earlier ticks, engine.py:363-371), and the whole run (all restart
// intervals, all ticks) is captured once into a CUDA graph at create time
// (the analogue of _prepare's pre-factorisation, engine.py:465-473).
//
// Level rings: level j < top keeps its last 2j+3 states in HBM (the greedy
// schedule's live window for the reader j+1, which lags j+1 ticks); the top
// level keeps 2 (or the whole trajectory when it is recorded).
#include <cuda.h>   // driver-API types only; entry points come from cudaGetDriverEntryPoint
#include <cuda_runtime.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <map>
#include <thread>
#include <climits>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/ridc_b200.h"
#include "ridc_device.cuh"
#include "ridc_tma.cuh"

using namespace ridc;

namespace {

thread_local std::string g_last_error;

struct EngineParams {
    DevProblem pb;
    DevSolve sv;
    long long V;    // points per state
    long long Vs;   // ring slot stride (even, >= V + 4: keeps every slot 16-byte aligned + guards)
    double dt;
    int levels;
    double* ring[kMaxLevels];
    long long cap[kMaxLevels];
    long long off[kMaxLevels];
    const double* weights;
    int steady_off[kMaxLevels];
    int startup_off[kMaxLevels];
    unsigned long long* err;
    double* mirror;            // pipeline: consumer's inbox ring (peer memory), or null
    long long mirror_cap, mirror_off;
};

struct TickParams {
    int nact;
    int level[kMaxLevels];
    long long target[kMaxLevels];
};

__device__ __forceinline__ double* ring_slot(const EngineParams& ep, int lev, long long s,
                                             long long off = -1)
{
    return ep.ring[lev] + (((off < 0 ? ep.off[lev] : off) + s) % ep.cap[lev]) * ep.Vs;
}

// Window assembly for (level j, target t): _window_span / _orient /
// _WeightTables.for_step (engine.py:124-157) with the lag terms of
// _correct_core (engine.py:179-181) folded into the node coefficients.
__device__ void build_item(const EngineParams& ep, int j, long long t, StepItem& it, long long off = -1)
{
    it.level = j;
    it.target = t;
    it.vec[0] = ring_slot(ep, j, t - 1, off);
    it.ca[0] = 1.0;
    it.cs[0] = 0.0;
    it.cn[0] = ep.dt;
    int nn = 1;
    if (j > 0) {
        const bool steady = t >= j;
        const double* w = steady ? ep.weights + ep.steady_off[j]
                                 : ep.weights + ep.startup_off[j] + (t - 1) * (j + 1);
        const int i_new = steady ? 0 : (int)t;
        const int i_old = steady ? 1 : (int)t - 1;
        for (int a = 0; a <= j; ++a) {
            const long long s = steady ? t - a : a;
            it.vec[nn] = ring_slot(ep, j - 1, s, off);
            it.ca[nn] = 0.0;
            it.cs[nn] = w[a] - (a == i_new ? ep.dt : 0.0);
            it.cn[nn] = w[a] - (a == i_old ? ep.dt : 0.0);
            ++nn;
        }
    }
    it.nnodes = nn;
    it.out = ring_slot(ep, j, t, off);
    it.out2 = ep.mirror ? ep.mirror + ((ep.mirror_off + t) % ep.mirror_cap) * ep.Vs : nullptr;
}

// The production tick kernel: persistent CTAs of NT compute threads; thread
// 0 doubles as the TMA producer (ridc_tma.cuh).  Items of the tick are dealt
// round-robin: item i -> level slot i % nact, tile i / nact.
template <int KIND, int NT, int KMAX, int ROWS, int NSTAGE>
__global__ void __launch_bounds__(NT, 1) k_tick_tma(EngineParams ep, TickParams tp, int ipl)
{
    using L = TmaSmem<NT, KMAX, ROWS, NSTAGE>;
    extern __shared__ __align__(128) double sm[];
    double* stage = sm;
    double* sbuf = sm + L::OFF_SBUF;
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + L::OFF_BAR);
    uint64_t* empty = full + NSTAGE;
    __shared__ StepItem items[kMaxLevels];   // one descriptor per active level (shared by all its tiles)
    __shared__ Aff swarp[2 * (NT / 32) + 1];
    const int total = tp.nact * ipl;
    if (threadIdx.x < tp.nact) build_item(ep, tp.level[threadIdx.x], tp.target[threadIdx.x], items[threadIdx.x]);
    if (threadIdx.x == 0) {
        for (int i = 0; i < NSTAGE; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], NT / 32);
        }
        mbar_fence_init();
    }
    __syncthreads();
    // producer cursor (thread 0): next (item, node) to load and its load number
    LoadCursor pc{(int)blockIdx.x, 0, 0};
    auto issue_next = [&](int s) {
        const int slot = pc.i % tp.nact, tile = pc.i / tp.nact;
        const Geo g = make_geo<KIND, NT, KMAX>(ep.pb, ep.sv, tile);
        issue_node<ROWS, L::SROW>(ep.pb, ep.sv, items[slot].vec[pc.a], g, stage + (size_t)s * L::STAGE,
                                  &full[s]);
        if (++pc.a == items[slot].nnodes) { pc.a = 0; pc.i += gridDim.x; }
        ++pc.n;
    };
    if (threadIdx.x == 0)
        for (int k = 0; k < NSTAGE && pc.i < total; ++k) issue_next(k);
    // after load n was released from stage s: wait for every warp, then load n + NSTAGE into s
    auto refill = [&](long long n, int s) {
        if (pc.i >= total) return;
        mbar_wait(&empty[s], (uint32_t)((n / NSTAGE) & 1));
        issue_next(s);
    };
    long long n = 0;
    int ino = 0;
    for (int i = blockIdx.x; i < total; i += gridDim.x, ++ino) {
        const int slot = i % tp.nact, tile = i / tp.nact;
        Geo geo = make_geo<KIND, NT, KMAX>(ep.pb, ep.sv, tile);
        geo.item_no = ino;
        auto ensure = [](long long) {};
        if (geo.fast)
            consume_item<KIND, NT, KMAX, ROWS, NSTAGE, true>(ep.pb, ep.sv, items[slot], geo, stage, full,
                                                            empty, n, refill, ensure, sbuf, swarp, ep.err);
        else
            consume_item<KIND, NT, KMAX, ROWS, NSTAGE, false>(ep.pb, ep.sv, items[slot], geo, stage,
                                                             full, empty, n, refill, ensure, sbuf, swarp,
                                                             ep.err);
        csync<NT>();   // sbuf reuse by the next item
    }
}

// ---------------------------------------------------------------- persistent run kernel
//
// One launch marches every interval and tick.  CTA b owns tiles b, b+G, ...
// of every level.  Cross-CTA ordering uses one completion flag per (level,
// tile): the last global step written (global step of (interval r, step t)
// = r*(per+1) + t; step 0 of an interval is its seed).  Before level j
// computes global step G of a tile, thread 0 acquires (engine.py:363-371):
//   (a) own level, neighbour tiles  >= G-1        (halo of the previous state)
//   (b) level j-1, neighbour tiles  >= G(hi)      (window, LevelBuffer.watermark)
//   (c) level j+1, neighbour tiles  >= G - C_j + j + 1   (ring slot free, .released)
// Every dependency is on an earlier tick and every CTA walks its items in
// tick order, so co-resident CTAs cannot deadlock; a %globaltimer watchdog
// still turns a stall into an error instead of a hang.
struct PersistParams {
    int ipl;                   // tiles per level
    int rx;                    // neighbour radius in segments
    int levels, restarts;
    long long per;
    long long* flags;          // [levels][ipl], init -1
    const double* y0;
    int* abort;
    unsigned long long timeout_ns;
};

__device__ __forceinline__ long long ld_acquire(const long long* p)
{
    long long v;
    asm volatile("ld.acquire.gpu.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release(long long* p, long long v)
{
    asm volatile("st.release.gpu.global.s64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned long long gtimer()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// pointer of node a of (level j, step t) -- the same order build_item uses
__device__ __forceinline__ const double* node_ptr(const EngineParams& ep, int j, long long t, int a,
                                                  long long off)
{
    if (a == 0) return ring_slot(ep, j, t - 1, off);
    const long long s = t >= j ? t - (a - 1) : (a - 1);
    return ring_slot(ep, j - 1, s, off);
}

// Are the dependencies of (level j, global step G, tile) satisfied?
template <int KIND>
__device__ bool deps_ready(const EngineParams& ep, const PersistParams& pp, int j, long long t,
                           long long G, long long Ghi, int tile)
{
    const int nseg = ep.sv.nseg, ny = ep.pb.ny;
    constexpr bool periodic = KIND != BURGERS_1D;
    const int row = tile / nseg, seg = tile - row * nseg;
    const int r0 = ny > 1 ? -1 : 0, r1 = ny > 1 ? 1 : 0;
    const int rx = nseg > 1 ? pp.rx : 0;
    const long long capj = ep.cap[j];
    bool ok = true;
    for (int dr = r0; dr <= r1; ++dr) {
        const int rr = (row + dr + ny) % ny;
        for (int ds = -rx; ds <= rx; ++ds) {
            int sg = seg + ds;
            if (periodic) sg = (sg % nseg + nseg) % nseg;
            else if (sg < 0 || sg >= nseg) continue;
            const int tl = rr * nseg + sg;
            ok &= ld_acquire(pp.flags + (size_t)j * pp.ipl + tl) >= G - 1;
            if (j > 0 && t >= 1) ok &= ld_acquire(pp.flags + (size_t)(j - 1) * pp.ipl + tl) >= Ghi;
            if (j < pp.levels - 1)
                ok &= ld_acquire(pp.flags + (size_t)(j + 1) * pp.ipl + tl) >= G - capj + j + 1;
        }
    }
    return ok;
}

template <int KIND>
__device__ bool wait_deps(const EngineParams& ep, const PersistParams& pp, int j, long long t, long long G,
                          long long Ghi, int tile)
{
    unsigned long long t0 = 0;
    for (;;) {
        if (deps_ready<KIND>(ep, pp, j, t, G, Ghi, tile)) {
            asm volatile("fence.proxy.async.global;" ::: "memory");   // generic writes -> TMA reads
            return true;
        }
        if (*(volatile int*)pp.abort) return false;
        const unsigned long long now = gtimer();
        if (t0 == 0) t0 = now;
        else if (now - t0 > pp.timeout_ns) {
            atomicExch(pp.abort, 1);
            return false;
        }
    }
}


struct PCursor {
    int r;            // interval
    long long k;      // tick
    int j;            // level
    int m;            // owned-tile ordinal
    int a;            // node
    long long n;      // load number
    bool done;
};

template <int KIND, int NT, int KMAX, int ROWS, int NSTAGE>
__global__ void __launch_bounds__(NT, 1) k_persist(EngineParams ep0, PersistParams pp)
{
    using L = TmaSmem<NT, KMAX, ROWS, NSTAGE>;
    extern __shared__ __align__(128) double sm[];
    double* stage = sm;
    double* sbuf = sm + L::OFF_SBUF;
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + L::OFF_BAR);
    uint64_t* empty = full + NSTAGE;
    __shared__ StepItem items[2][kMaxLevels];
    __shared__ Aff swarp[2 * (NT / 32) + 1];
    __shared__ volatile int s_abort;
    const int tid = threadIdx.x;
    const int G = gridDim.x;
    const int my_tiles = pp.ipl > (int)blockIdx.x ? (pp.ipl - 1 - (int)blockIdx.x) / G + 1 : 0;
    const int top = pp.levels - 1;
    const long long ticks = pp.per + (long long)top * (top + 1) / 2;
    if (tid == 0) {
        for (int i = 0; i < NSTAGE; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], NT / 32);
        }
        mbar_fence_init();
        s_abort = 0;
    }
    __syncthreads();
    if (my_tiles == 0) return;
    const EngineParams& ep = ep0;

    // ---- producer cursor (thread 0) over compute items: (r, k, j active, m, a)
    auto delay = [](int j) { return (long long)j * (j + 1) / 2; };
    auto active = [&](long long k, int j) { const long long t = k - delay(j); return t >= 1 && t <= pp.per; };
    PCursor pc{0, 1, 0, 0, 0, 0, false};
    auto first_level = [&](long long k, int from) {
        for (int j = from; j <= top; ++j)
            if (active(k, j)) return j;
        return -1;
    };
    pc.j = first_level(1, 0);
    auto advance_item = [&]() {
        pc.a = 0;
        if (++pc.m < my_tiles) return;
        pc.m = 0;
        int nj = first_level(pc.k, pc.j + 1);
        while (nj < 0) {
            if (++pc.k > ticks) {
                pc.k = 1;
                if (++pc.r >= pp.restarts) { pc.done = true; return; }
            }
            nj = first_level(pc.k, 0);
        }
        pc.j = nj;
    };
    const EngineParams& epp = ep0;
    bool pc_ready = false;    // dependencies of the cursor's current item acquired
    auto try_issue = [&](int s, bool blocking) -> bool {
        if (pc.done) return false;
        const long long poff = (long long)pc.r * (pp.per + 1);
        const long long t = pc.k - delay(pc.j);
        const int tile = (int)blockIdx.x + pc.m * G;
        if (pc.a == 0 && !pc_ready) {
            const long long Gs = (long long)pc.r * (pp.per + 1) + t;
            const long long hi = pc.j > 0 ? (t < pc.j ? pc.j : t) : 0;
            const long long Ghi = (long long)pc.r * (pp.per + 1) + hi;
            if (blocking) {
                if (!wait_deps<KIND>(epp, pp, pc.j, t, Gs, Ghi, tile)) return false;
            } else if (!deps_ready<KIND>(epp, pp, pc.j, t, Gs, Ghi, tile)) {
                return false;
            } else {
                asm volatile("fence.proxy.async.global;" ::: "memory");
            }
            pc_ready = true;
        }
        const Geo g = make_geo<KIND, NT, KMAX>(epp.pb, epp.sv, tile);
        issue_node<ROWS, L::SROW>(epp.pb, epp.sv, node_ptr(epp, pc.j, t, pc.a, poff), g,
                                  stage + (size_t)s * L::STAGE, &full[s]);
        const int nn = pc.j > 0 ? pc.j + 2 : 1;
        ++pc.n;
        if (++pc.a == nn) { pc_ready = false; advance_item(); }
        return true;
    };
    // released load n from stage s: refill with load n + NSTAGE if ready (never blocks on peers)
    auto refill = [&](long long n, int s) {
        if (pc.done || pc.n != n + NSTAGE) return;
        mbar_wait(&empty[s], (uint32_t)((n / NSTAGE) & 1));
        try_issue(s, false);
    };
    // before consuming load n: make sure loads up to n are issued (may block on peers)
    auto ensure = [&](long long n) {
        while (pc.n <= n && !pc.done) {
            const int s = (int)(pc.n % NSTAGE);
            if (pc.n >= NSTAGE) mbar_wait(&empty[s], (uint32_t)(((pc.n - NSTAGE) / NSTAGE) & 1));
            if (!try_issue(s, true)) {   // watchdog fired: release everyone waiting on this stage
                s_abort = 1;
                mbar_arrive_expect_tx(&full[s], 0);
                return;
            }
        }
    };

    long long n = 0;
    int ino = 0;
    for (int r = 0; r < pp.restarts; ++r) {
        const long long g0 = (long long)r * (pp.per + 1);   // ring offset of the interval
        // ---- seeds: step 0 of every level = the interval's state0 (top-level final before)
        const double* src = r == 0 ? pp.y0 : ring_slot(ep, top, pp.per, g0 - (pp.per + 1));
        for (int j = 0; j <= top; ++j) {
            for (int m = 0; m < my_tiles; ++m) {
                const int tile = (int)blockIdx.x + m * G;
                if (tid == 0 && !wait_deps<KIND>(ep, pp, j, 0, g0, 0, tile)) s_abort = 1;
                csync<NT>();
                if (s_abort) return;
                const Geo g = make_geo<KIND, NT, KMAX>(ep.pb, ep.sv, tile);
                const size_t base = (size_t)g.row * ep.pb.nx + g.c0;
                double* dst = ring_slot(ep, j, 0, g0) + base;
                for (int i = tid; i < g.tlen; i += NT) dst[i] = src[base + i];
                csync<NT>();
                if (tid == 0) {
                    __threadfence();
                    st_release(pp.flags + (size_t)j * pp.ipl + tile, g0);
                }
            }
        }
        // ---- ticks
        for (long long k = 1; k <= ticks; ++k) {
            int nact = 0;
            for (int j = 0; j <= top; ++j)
                if (active(k, j)) {
                    if (tid == 0) build_item(ep, j, k - delay(j), items[k & 1][nact], g0);
                    ++nact;
                }
            csync<NT>();
            int slot = 0;
            for (int j = 0; j <= top; ++j) {
                if (!active(k, j)) continue;
                const long long t = k - delay(j);
                const StepItem& it = items[k & 1][slot++];
                for (int m = 0; m < my_tiles; ++m, ++ino) {
                    const int tile = (int)blockIdx.x + m * G;
                    Geo geo = make_geo<KIND, NT, KMAX>(ep.pb, ep.sv, tile);
                    geo.item_no = ino;
                    if (geo.fast)
                        consume_item<KIND, NT, KMAX, ROWS, NSTAGE, true>(ep.pb, ep.sv, it, geo, stage, full, empty, n,
                                                                        refill, ensure, sbuf, swarp, ep.err,
                                                                        &s_abort);
                    else
                        consume_item<KIND, NT, KMAX, ROWS, NSTAGE, false>(ep.pb, ep.sv, it, geo, stage, full, empty,
                                                                         n, refill, ensure, sbuf, swarp, ep.err,
                                                                         &s_abort);
                    csync<NT>();
                    if (s_abort) return;
                    if (tid == 0) {
                        __threadfence();
                        st_release(pp.flags + (size_t)j * pp.ipl + tile, g0 + t);
                    }
                }
            }
        }
    }
}

template <int KIND, int NT, int KMAX>
__global__ void __launch_bounds__(NT) k_item(DevProblem pb, DevSolve sv, StepItem it,
                                             unsigned long long* err)
{
    extern __shared__ double sbuf[];
    __shared__ Aff swarp[2 * (NT / 32) + 1];
    process_item<KIND, NT, KMAX>(pb, sv, it, blockIdx.x, sbuf, swarp, err);
}

// state0 -> slot 0 of every level ring (engine.py:357-360: step 0 = initial data)
__global__ void k_seed(const double* __restrict__ src, EngineParams ep)
{
    const long long V = ep.V;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < V;
         i += (long long)gridDim.x * blockDim.x) {
        const double v = src[i];
        for (int j = 0; j < ep.levels; ++j) ring_slot(ep, j, 0)[i] = v;
    }
}

template <int KIND>
__global__ void k_apply(DevProblem pb, int op, const double* __restrict__ in, double* __restrict__ out)
{
    const long long V = (long long)pb.nx * pb.ny;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < V;
         i += (long long)gridDim.x * blockDim.x) {
        const int row = (int)(i / pb.nx), col = (int)(i - (long long)row * pb.nx);
        const double* rp = in + (size_t)row * pb.nx;
        const double* rn = in + (size_t)(row == 0 ? pb.ny - 1 : row - 1) * pb.nx;
        const double* rs = in + (size_t)(row == pb.ny - 1 ? 0 : row + 1) * pb.nx;
        double u, fs, fn;
        eval_point<KIND>(pb, rp, rn, rs, col, op == RIDC_OP_STIFF, op == RIDC_OP_NONSTIFF, u, fs, fn);
        out[i] = op == RIDC_OP_STIFF ? fs : fn;
    }
}

// ---------------------------------------------------------------- dispatch

struct LaunchCfg {
    int id;       // 0: 128x8, 1: 256x8, 2: 512x8
    int nt, kmax;
    size_t smem;
};

// Largest extended range one item handles (positions incl. the two stencil
// neighbours): 512 threads x 8 points.
constexpr int kCap = 512 * 8;

LaunchCfg pick_cfg(int Q)
{
    LaunchCfg c;
    if (Q <= 128 * 8) { c.id = 0; c.nt = 128; c.kmax = 8; }
    else if (Q <= 256 * 8) { c.id = 1; c.nt = 256; c.kmax = 8; }
    else { c.id = 2; c.nt = 512; c.kmax = 8; }
    const int cap = c.nt * c.kmax;
    c.smem = (size_t)(cap + cap / 16 + 1) * sizeof(double);
    return c;
}

template <int KIND, int NT, int KMAX>
cudaError_t launch_item_t(int items, size_t smem, cudaStream_t st, const DevProblem& pb,
                          const DevSolve& sv, const StepItem& it, unsigned long long* err)
{
    static bool attr[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
    if (!attr[dev]) {
        cudaError_t e = cudaFuncSetAttribute(k_item<KIND, NT, KMAX>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        attr[dev] = true;
    }
    k_item<KIND, NT, KMAX><<<items, NT, smem, st>>>(pb, sv, it, err);
    return cudaGetLastError();
}

#define RIDC_DISPATCH_CFG(FN, KIND, CFG, ...)                          \
    ((CFG).id == 0 ? FN<KIND, 128, 8>(__VA_ARGS__)                     \
     : (CFG).id == 1 ? FN<KIND, 256, 8>(__VA_ARGS__)                   \
                     : FN<KIND, 512, 8>(__VA_ARGS__))

// ---- TMA tick kernel configurations (NT consumers x KMAX points, ROWS staged
// rows per node, NSTAGE stages).  Many warps per SM hide the fp64 / shared
// memory latencies of the scans; 1-D items are sized so one item per level
// per CTA covers the line (see make_solve's balancing).
struct TmaCfg {
    int id;
    int nt, kmax, rows, nstage, cap;
    size_t smem;
};

template <int NT, int KMAX, int ROWS, int NSTAGE>
TmaCfg tma_cfg_of(int id)
{
    TmaCfg c;
    c.id = id;
    c.nt = NT;
    c.kmax = KMAX;
    c.rows = ROWS;
    c.nstage = NSTAGE;
    c.cap = NT * KMAX;
    c.smem = TmaSmem<NT, KMAX, ROWS, NSTAGE>::BYTES;
    return c;
}

#define RIDC_TMA_CONFIGS(X)        \
    X(0, 128, 8, 1, 4)             \
    X(1, 256, 8, 1, 4)             \
    X(2, 512, 8, 1, 3)             \
    X(3, 1024, 8, 1, 2)            \
    X(4, 256, 4, 3, 3)             \
    X(5, 512, 4, 3, 3)             \
    X(6, 512, 16, 1, 2)

TmaCfg pick_tma(int kind, int Q)
{
    const bool two_d = kind == ADV_DIFF_2D || kind == RD_2D;
    if (two_d) return Q <= 1024 ? tma_cfg_of<256, 4, 3, 3>(4) : tma_cfg_of<512, 4, 3, 3>(5);
    if (Q <= 1024) return tma_cfg_of<128, 8, 1, 4>(0);
    if (Q <= 2048) return tma_cfg_of<256, 8, 1, 4>(1);
    if (Q <= 4096) return tma_cfg_of<512, 8, 1, 3>(2);
    if (getenv("RIDC_CFG1024")) return tma_cfg_of<1024, 8, 1, 2>(3);
    return tma_cfg_of<512, 16, 1, 2>(6);
}

int tma_cap(int kind) { return (kind == ADV_DIFF_2D || kind == RD_2D) ? 2048 : 8192; }

template <int KIND, int NT, int KMAX, int ROWS, int NSTAGE>
cudaError_t launch_tma_t(int grid, size_t smem, cudaStream_t st, const EngineParams& ep,
                         const TickParams& tp, int ipl)
{
    auto kfn = k_tick_tma<KIND, NT, KMAX, ROWS, NSTAGE>;
    static bool attr[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
    if (!attr[dev]) {
        cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        attr[dev] = true;
    }
    kfn<<<grid, NT, smem, st>>>(ep, tp, ipl);
    return cudaGetLastError();
}

template <int KIND>
cudaError_t launch_tma_k(const TmaCfg& c, int grid, cudaStream_t st, const EngineParams& ep,
                         const TickParams& tp, int ipl)
{
    constexpr bool two_d = KIND == ADV_DIFF_2D || KIND == RD_2D;
#define RIDC_TMA_CASE(ID, NT, KMAX, ROWS, NSTAGE)                                      \
    if (c.id == ID && two_d == (ROWS == 3)) {                                          \
        if constexpr (two_d == (ROWS == 3))                                            \
            return launch_tma_t<KIND, NT, KMAX, ROWS, NSTAGE>(grid, c.smem, st, ep, tp, ipl); \
    }
    RIDC_TMA_CONFIGS(RIDC_TMA_CASE)
#undef RIDC_TMA_CASE
    return cudaErrorInvalidValue;
}

template <int KIND, int NT, int KMAX, int ROWS, int NSTAGE>
cudaError_t launch_persist_t(int grid, size_t smem, cudaStream_t st, const EngineParams& ep,
                             const PersistParams& pp)
{
    auto kfn = k_persist<KIND, NT, KMAX, ROWS, NSTAGE>;
    static bool attr[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
    if (!attr[dev]) {
        cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        attr[dev] = true;
    }
    // cooperative: every CTA co-resident (the flag protocol needs it), else the launch fails
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kfn, ep, pp);
}

template <int KIND>
cudaError_t launch_persist_k(const TmaCfg& c, int grid, cudaStream_t st, const EngineParams& ep,
                             const PersistParams& pp)
{
    constexpr bool two_d = KIND == ADV_DIFF_2D || KIND == RD_2D;
#define RIDC_PERSIST_CASE(ID, NT, KMAX, ROWS, NSTAGE)                                  \
    if (c.id == ID && two_d == (ROWS == 3)) {                                          \
        if constexpr (two_d == (ROWS == 3))                                            \
            return launch_persist_t<KIND, NT, KMAX, ROWS, NSTAGE>(grid, c.smem, st, ep, pp); \
    }
    RIDC_TMA_CONFIGS(RIDC_PERSIST_CASE)
#undef RIDC_PERSIST_CASE
    return cudaErrorInvalidValue;
}

cudaError_t launch_persist(int kind, const TmaCfg& c, int grid, cudaStream_t st, const EngineParams& ep,
                           const PersistParams& pp)
{
    switch (kind) {
    case ADV_DIFF_1D: return launch_persist_k<ADV_DIFF_1D>(c, grid, st, ep, pp);
    case BURGERS_1D: return launch_persist_k<BURGERS_1D>(c, grid, st, ep, pp);
    case RD_1D: return launch_persist_k<RD_1D>(c, grid, st, ep, pp);
    case ADV_DIFF_2D: return launch_persist_k<ADV_DIFF_2D>(c, grid, st, ep, pp);
    case RD_2D: return launch_persist_k<RD_2D>(c, grid, st, ep, pp);
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_tma(int kind, const TmaCfg& c, int grid, cudaStream_t st, const EngineParams& ep,
                       const TickParams& tp, int ipl)
{
    const bool two_d = kind == ADV_DIFF_2D || kind == RD_2D;
    if (two_d != (c.rows == 3)) return cudaErrorInvalidValue;
    switch (kind) {
    case ADV_DIFF_1D: return launch_tma_k<ADV_DIFF_1D>(c, grid, st, ep, tp, ipl);
    case BURGERS_1D: return launch_tma_k<BURGERS_1D>(c, grid, st, ep, tp, ipl);
    case RD_1D: return launch_tma_k<RD_1D>(c, grid, st, ep, tp, ipl);
    case ADV_DIFF_2D: return launch_tma_k<ADV_DIFF_2D>(c, grid, st, ep, tp, ipl);
    case RD_2D: return launch_tma_k<RD_2D>(c, grid, st, ep, tp, ipl);
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_item(int kind, const LaunchCfg& c, int items, cudaStream_t st,
                        const DevProblem& pb, const DevSolve& sv, const StepItem& it,
                        unsigned long long* err)
{
    switch (kind) {
    case ADV_DIFF_1D: return RIDC_DISPATCH_CFG(launch_item_t, ADV_DIFF_1D, c, items, c.smem, st, pb, sv, it, err);
    case BURGERS_1D: return RIDC_DISPATCH_CFG(launch_item_t, BURGERS_1D, c, items, c.smem, st, pb, sv, it, err);
    case RD_1D: return RIDC_DISPATCH_CFG(launch_item_t, RD_1D, c, items, c.smem, st, pb, sv, it, err);
    case ADV_DIFF_2D: return RIDC_DISPATCH_CFG(launch_item_t, ADV_DIFF_2D, c, items, c.smem, st, pb, sv, it, err);
    case RD_2D: return RIDC_DISPATCH_CFG(launch_item_t, RD_2D, c, items, c.smem, st, pb, sv, it, err);
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_apply(const DevProblem& pb, int op, const double* in, double* out, cudaStream_t st)
{
    const long long V = (long long)pb.nx * pb.ny;
    int blocks = (int)std::min<long long>((V + 255) / 256, 148 * 16);
    switch (pb.kind) {
    case ADV_DIFF_1D: k_apply<ADV_DIFF_1D><<<blocks, 256, 0, st>>>(pb, op, in, out); break;
    case BURGERS_1D: k_apply<BURGERS_1D><<<blocks, 256, 0, st>>>(pb, op, in, out); break;
    case RD_1D: k_apply<RD_1D><<<blocks, 256, 0, st>>>(pb, op, in, out); break;
    case ADV_DIFF_2D: k_apply<ADV_DIFF_2D><<<blocks, 256, 0, st>>>(pb, op, in, out); break;
    case RD_2D: k_apply<RD_2D><<<blocks, 256, 0, st>>>(pb, op, in, out); break;
    default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

// ---------------------------------------------------------------- host setup

int fail(std::string* dst, int code, const std::string& msg)
{
    g_last_error = msg;
    if (dst) *dst = msg;
    return code;
}

#define CUDA_TRY(dst, expr)                                                            \
    do {                                                                               \
        cudaError_t _e = (expr);                                                       \
        if (_e != cudaSuccess)                                                         \
            return fail(dst, RIDC_E_CUDA, std::string(#expr " failed: ") +             \
                                              cudaGetErrorString(_e));                 \
    } while (0)

int validate_problem(const ridc_problem* p)
{
    if (!p) return fail(nullptr, RIDC_E_CONFIG, "problem is NULL");
    if (p->kind < 1 || p->kind > 5) return fail(nullptr, RIDC_E_CONFIG, "unknown problem kind");
    if (p->nx < 3 || p->ny < 1) return fail(nullptr, RIDC_E_DIMENSION, "grid too small (nx >= 3)");
    const bool two_d = p->kind == ADV_DIFF_2D || p->kind == RD_2D;
    if (two_d && p->ny < 3) return fail(nullptr, RIDC_E_DIMENSION, "2-D problems need ny >= 3");
    if (!two_d && p->ny != 1) return fail(nullptr, RIDC_E_DIMENSION, "1-D problems need ny == 1");
    if (!(p->d_x > 0.0) || !(p->h_x > 0.0) || (two_d && !(p->h_y > 0.0)))
        return fail(nullptr, RIDC_E_CONFIG, "need d_x > 0 and positive grid spacings");
    return RIDC_OK;
}

DevProblem make_problem(const ridc_problem* p)
{
    DevProblem d;
    d.kind = p->kind;
    d.nx = p->nx;
    d.ny = p->ny;
    d.periodic = p->kind != BURGERS_1D;
    d.cax = p->c_x / p->h_x;
    d.cay = p->ny > 1 ? p->c_y / p->h_y : 0.0;
    d.cdx = p->d_x / (p->h_x * p->h_x);
    d.cdy = p->ny > 1 ? p->d_y / (p->h_y * p->h_y) : 0.0;
    d.rho = p->rho;
    d.bs = 1.0 / (4.0 * p->h_x);
    return d;
}

// Host precompute of the shifted-operator factors (the analogue of
// qr_factor(I - dt L), linalg.py:33-56, done once per run).
struct SolveSetup {
    DevSolve sv;
    std::vector<double> tab;   // [m_0..m_{n-1}, g_0..g_{n-1}]
    std::vector<PlanRow> plans;  // TMA staging plans [nseg][row parity]
    double r;
    LaunchCfg cfg;             // register-path (single-op) launch
    TmaCfg tcfg;               // TMA tick-kernel launch (engine)
    std::string err;
};

// Host mirror of make_geo (ridc_device.cuh) for one segment.
void seg_range(const DevProblem& pb, const DevSolve& sv, int seg, int& cf, int& Q)
{
    const int nx = pb.nx;
    const int c0 = seg * sv.tile;
    const int tlen = std::min(sv.tile, nx - c0);
    int s0, S;
    if (sv.nseg == 1) { s0 = 0; S = nx; }
    else if (pb.periodic) { s0 = c0 - sv.halo; S = tlen + 2 * sv.halo; }
    else {
        s0 = std::max(c0 - sv.halo, 0);
        S = std::min(c0 + tlen + sv.halo, nx) - s0;
    }
    cf = s0 - 1;
    Q = S + 2;
}

// Staging plan of one row-segment (see PlanRow in ridc_tma.cuh): aligned
// bulk runs for the TMA engine, the rest as consumer fills.
PlanRow make_plan_host(const DevProblem& pb, int cf, int Q, int par)
{
    const int nx = pb.nx;
    struct Run { int q0, c0, n; };
    std::vector<Run> runs;
    std::vector<std::pair<int, int>> fills;   // [q0, q1)
    int q = 0;
    while (q < Q) {
        const int c = cf + q;
        if (!pb.periodic && (c < 0 || c >= nx)) {   // Dirichlet ghost
            fills.push_back({q, q + 1});
            ++q;
            continue;
        }
        const int cc = pb.periodic ? ((c % nx) + nx) % nx : c;
        const int n = std::min(Q - q, nx - cc);
        runs.push_back({q, cc, n});
        q += n;
    }
    PlanRow pl;
    memset(&pl, 0, sizeof pl);
    int best = 0;
    for (int k = 1; k < (int)runs.size(); ++k)
        if (runs[k].n > runs[best].n) best = k;
    pl.sigma = runs.empty() ? 0 : ((par + runs[best].c0 - runs[best].q0) & 1);
    const bool single = runs.size() == 1 && runs[0].q0 == 0 && runs[0].n == Q;
    bool overflow = runs.size() > (size_t)kMaxBulk;
    for (const Run& r : runs) {
        const int dpar = (pl.sigma + r.q0) & 1, spar = (par + r.c0) & 1;
        if (dpar != spar || overflow) { fills.push_back({r.q0, r.q0 + r.n}); continue; }
        int q0, col, n;
        if (single) {
            const int h = (pl.sigma + r.q0) & 1;
            q0 = r.q0 - h; col = r.c0 - h; n = r.n + h; n += n & 1;
        } else {
            const int h = (pl.sigma + r.q0) & 1;
            q0 = r.q0 + h; col = r.c0 + h; n = r.n - h; n -= n & 1;
            if (n <= 0) { fills.push_back({r.q0, r.q0 + r.n}); continue; }
            if (q0 > r.q0) fills.push_back({r.q0, q0});
            if (q0 + n < r.q0 + r.n) fills.push_back({q0 + n, r.q0 + r.n});
        }
        pl.bq0[pl.nb] = q0;
        pl.bcol[pl.nb] = col;
        pl.bn[pl.nb] = n;
        pl.bytes += n * 8;
        ++pl.nb;
    }
    std::sort(fills.begin(), fills.end());
    std::vector<std::pair<int, int>> merged;
    for (auto& f : fills) {
        if (!merged.empty() && merged.back().second >= f.first)
            merged.back().second = std::max(merged.back().second, f.second);
        else
            merged.push_back(f);
    }
    if (merged.size() > (size_t)kMaxFill) {   // degenerate: consumers stage everything
        pl.nb = 0;
        pl.bytes = 0;
        merged.assign(1, {0, Q});
    }
    pl.nf = (int)merged.size();
    for (int f = 0; f < pl.nf; ++f) {
        pl.fq0[f] = merged[f].first;
        pl.fn[f] = merged[f].second - merged[f].first;
    }
    return pl;
}

void build_plans(const DevProblem& pb, SolveSetup& ss)
{
    ss.plans.clear();
    for (int seg = 0; seg < ss.sv.nseg; ++seg) {
        int cf, Q;
        seg_range(pb, ss.sv, seg, cf, Q);
        for (int par = 0; par < 2; ++par) ss.plans.push_back(make_plan_host(pb, cf, Q, par));
    }
}

// Factors + tiling.  cap: largest item range (positions incl. 2 stencil
// neighbours) the chosen kernel holds; balance_items > 0 asks for the
// segment count that best balances `balance_items` items-per-segment over
// `nsm` persistent CTAs (engine), 0 for the minimal count (single ops).
int make_solve(const DevProblem& pb, double coeff, int cap, int balance_items, int nsm,
               SolveSetup& ss)
{
    const double r = coeff * pb.cdx;
    ss.r = r;
    DevSolve& sv = ss.sv;
    memset(&sv, 0, sizeof sv);
    const double b = 1.0 + 2.0 * r;
    const double s = std::sqrt(1.0 + 4.0 * r);
    sv.lam = 2.0 * r / (b + s);
    sv.g = 2.0 / (b + s);
    if (!pb.periodic) {
        // Thomas pivots den_i = b - r^2/den_{i-1} converge geometrically;
        // keep the exact prefix, then the fixed point.
        std::vector<double> m, g;
        double den = b;
        for (int i = 0; i < pb.nx; ++i) {
            if (i > 0) {
                const double nd = b - r * r / den;
                if (nd == den && i > 1) break;
                den = nd;
            }
            m.push_back(r / den);
            g.push_back(1.0 / den);
        }
        sv.ntab = (int)m.size();
        sv.lam = m.back();
        sv.g = g.back();
        ss.tab.assign(m.begin(), m.end());
        ss.tab.insert(ss.tab.end(), g.begin(), g.end());
    }
    double pw = 1.0;
    for (int e = 0; e < kMaxChunk; ++e) {
        pw *= sv.lam;
        sv.pw[e] = pw;
    }
    // zf[e] = sum_{k=e}^{K-1} lam^(k-e) lam^(k+1)  (fast_solve, ridc_device.cuh)
    auto fill_zf = [&](double* zf, int K) {
        for (int e = 0; e < K; ++e) {
            double acc = 0.0;
            for (int k = K - 1; k >= e; --k) acc = acc * sv.lam + sv.pw[k];
            zf[e] = acc;   // Horner in lam over k: sum lam^(k-e) * lam^(k+1)
        }
    };
    fill_zf(sv.zf4, 4);
    fill_zf(sv.zf8, 8);
    fill_zf(sv.zf16, 16);
    if (pb.nx + 2 <= cap) {
        sv.nseg = 1;
        sv.tile = pb.nx;
        sv.halo = 0;
        ss.cfg = pick_cfg(pb.nx + 2);
        ss.tcfg = pick_tma(pb.kind, pb.nx + 2);
        build_plans(pb, ss);
        return RIDC_OK;
    }
    // truncated halo: lam^H <= 2^-60 relative to the recurrence magnitude
    int H = 0;
    if (sv.lam > 0.0) H = (int)std::ceil(60.0 * std::log(2.0) / -std::log(sv.lam)) + 1;
    const int Tmax = cap - 2 - 2 * H;
    if (Tmax < 256) {
        char buf[256];
        snprintf(buf, sizeof buf,
                 "stiffness r=%.4g needs a truncation halo of %d points; the segmented "
                 "line solve supports at most %d (use fewer points or a smaller dt)",
                 r, H, (cap - 2 - 256) / 2);
        ss.err = buf;
        return RIDC_E_CONFIG;
    }
    const int n0 = (pb.nx + Tmax - 1) / Tmax;
    int nbest = n0;
    if (balance_items > 0 && nsm > 0) {
        // minimise the per-CTA positions of the busiest CTA (+ a fixed per-item cost)
        long long best = LLONG_MAX;
        for (int n = n0; n <= 4 * n0; ++n) {
            const int T = (pb.nx + n - 1) / n;
            const long long items = (long long)balance_items * n;
            const long long per = (items + nsm - 1) / nsm;
            const long long cost = per * (T + 2LL * H + 2 + 512);
            if (cost < best) { best = cost; nbest = n; }
        }
    }
    sv.halo = H;
    sv.tile = (pb.nx + nbest - 1) / nbest;
    sv.nseg = (pb.nx + sv.tile - 1) / sv.tile;
    ss.cfg = pick_cfg(cap);
    ss.tcfg = pick_tma(pb.kind, cap);
    build_plans(pb, ss);
    return RIDC_OK;
}

}  // namespace

// ================================================================ context

struct ridc_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    ridc_problem prob;
    DevProblem pb;
    SolveSetup ss;
    double t_start = 0, t_end = 0, dt = 0;
    int levels = 0, restarts = 0;
    long long steps = 0, per = 0, ticks = 0;
    uint32_t flags = 0;
    long long V = 0;
    double* d_weights = nullptr;
    double* d_tab = nullptr;
    PlanRow* d_plans = nullptr;
    long long* d_dbg = nullptr;
    double* d_ring[kMaxLevels] = {};
    long long cap[kMaxLevels] = {};
    double* d_y0 = nullptr;
    unsigned long long* d_err = nullptr;
    EngineParams ep;
    std::vector<int> steady_off, startup_off;
    cudaGraphExec_t gexec = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    long long launches = 0;
    long long ring_vectors = 0;
    long long Vs = 0;          // ring slot stride (doubles)
    int nsm = 148;             // persistent CTAs per tick launch
    bool persistent = false;   // one k_persist launch per run (else a graph of tick launches)
    long long* d_flags = nullptr;
    int* d_abort = nullptr;
    PersistParams pp;
    double* d_ring_base[kMaxLevels] = {};
    std::string err;
};

namespace {

long long delay(int j) { return (long long)j * (j + 1) / 2; }   // engine.py:50-54

// Offsets of the packed weight tables (quadrature.pack_weight_tables).
void weight_offsets(int L, std::vector<int>& st, std::vector<int>& su, long long& total)
{
    st.assign(kMaxLevels, 0);
    su.assign(kMaxLevels, 0);
    long long off = 0;
    for (int j = 1; j < L; ++j) { st[j] = (int)off; off += j + 1; }
    for (int j = 2; j < L; ++j) { su[j] = (int)off; off += (long long)(j - 1) * (j + 1); }
    total = off;
}

EngineParams interval_params(ridc_ctx* c, int interval)
{
    EngineParams ep = c->ep;
    for (int j = 0; j < c->levels; ++j) ep.off[j] = c->persistent ? (long long)interval * (c->per + 1) : 0;
    if (c->flags & RIDC_RECORD_TRAJECTORY) ep.off[c->levels - 1] = (long long)interval * c->per;
    return ep;
}

// Capture the whole run: per interval one seed + one launch per tick.
int capture_graph(ridc_ctx* c)
{
    const int L = c->levels;
    const int items = c->pb.ny * c->ss.sv.nseg;
    cudaGraph_t graph = nullptr;
    CUDA_TRY(&c->err, cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    long long launches = 0;
    cudaError_t le = cudaSuccess;
    for (int r = 0; r < c->restarts && le == cudaSuccess; ++r) {
        EngineParams ep = interval_params(c, r);
        const double* src = c->d_y0;
        if (r > 0) {
            EngineParams prev = interval_params(c, r - 1);
            const int top = L - 1;
            src = prev.ring[top] + ((prev.off[top] + c->per) % prev.cap[top]) * c->Vs;
        }
        int sb = (int)std::min<long long>((c->V + 255) / 256, 148 * 8);
        k_seed<<<sb, 256, 0, c->stream>>>(src, ep);
        le = cudaGetLastError();
        ++launches;
        for (long long k = 1; k <= c->ticks && le == cudaSuccess; ++k) {
            TickParams tp;
            memset(&tp, 0, sizeof tp);
            for (int j = 0; j < L; ++j) {
                const long long t = k - delay(j);
                if (t >= 1 && t <= c->per) {
                    tp.level[tp.nact] = j;
                    tp.target[tp.nact] = t;
                    ++tp.nact;
                }
            }
            if (tp.nact == 0) continue;
            le = launch_tma(c->pb.kind, c->ss.tcfg, std::min(c->nsm, tp.nact * items), c->stream, ep,
                            tp, items);
            ++launches;
        }
    }
    cudaError_t ce = cudaStreamEndCapture(c->stream, &graph);
    if (le != cudaSuccess) {
        if (graph) cudaGraphDestroy(graph);
        return fail(&c->err, RIDC_E_CUDA, std::string("kernel launch during capture: ") +
                                              cudaGetErrorString(le));
    }
    CUDA_TRY(&c->err, ce);
    cudaError_t ie = cudaGraphInstantiate(&c->gexec, graph, 0);
    cudaGraphDestroy(graph);
    CUDA_TRY(&c->err, ie);
    c->launches = launches;
    return RIDC_OK;
}

int check_err_word(ridc_ctx* c)
{
    unsigned long long w = 0;
    CUDA_TRY(&c->err, cudaMemcpyAsync(&w, c->d_err, sizeof w, cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(&c->err, cudaStreamSynchronize(c->stream));
    if (w != ULLONG_MAX) {
        char buf[160];
        snprintf(buf, sizeof buf, "level %d produced non-finite entries at step %lld",
                 (int)(w & 0xff), (long long)(w >> 8));
        return fail(&c->err, RIDC_E_NONFINITE, buf);
    }
    return RIDC_OK;
}

int march(ridc_ctx* c, double* wall_seconds)
{
    CUDA_TRY(&c->err, cudaMemsetAsync(c->d_err, 0xff, sizeof(unsigned long long), c->stream));
    if (c->persistent) {
        CUDA_TRY(&c->err, cudaMemsetAsync(c->d_flags, 0xff,
                                          sizeof(long long) * c->levels * c->pp.ipl, c->stream));
        CUDA_TRY(&c->err, cudaMemsetAsync(c->d_abort, 0, sizeof(int), c->stream));
    }
    CUDA_TRY(&c->err, cudaEventRecord(c->ev0, c->stream));
    if (c->persistent)
        CUDA_TRY(&c->err, launch_persist(c->pb.kind, c->ss.tcfg, std::min(c->nsm, c->pp.ipl), c->stream,
                                         interval_params(c, 0), c->pp));
    else
        CUDA_TRY(&c->err, cudaGraphLaunch(c->gexec, c->stream));
    CUDA_TRY(&c->err, cudaEventRecord(c->ev1, c->stream));
    CUDA_TRY(&c->err, cudaEventSynchronize(c->ev1));
    if (c->persistent) {
        int ab = 0;
        CUDA_TRY(&c->err, cudaMemcpy(&ab, c->d_abort, sizeof ab, cudaMemcpyDeviceToHost));
        if (ab) return fail(&c->err, RIDC_E_PROTOCOL, "tile pipeline made no progress within the watchdog");
    }
    if (wall_seconds) {
        float ms = 0.f;
        CUDA_TRY(&c->err, cudaEventElapsedTime(&ms, c->ev0, c->ev1));
        *wall_seconds = ms * 1e-3;
    }
    return check_err_word(c);
}

const double* final_slot(ridc_ctx* c, int level)
{
    EngineParams ep = interval_params(c, c->restarts - 1);
    return ep.ring[level] + ((ep.off[level] + c->per) % ep.cap[level]) * c->Vs;
}

}  // namespace

extern "C" {

int ridc_create(const ridc_problem* problem, double t_start, double t_end, int32_t levels,
                int64_t steps, int32_t restarts, const double* weights, int64_t nweights,
                int32_t device, uint32_t flags, ridc_ctx** out)
{
    if (!out) return fail(nullptr, RIDC_E_CONFIG, "out is NULL");
    *out = nullptr;
    int rc = validate_problem(problem);
    if (rc) return rc;
    // RidcConfig.__post_init__ (engine.py:71-87)
    if (levels < 1 || levels > kMaxLevels)
        return fail(nullptr, RIDC_E_CONFIG, "levels must be in 1..12");
    if (steps < 1 || restarts < 1) return fail(nullptr, RIDC_E_CONFIG, "steps and restarts must be positive");
    if (steps % restarts) return fail(nullptr, RIDC_E_CONFIG, "steps must be divisible by restarts");
    const long long per = steps / restarts;
    if (per < delay(levels) + 1) {
        char buf[160];
        snprintf(buf, sizeof buf, "each restart interval has %lld steps; %d levels need >= %lld",
                 per, levels, delay(levels) + 1);
        return fail(nullptr, RIDC_E_CONFIG, buf);
    }
    if (!(t_start < t_end)) return fail(nullptr, RIDC_E_CONFIG, "need t_start < t_end");
    std::vector<int> st, su;
    long long wtotal = 0;
    weight_offsets(levels, st, su, wtotal);
    if (nweights < wtotal || (wtotal > 0 && !weights))
        return fail(nullptr, RIDC_E_DIMENSION, "weight table shorter than levels require");

    ridc_ctx* c = new ridc_ctx();
    c->device = device;
    c->prob = *problem;
    c->pb = make_problem(problem);
    c->t_start = t_start;
    c->t_end = t_end;
    c->levels = levels;
    c->steps = steps;
    c->restarts = restarts;
    c->per = per;
    c->ticks = per + delay(levels - 1);
    c->flags = flags;
    c->V = (long long)problem->nx * problem->ny;
    c->Vs = ((c->V + 1) & ~1LL) + 4;
    c->dt = (t_end - t_start) / (double)steps;   // engine.py:468 global dt
    c->steady_off = st;
    c->startup_off = su;
    auto bail = [&](int code) {
        std::string m = c->err.empty() ? g_last_error : c->err;
        ridc_destroy(c);
        g_last_error = m;
        return code;
    };
    if (cudaSetDevice(device) != cudaSuccess) {
        c->err = "cudaSetDevice failed";
        return bail(RIDC_E_CUDA);
    }
    if (cudaDeviceGetAttribute(&c->nsm, cudaDevAttrMultiProcessorCount, device) != cudaSuccess)
        c->nsm = 148;
    // tiling depends only on the problem and dt (not on levels or devices): the
    // one-level-per-GPU pipeline then reproduces these states bitwise
    if ((rc = make_solve(c->pb, c->dt, tma_cap(c->pb.kind), c->pb.ny, c->nsm, c->ss)) !=
        RIDC_OK) {
        c->err = c->ss.err;
        return bail(rc);
    }
#define CTX_TRY(expr)                                                                        \
    do {                                                                                     \
        cudaError_t _e = (expr);                                                             \
        if (_e != cudaSuccess) {                                                             \
            c->err = std::string(#expr " failed: ") + cudaGetErrorString(_e);               \
            return bail(RIDC_E_CUDA);                                                        \
        }                                                                                    \
    } while (0)
    CTX_TRY(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    CTX_TRY(cudaEventCreate(&c->ev0));
    CTX_TRY(cudaEventCreate(&c->ev1));
    const size_t vb = (size_t)c->V * sizeof(double);
    CTX_TRY(cudaMalloc(&c->d_weights, std::max<long long>(wtotal, 1) * sizeof(double)));
    if (wtotal > 0)
        CTX_TRY(cudaMemcpy(c->d_weights, weights, wtotal * sizeof(double), cudaMemcpyHostToDevice));
    if (!c->ss.tab.empty()) {
        CTX_TRY(cudaMalloc(&c->d_tab, c->ss.tab.size() * sizeof(double)));
        CTX_TRY(cudaMemcpy(c->d_tab, c->ss.tab.data(), c->ss.tab.size() * sizeof(double),
                           cudaMemcpyHostToDevice));
        c->ss.sv.tab_m = c->d_tab;
        c->ss.sv.tab_g = c->d_tab + c->ss.sv.ntab;
    }
    CTX_TRY(cudaMalloc(&c->d_plans, c->ss.plans.size() * sizeof(PlanRow)));
    CTX_TRY(cudaMemcpy(c->d_plans, c->ss.plans.data(), c->ss.plans.size() * sizeof(PlanRow),
                       cudaMemcpyHostToDevice));
    c->ss.sv.plans = c->d_plans;
    if (getenv("RIDC_PHASE_TIMING") && atoi(getenv("RIDC_PHASE_TIMING")) > 0) {
        CTX_TRY(cudaMalloc(&c->d_dbg, 128 * sizeof(long long)));
        CTX_TRY(cudaMemset(c->d_dbg, 0, 128 * sizeof(long long)));
        c->ss.sv.dbg = c->d_dbg;
    }
    for (int j = 0; j < levels; ++j) {
        const bool top = j == levels - 1;
        long long cap = top ? 2 : 2LL * j + 3;
        if (top && (flags & RIDC_RECORD_TRAJECTORY)) cap = steps + 1;
        c->cap[j] = cap;
        c->ring_vectors += cap;
        // slot stride Vs (even) keeps every slot 16-byte aligned for the bulk
        // copies; 2 guard doubles before slot 0 and >= 4 after each state
        CTX_TRY(cudaMalloc(&c->d_ring_base[j], ((size_t)cap * c->Vs + 4) * sizeof(double)));
        c->d_ring[j] = c->d_ring_base[j] + 2;
    }
    CTX_TRY(cudaMalloc(&c->d_y0, vb));
    CTX_TRY(cudaMalloc(&c->d_err, sizeof(unsigned long long)));
    EngineParams& ep = c->ep;
    memset(&ep, 0, sizeof ep);
    ep.pb = c->pb;
    ep.sv = c->ss.sv;
    ep.V = c->V;
    ep.Vs = c->Vs;
    ep.dt = c->dt;
    ep.levels = levels;
    for (int j = 0; j < levels; ++j) {
        ep.ring[j] = c->d_ring[j];
        ep.cap[j] = c->cap[j];
    }
    ep.weights = c->d_weights;
    for (int j = 0; j < kMaxLevels; ++j) {
        ep.steady_off[j] = st[j];
        ep.startup_off[j] = su[j];
    }
    ep.err = c->d_err;
    // opt-in (RIDC_PERSIST=1): one persistent launch per run with per-tile
    // dependency flags.  Measured slower than the tick graph on B200 for every
    // workload (flag hand-off + unprefetchable dependent loads ~ the launch gap),
    // so the graph of tick launches is the default.
    const char* ps = getenv("RIDC_PERSIST");
    c->persistent = !(flags & RIDC_RECORD_TRAJECTORY) && (ps && atoi(ps) > 0);
    if (c->persistent) {
        const DevSolve& sv = c->ss.sv;
        PersistParams& pp = c->pp;
        memset(&pp, 0, sizeof pp);
        pp.ipl = c->pb.ny * sv.nseg;
        pp.rx = sv.nseg > 1 ? (sv.halo + 1 + sv.tile - 1) / sv.tile : 0;
        pp.levels = levels;
        pp.restarts = restarts;
        pp.per = per;
        CTX_TRY(cudaMalloc(&c->d_flags, sizeof(long long) * levels * pp.ipl));
        CTX_TRY(cudaMalloc(&c->d_abort, sizeof(int)));
        pp.flags = c->d_flags;
        pp.abort = c->d_abort;
        pp.y0 = c->d_y0;
        pp.timeout_ns = 10ull * 1000 * 1000 * 1000;
        c->launches = 1;
    } else if ((rc = capture_graph(c)) != RIDC_OK) {
        return bail(rc);
    }
#undef CTX_TRY
    *out = c;
    return RIDC_OK;
}

int ridc_run(ridc_ctx* c, const double* y0_host, double* final_host, double* level_finals_host,
             double* traj_host, double* wall_seconds)
{
    if (!c || !y0_host || !final_host) return fail(c ? &c->err : nullptr, RIDC_E_CONFIG, "NULL argument");
    if (traj_host && !(c->flags & RIDC_RECORD_TRAJECTORY))
        return fail(&c->err, RIDC_E_CONFIG, "trajectory requested but not recorded (flags)");
    CUDA_TRY(&c->err, cudaSetDevice(c->device));
    const size_t vb = (size_t)c->V * sizeof(double);
    CUDA_TRY(&c->err, cudaMemcpyAsync(c->d_y0, y0_host, vb, cudaMemcpyHostToDevice, c->stream));
    int rc = march(c, wall_seconds);
    if (rc) return rc;
    CUDA_TRY(&c->err, cudaMemcpyAsync(final_host, final_slot(c, c->levels - 1), vb,
                                      cudaMemcpyDeviceToHost, c->stream));
    if (level_finals_host)
        for (int j = 0; j < c->levels; ++j)
            CUDA_TRY(&c->err, cudaMemcpyAsync(level_finals_host + (size_t)j * c->V, final_slot(c, j),
                                              vb, cudaMemcpyDeviceToHost, c->stream));
    if (traj_host)
        CUDA_TRY(&c->err, cudaMemcpy2DAsync(traj_host, vb, c->d_ring[c->levels - 1],
                                            (size_t)c->Vs * sizeof(double), vb,
                                            (size_t)(c->steps + 1), cudaMemcpyDeviceToHost,
                                            c->stream));
    CUDA_TRY(&c->err, cudaStreamSynchronize(c->stream));
    return RIDC_OK;
}

int ridc_run_device(ridc_ctx* c, const double* y0_dev, double* final_dev, double* wall_seconds)
{
    if (!c || !y0_dev || !final_dev) return fail(c ? &c->err : nullptr, RIDC_E_CONFIG, "NULL argument");
    CUDA_TRY(&c->err, cudaSetDevice(c->device));
    const size_t vb = (size_t)c->V * sizeof(double);
    CUDA_TRY(&c->err, cudaMemcpyAsync(c->d_y0, y0_dev, vb, cudaMemcpyDeviceToDevice, c->stream));
    int rc = march(c, wall_seconds);
    if (rc) return rc;
    CUDA_TRY(&c->err, cudaMemcpyAsync(final_dev, final_slot(c, c->levels - 1), vb,
                                      cudaMemcpyDeviceToDevice, c->stream));
    CUDA_TRY(&c->err, cudaStreamSynchronize(c->stream));
    return RIDC_OK;
}

int ridc_info_get(const ridc_ctx* c, ridc_info* info)
{
    if (!c || !info) return fail(nullptr, RIDC_E_CONFIG, "NULL argument");
    info->levels = c->levels;
    info->restarts = c->restarts;
    info->steps = c->steps;
    info->ticks_per_interval = c->ticks;
    info->kernel_launches = c->launches;
    info->tile = c->ss.sv.tile;
    info->halo = c->ss.sv.halo;
    info->items_per_level = c->pb.ny * c->ss.sv.nseg;
    info->threads = c->ss.tcfg.nt;
    info->ring_vectors = c->ring_vectors;
    info->lambda = c->ss.sv.lam;
    info->r = c->ss.r;
    return RIDC_OK;
}

int ridc_destroy(ridc_ctx* c)
{
    if (!c) return RIDC_OK;
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    if (c->gexec) cudaGraphExecDestroy(c->gexec);
    for (int j = 0; j < kMaxLevels; ++j)
        if (c->d_ring_base[j]) cudaFree(c->d_ring_base[j]);
    if (c->d_weights) cudaFree(c->d_weights);
    if (c->d_tab) cudaFree(c->d_tab);
    if (c->d_plans) cudaFree(c->d_plans);
    if (c->d_dbg) cudaFree(c->d_dbg);
    if (c->d_flags) cudaFree(c->d_flags);
    if (c->d_abort) cudaFree(c->d_abort);
    if (c->d_y0) cudaFree(c->d_y0);
    if (c->d_err) cudaFree(c->d_err);
    if (c->ev0) cudaEventDestroy(c->ev0);
    if (c->ev1) cudaEventDestroy(c->ev1);
    if (c->stream) cudaStreamDestroy(c->stream);
    delete c;
    return RIDC_OK;
}

const char* ridc_last_error(const ridc_ctx* c)
{
    if (c && !c->err.empty()) return c->err.c_str();
    return g_last_error.c_str();
}

// ---------------------------------------------------------------- single ops

int ridc_op_apply(const ridc_problem* problem, int32_t op, const double* in_dev, double* out_dev,
                  int32_t device)
{
    int rc = validate_problem(problem);
    if (rc) return rc;
    if (op != RIDC_OP_STIFF && op != RIDC_OP_NONSTIFF) return fail(nullptr, RIDC_E_CONFIG, "bad op");
    CUDA_TRY(nullptr, cudaSetDevice(device));
    DevProblem pb = make_problem(problem);
    CUDA_TRY(nullptr, launch_apply(pb, op, in_dev, out_dev, 0));
    CUDA_TRY(nullptr, cudaDeviceSynchronize());
    return RIDC_OK;
}

static int run_single_item(const ridc_problem* problem, double coeff, StepItem& it, int32_t device)
{
    int rc = validate_problem(problem);
    if (rc) return rc;
    CUDA_TRY(nullptr, cudaSetDevice(device));
    DevProblem pb = make_problem(problem);
    SolveSetup ss;
    if ((rc = make_solve(pb, coeff, kCap, 0, 0, ss)) != RIDC_OK) return fail(nullptr, rc, ss.err);
    double* d_tab = nullptr;
    unsigned long long* d_err = nullptr;
    auto cleanup = [&]() {
        if (d_tab) cudaFree(d_tab);
        if (d_err) cudaFree(d_err);
    };
    if (!ss.tab.empty()) {
        if (cudaMalloc(&d_tab, ss.tab.size() * sizeof(double)) != cudaSuccess ||
            cudaMemcpy(d_tab, ss.tab.data(), ss.tab.size() * sizeof(double),
                       cudaMemcpyHostToDevice) != cudaSuccess) {
            cleanup();
            return fail(nullptr, RIDC_E_CUDA, "factor table upload failed");
        }
        ss.sv.tab_m = d_tab;
        ss.sv.tab_g = d_tab + ss.sv.ntab;
    }
    if (cudaMalloc(&d_err, sizeof(unsigned long long)) != cudaSuccess ||
        cudaMemset(d_err, 0xff, sizeof(unsigned long long)) != cudaSuccess) {
        cleanup();
        return fail(nullptr, RIDC_E_CUDA, "error word allocation failed");
    }
    cudaError_t e = launch_item(pb.kind, ss.cfg, pb.ny * ss.sv.nseg, 0, pb, ss.sv, it, d_err);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    unsigned long long w = ULLONG_MAX;
    if (e == cudaSuccess) e = cudaMemcpy(&w, d_err, sizeof w, cudaMemcpyDeviceToHost);
    cleanup();
    if (e != cudaSuccess) return fail(nullptr, RIDC_E_CUDA, cudaGetErrorString(e));
    if (w != ULLONG_MAX) return fail(nullptr, RIDC_E_NONFINITE, "step produced non-finite entries");
    return RIDC_OK;
}

int ridc_op_solve(const ridc_problem* problem, double coeff, const double* rhs_dev, double* x_dev,
                  int32_t device)
{
    StepItem it;
    memset(&it, 0, sizeof it);
    it.nnodes = 1;
    it.vec[0] = rhs_dev;
    it.ca[0] = 1.0;
    it.out = x_dev;
    it.level = 0;
    it.target = -1;
    return run_single_item(problem, coeff, it, device);
}

int ridc_op_step(const ridc_problem* problem, double dt, const double* eta_dev, int32_t nwin,
                 const double* const* win_dev, const double* cs, const double* cn, double* out_dev,
                 int32_t device)
{
    if (nwin < 0 || nwin > kMaxNodes - 1) return fail(nullptr, RIDC_E_PROTOCOL, "window too large");
    if (nwin > 0 && (!win_dev || !cs || !cn)) return fail(nullptr, RIDC_E_CONFIG, "NULL window");
    StepItem it;
    memset(&it, 0, sizeof it);
    it.nnodes = 1 + nwin;
    it.vec[0] = eta_dev;
    it.ca[0] = 1.0;
    it.cs[0] = 0.0;
    it.cn[0] = dt;
    for (int a = 0; a < nwin; ++a) {
        it.vec[1 + a] = win_dev[a];
        it.ca[1 + a] = 0.0;
        it.cs[1 + a] = cs[a];
        it.cn[1 + a] = cn[a];
    }
    it.out = out_dev;
    it.level = nwin > 0 ? nwin - 1 : 0;
    it.target = -1;
    return run_single_item(problem, dt, it, device);
}

int ridc_op_step_rows(const ridc_problem* problem, double dt, const double* eta_dev, int32_t nrows,
                      const double* const* rows_dev, const double* ca, double* out_dev,
                      int32_t device)
{
    if (nrows < 0 || nrows > kMaxNodes - 1) return fail(nullptr, RIDC_E_PROTOCOL, "window too large");
    if (nrows > 0 && (!rows_dev || !ca)) return fail(nullptr, RIDC_E_CONFIG, "NULL window");
    StepItem it;
    memset(&it, 0, sizeof it);
    it.nnodes = 1 + nrows;
    it.vec[0] = eta_dev;
    it.ca[0] = 1.0;
    it.cn[0] = dt;
    for (int a = 0; a < nrows; ++a) {
        it.vec[1 + a] = rows_dev[a];
        it.ca[1 + a] = ca[a];
    }
    it.out = out_dev;
    it.target = -1;
    return run_single_item(problem, dt, it, device);
}

// Phase trace of the last tick launch (RIDC_PHASE_TIMING=1 at create): CTA 0,
// thread 0, up to 8 items x 16 clock64 stamps.  Diagnostic only.
int ridc_debug_phase_trace(const ridc_ctx* c, long long* out, int n)
{
    if (!c || !out || n < 128) return fail(nullptr, RIDC_E_CONFIG, "need a 128-entry buffer");
    if (!c->d_dbg) return fail(nullptr, RIDC_E_CONFIG, "create with RIDC_PHASE_TIMING=1");
    CUDA_TRY(nullptr, cudaMemcpy(out, c->d_dbg, 128 * sizeof(long long), cudaMemcpyDeviceToHost));
    return RIDC_OK;
}

}  // extern "C"

// ================================================================ level pipeline

namespace {

typedef CUresult (*PfnWaitValue64)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
typedef CUresult (*PfnWriteValue64)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);

struct DriverOps {
    PfnWaitValue64 wait = nullptr;
    PfnWriteValue64 write = nullptr;
};

// Stream memory operations, resolved at run time (no link-time libcuda
// dependency, so the library also loads on hosts without a driver).
const DriverOps& driver_ops()
{
    static DriverOps ops = [] {
        DriverOps o;
        cudaDriverEntryPointQueryResult q;
        void* f = nullptr;
        if (cudaGetDriverEntryPoint("cuStreamWaitValue64", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            o.wait = reinterpret_cast<PfnWaitValue64>(f);
        f = nullptr;
        if (cudaGetDriverEntryPoint("cuStreamWriteValue64", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            o.write = reinterpret_cast<PfnWriteValue64>(f);
        return o;
    }();
    return ops;
}

constexpr uint32_t kBlobMagic = 0x52494443u;   // "RIDC"
constexpr size_t kFlagBytes = 256;             // wm (+0), rel (+8), then the inbox ring

struct PipeBlob {
    uint32_t magic;
    int32_t pid, device, level;
    cudaIpcMemHandle_t handle;
    uint64_t direct;       // mailbox base (valid inside the exporting process)
    int64_t inbox_cap;
    int64_t vs;
};

}  // namespace

struct ridc_pipe {
    int device = 0, level = 0, levels = 0, restarts = 0;
    long long steps = 0, per = 0, V = 0, Vs = 0;
    double t_start = 0, t_end = 0, dt = 0, watchdog = 30.0;
    DevProblem pb;
    SolveSetup ss;
    int nsm = 148;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    char* mailbox = nullptr;
    long long inbox_cap = 0;
    unsigned long long* wm = nullptr;    // my inbox watermark (written by level-1)
    unsigned long long* rel = nullptr;   // released-below counter (written by level+1)
    double* inbox = nullptr;             // slot 0 of my inbox ring
    double* own_base = nullptr;
    double* own = nullptr;               // my 2-slot state ring
    double* next_inbox = nullptr;        // peer: level+1's inbox ring
    long long next_cap = 0;
    unsigned long long* next_wm = nullptr;
    unsigned long long* prev_rel = nullptr;
    void* opened[2] = {nullptr, nullptr};
    double* d_weights = nullptr;
    double* d_tab = nullptr;
    PlanRow* d_plans = nullptr;
    unsigned long long* d_err = nullptr;
    std::vector<int> st, su;
    std::map<int, cudaGraphExec_t> graphs;
    long long launches = 0;
    std::string err;
};

namespace {

int pipe_fail(ridc_pipe* p, int code, const std::string& m)
{
    g_last_error = m;
    if (p) p->err = m;
    return code;
}

#define PIPE_TRY(p, expr)                                                                    \
    do {                                                                                     \
        cudaError_t _e = (expr);                                                             \
        if (_e != cudaSuccess)                                                               \
            return pipe_fail(p, RIDC_E_CUDA, std::string(#expr " failed: ") + cudaGetErrorString(_e)); \
    } while (0)

EngineParams pipe_params(ridc_pipe* p, long long g0)
{
    EngineParams ep;
    memset(&ep, 0, sizeof ep);
    ep.pb = p->pb;
    ep.sv = p->ss.sv;
    ep.V = p->V;
    ep.Vs = p->Vs;
    ep.dt = p->dt;
    ep.levels = p->levels;
    const int j = p->level;
    ep.ring[j] = p->own;
    ep.cap[j] = 2;
    ep.off[j] = g0;
    if (j > 0) {
        ep.ring[j - 1] = p->inbox;
        ep.cap[j - 1] = p->inbox_cap;
        ep.off[j - 1] = g0;
    }
    ep.weights = p->d_weights;
    for (int k = 0; k < kMaxLevels; ++k) {
        ep.steady_off[k] = p->st[k];
        ep.startup_off[k] = p->su[k];
    }
    ep.err = p->d_err;
    if (j < p->levels - 1 && p->next_inbox) {
        ep.mirror = p->next_inbox;
        ep.mirror_cap = p->next_cap;
        ep.mirror_off = g0;
    }
    return ep;
}

// Enqueue one interval: per step t, wait for the window (inbox watermark)
// and for ring space at the consumer (its release counter), run the level's
// tick kernel (which also stores into the consumer's inbox), publish the
// watermark to the consumer and the release to the producer.
int pipe_enqueue(ridc_pipe* p, int interval, long long* launches)
{
    const DriverOps& ops = driver_ops();
    const int j = p->level, top = p->levels - 1;
    const long long g0 = (long long)interval * p->per;
    const EngineParams ep = pipe_params(p, g0);
    const int items = p->pb.ny * p->ss.sv.nseg;
    CUstream cs = reinterpret_cast<CUstream>(p->stream);
    long long n = 0;
    for (long long t = 1; t <= p->per; ++t) {
        if (j > 0) {
            const long long need = g0 + (t < j ? j : t);
            if (ops.wait(cs, (CUdeviceptr)p->wm, (cuuint64_t)need, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
                return pipe_fail(p, RIDC_E_CUDA, "cuStreamWaitValue64 (watermark) failed");
        }
        if (j < top) {
            const long long need_rel = g0 + t - p->next_cap + 1;
            if (need_rel > 0 &&
                ops.wait(cs, (CUdeviceptr)p->rel, (cuuint64_t)need_rel, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
                return pipe_fail(p, RIDC_E_CUDA, "cuStreamWaitValue64 (release) failed");
        }
        TickParams tp;
        memset(&tp, 0, sizeof tp);
        tp.nact = 1;
        tp.level[0] = j;
        tp.target[0] = t;
        cudaError_t le = launch_tma(p->pb.kind, p->ss.tcfg, std::min(p->nsm, items), p->stream, ep, tp, items);
        if (le != cudaSuccess) return pipe_fail(p, RIDC_E_CUDA, std::string("tick launch: ") + cudaGetErrorString(le));
        ++n;
        if (j < top &&
            ops.write(cs, (CUdeviceptr)p->next_wm, (cuuint64_t)(g0 + t), CU_STREAM_WRITE_VALUE_DEFAULT) != CUDA_SUCCESS)
            return pipe_fail(p, RIDC_E_CUDA, "cuStreamWriteValue64 (watermark) failed");
        if (j > 0) {
            const long long below = g0 + std::max(0LL, t + 1 - j);
            if (ops.write(cs, (CUdeviceptr)p->prev_rel, (cuuint64_t)below, CU_STREAM_WRITE_VALUE_DEFAULT) != CUDA_SUCCESS)
                return pipe_fail(p, RIDC_E_CUDA, "cuStreamWriteValue64 (release) failed");
        }
    }
    *launches = n;
    return RIDC_OK;
}

}  // namespace

extern "C" {

int64_t ridc_pipe_handle_bytes(void) { return (int64_t)sizeof(PipeBlob); }

int ridc_pipe_create(const ridc_problem* problem, double t_start, double t_end, int32_t levels,
                     int64_t steps, int32_t restarts, const double* weights, int64_t nweights,
                     int32_t level, int32_t device, int32_t inbox_capacity, double watchdog_seconds,
                     ridc_pipe** out)
{
    if (!out) return pipe_fail(nullptr, RIDC_E_CONFIG, "out is NULL");
    *out = nullptr;
    int rc = validate_problem(problem);
    if (rc) return rc;
    if (levels < 1 || levels > kMaxLevels) return pipe_fail(nullptr, RIDC_E_CONFIG, "levels must be in 1..12");
    if (level < 0 || level >= levels) return pipe_fail(nullptr, RIDC_E_CONFIG, "level out of range");
    if (steps < 1 || restarts < 1 || steps % restarts)
        return pipe_fail(nullptr, RIDC_E_CONFIG, "steps must be a positive multiple of restarts");
    const long long per = steps / restarts;
    if (per < delay(levels) + 1) return pipe_fail(nullptr, RIDC_E_CONFIG, "restart interval shorter than the pipeline fill");
    if (!(t_start < t_end)) return pipe_fail(nullptr, RIDC_E_CONFIG, "need t_start < t_end");
    const DriverOps& ops = driver_ops();
    if (!ops.wait || !ops.write) return pipe_fail(nullptr, RIDC_E_CUDA, "driver stream memory operations unavailable");
    std::vector<int> st, su;
    long long wtotal = 0;
    weight_offsets(levels, st, su, wtotal);
    if (nweights < wtotal || (wtotal > 0 && !weights))
        return pipe_fail(nullptr, RIDC_E_DIMENSION, "weight table shorter than levels require");
    ridc_pipe* p = new ridc_pipe();
    p->device = device;
    p->level = level;
    p->levels = levels;
    p->restarts = restarts;
    p->steps = steps;
    p->per = per;
    p->t_start = t_start;
    p->t_end = t_end;
    p->dt = (t_end - t_start) / (double)steps;
    p->watchdog = watchdog_seconds > 0 ? watchdog_seconds : 30.0;
    p->pb = make_problem(problem);
    p->V = (long long)problem->nx * problem->ny;
    p->Vs = ((p->V + 1) & ~1LL) + 4;
    p->st = st;
    p->su = su;
    p->inbox_cap = inbox_capacity > 0 ? inbox_capacity : 2LL * level + 5;
    auto bail = [&](int code) {
        std::string m = p->err.empty() ? g_last_error : p->err;
        ridc_pipe_destroy(p);
        g_last_error = m;
        return code;
    };
#define P_TRY(expr)                                                                          \
    do {                                                                                     \
        cudaError_t _e = (expr);                                                             \
        if (_e != cudaSuccess) {                                                             \
            p->err = std::string(#expr " failed: ") + cudaGetErrorString(_e);               \
            return bail(RIDC_E_CUDA);                                                        \
        }                                                                                    \
    } while (0)
    P_TRY(cudaSetDevice(device));
    if (cudaDeviceGetAttribute(&p->nsm, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) p->nsm = 148;
    // tiling depends only on the problem and dt (not on levels or devices), so a
    // level computes bitwise the same states here as in the single-device engine
    if ((rc = make_solve(p->pb, p->dt, tma_cap(p->pb.kind), p->pb.ny, p->nsm, p->ss)) != RIDC_OK) {
        p->err = p->ss.err;
        return bail(rc);
    }
    P_TRY(cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking));
    P_TRY(cudaEventCreate(&p->ev0));
    P_TRY(cudaEventCreate(&p->ev1));
    P_TRY(cudaMalloc(&p->d_weights, std::max<long long>(wtotal, 1) * sizeof(double)));
    if (wtotal > 0) P_TRY(cudaMemcpy(p->d_weights, weights, wtotal * sizeof(double), cudaMemcpyHostToDevice));
    if (!p->ss.tab.empty()) {
        P_TRY(cudaMalloc(&p->d_tab, p->ss.tab.size() * sizeof(double)));
        P_TRY(cudaMemcpy(p->d_tab, p->ss.tab.data(), p->ss.tab.size() * sizeof(double), cudaMemcpyHostToDevice));
        p->ss.sv.tab_m = p->d_tab;
        p->ss.sv.tab_g = p->d_tab + p->ss.sv.ntab;
    }
    P_TRY(cudaMalloc(&p->d_plans, p->ss.plans.size() * sizeof(PlanRow)));
    P_TRY(cudaMemcpy(p->d_plans, p->ss.plans.data(), p->ss.plans.size() * sizeof(PlanRow), cudaMemcpyHostToDevice));
    p->ss.sv.plans = p->d_plans;
    P_TRY(cudaMalloc(&p->d_err, sizeof(unsigned long long)));
    // mailbox: flags, then the inbox ring (2 guard doubles + cap slots of Vs)
    const size_t ring_bytes = ((size_t)p->inbox_cap * p->Vs + 4) * sizeof(double);
    P_TRY(cudaMalloc(&p->mailbox, kFlagBytes + ring_bytes));
    P_TRY(cudaMemset(p->mailbox, 0, kFlagBytes));
    p->wm = reinterpret_cast<unsigned long long*>(p->mailbox);
    p->rel = reinterpret_cast<unsigned long long*>(p->mailbox + 8);
    p->inbox = reinterpret_cast<double*>(p->mailbox + kFlagBytes) + 2;
    P_TRY(cudaMalloc(&p->own_base, ((size_t)2 * p->Vs + 4) * sizeof(double)));
    p->own = p->own_base + 2;
#undef P_TRY
    *out = p;
    return RIDC_OK;
}

int ridc_pipe_export(ridc_pipe* p, void* blob)
{
    if (!p || !blob) return pipe_fail(p, RIDC_E_CONFIG, "NULL argument");
    PipeBlob b;
    memset(&b, 0, sizeof b);
    b.magic = kBlobMagic;
    b.pid = (int32_t)getpid();
    b.device = p->device;
    b.level = p->level;
    b.direct = (uint64_t)(uintptr_t)p->mailbox;
    b.inbox_cap = p->inbox_cap;
    b.vs = p->Vs;
    PIPE_TRY(p, cudaSetDevice(p->device));
    PIPE_TRY(p, cudaIpcGetMemHandle(&b.handle, p->mailbox));
    memcpy(blob, &b, sizeof b);
    return RIDC_OK;
}

static int open_blob(ridc_pipe* p, const void* blob, int want_level, char** base, int slot, long long* cap)
{
    PipeBlob b;
    memcpy(&b, blob, sizeof b);
    if (b.magic != kBlobMagic || b.level != want_level || b.vs != p->Vs)
        return pipe_fail(p, RIDC_E_PROTOCOL, "pipeline handle from an incompatible rank");
    if (b.pid == (int32_t)getpid()) {
        *base = reinterpret_cast<char*>((uintptr_t)b.direct);
        if (b.device != p->device) {
            cudaError_t e = cudaDeviceEnablePeerAccess(b.device, 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
                return pipe_fail(p, RIDC_E_CUDA, std::string("peer access: ") + cudaGetErrorString(e));
            cudaGetLastError();
        }
    } else {
        void* ptr = nullptr;
        PIPE_TRY(p, cudaIpcOpenMemHandle(&ptr, b.handle, cudaIpcMemLazyEnablePeerAccess));
        p->opened[slot] = ptr;
        *base = reinterpret_cast<char*>(ptr);
    }
    *cap = b.inbox_cap;
    return RIDC_OK;
}

int ridc_pipe_connect(ridc_pipe* p, const void* prev_blob, const void* next_blob)
{
    if (!p) return pipe_fail(nullptr, RIDC_E_CONFIG, "NULL pipe");
    PIPE_TRY(p, cudaSetDevice(p->device));
    const int j = p->level, top = p->levels - 1;
    if ((j > 0) != (prev_blob != nullptr) || (j < top) != (next_blob != nullptr))
        return pipe_fail(p, RIDC_E_CONFIG, "level needs exactly its existing neighbours");
    int rc;
    long long cap = 0;
    char* base = nullptr;
    if (prev_blob) {
        if ((rc = open_blob(p, prev_blob, j - 1, &base, 0, &cap)) != RIDC_OK) return rc;
        p->prev_rel = reinterpret_cast<unsigned long long*>(base + 8);
    }
    if (next_blob) {
        if ((rc = open_blob(p, next_blob, j + 1, &base, 1, &cap)) != RIDC_OK) return rc;
        p->next_wm = reinterpret_cast<unsigned long long*>(base);
        p->next_inbox = reinterpret_cast<double*>(base + kFlagBytes) + 2;
        p->next_cap = cap;
    }
    return RIDC_OK;
}

int ridc_pipe_run_interval(ridc_pipe* p, int32_t interval, const double* state0_dev, double* final_dev,
                           double* wall_seconds)
{
    if (!p || !state0_dev || !final_dev) return pipe_fail(p, RIDC_E_CONFIG, "NULL argument");
    if (interval < 0 || interval >= p->restarts) return pipe_fail(p, RIDC_E_CONFIG, "interval out of range");
    const int j = p->level, top = p->levels - 1;
    if ((j > 0 && !p->prev_rel) || (j < top && !p->next_inbox))
        return pipe_fail(p, RIDC_E_CONFIG, "pipeline rank not connected");
    PIPE_TRY(p, cudaSetDevice(p->device));
    const long long g0 = (long long)interval * p->per;
    const size_t vb = (size_t)p->V * sizeof(double);
    // seed: step g0 of my own ring and of my inbox is the interval's state0
    EngineParams ep = pipe_params(p, g0);
    PIPE_TRY(p, cudaMemcpyAsync(ep.ring[j] + ((ep.off[j]) % 2) * p->Vs, state0_dev, vb,
                                cudaMemcpyDeviceToDevice, p->stream));
    if (j > 0)
        PIPE_TRY(p, cudaMemcpyAsync(p->inbox + (g0 % p->inbox_cap) * p->Vs, state0_dev, vb,
                                    cudaMemcpyDeviceToDevice, p->stream));
    PIPE_TRY(p, cudaMemsetAsync(p->d_err, 0xff, sizeof(unsigned long long), p->stream));
    PIPE_TRY(p, cudaEventRecord(p->ev0, p->stream));
    // the interval's ops: captured into a graph on first use (memops included)
    auto it = p->graphs.find(interval);
    long long launches = 0;
    if (it == p->graphs.end()) {
        cudaGraph_t graph = nullptr;
        cudaGraphExec_t exec = nullptr;
        bool captured = false;
        if (cudaStreamBeginCapture(p->stream, cudaStreamCaptureModeThreadLocal) == cudaSuccess) {
            int rc = pipe_enqueue(p, interval, &launches);
            cudaError_t ce = cudaStreamEndCapture(p->stream, &graph);
            if (rc == RIDC_OK && ce == cudaSuccess && cudaGraphInstantiate(&exec, graph, 0) == cudaSuccess)
                captured = true;
            if (graph) cudaGraphDestroy(graph);
        }
        cudaGetLastError();
        if (captured) {
            p->graphs[interval] = exec;
            PIPE_TRY(p, cudaGraphLaunch(exec, p->stream));
        } else {
            int rc = pipe_enqueue(p, interval, &launches);   // direct enqueue fallback
            if (rc) return rc;
        }
    } else {
        PIPE_TRY(p, cudaGraphLaunch(it->second, p->stream));
        launches = p->per;
    }
    p->launches = launches;
    PIPE_TRY(p, cudaMemcpyAsync(final_dev, ep.ring[j] + ((ep.off[j] + p->per) % 2) * p->Vs, vb,
                                cudaMemcpyDeviceToDevice, p->stream));
    PIPE_TRY(p, cudaEventRecord(p->ev1, p->stream));
    // watchdog (engine.py:432-439): neighbours that never publish turn into an error
    const auto t0 = std::chrono::steady_clock::now();
    for (;;) {
        cudaError_t q = cudaEventQuery(p->ev1);
        if (q == cudaSuccess) break;
        if (q != cudaErrorNotReady) return pipe_fail(p, RIDC_E_CUDA, cudaGetErrorString(q));
        const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (el > p->watchdog) {
            char buf[160];
            snprintf(buf, sizeof buf, "pipeline made no progress within %gs; waiting levels: %d@interval%d",
                     p->watchdog, j, interval);
            return pipe_fail(p, RIDC_E_PROTOCOL, buf);
        }
        std::this_thread::sleep_for(std::chrono::microseconds(200));
    }
    if (wall_seconds) {
        float ms = 0.f;
        PIPE_TRY(p, cudaEventElapsedTime(&ms, p->ev0, p->ev1));
        *wall_seconds = ms * 1e-3;
    }
    unsigned long long w = 0;
    PIPE_TRY(p, cudaMemcpy(&w, p->d_err, sizeof w, cudaMemcpyDeviceToHost));
    if (w != ULLONG_MAX) {
        char buf[160];
        snprintf(buf, sizeof buf, "level %d produced non-finite entries at step %lld", (int)(w & 0xff),
                 (long long)(w >> 8));
        return pipe_fail(p, RIDC_E_NONFINITE, buf);
    }
    return RIDC_OK;
}

int ridc_pipe_info(const ridc_pipe* p, ridc_info* info)
{
    if (!p || !info) return pipe_fail(nullptr, RIDC_E_CONFIG, "NULL argument");
    memset(info, 0, sizeof *info);
    info->levels = p->levels;
    info->restarts = p->restarts;
    info->steps = p->steps;
    info->ticks_per_interval = p->per;
    info->kernel_launches = p->per;
    info->tile = p->ss.sv.tile;
    info->halo = p->ss.sv.halo;
    info->items_per_level = p->pb.ny * p->ss.sv.nseg;
    info->threads = p->ss.tcfg.nt;
    info->ring_vectors = 2 + (p->level > 0 ? p->inbox_cap : 0);
    info->lambda = p->ss.sv.lam;
    info->r = p->ss.r;
    return RIDC_OK;
}

int ridc_pipe_destroy(ridc_pipe* p)
{
    if (!p) return RIDC_OK;
    cudaSetDevice(p->device);
    if (p->stream) cudaStreamSynchronize(p->stream);
    for (auto& kv : p->graphs) cudaGraphExecDestroy(kv.second);
    for (void* o : p->opened)
        if (o) cudaIpcCloseMemHandle(o);
    if (p->mailbox) cudaFree(p->mailbox);
    if (p->own_base) cudaFree(p->own_base);
    if (p->d_weights) cudaFree(p->d_weights);
    if (p->d_tab) cudaFree(p->d_tab);
    if (p->d_plans) cudaFree(p->d_plans);
    if (p->d_err) cudaFree(p->d_err);
    if (p->ev0) cudaEventDestroy(p->ev0);
    if (p->ev1) cudaEventDestroy(p->ev1);
    if (p->stream) cudaStreamDestroy(p->stream);
    delete p;
    return RIDC_OK;
}

const char* ridc_pipe_last_error(const ridc_pipe* p)
{
    if (p && !p->err.empty()) return p->err.c_str();
    return g_last_error.c_str();
}

}  // extern "C"
