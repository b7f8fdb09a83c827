// ridc_kernels.cuh -- kernel templates and launch-configuration tables shared by
// the host runtime (ridc_engine.cu) and the per-kind instantiation units
// (ridc_inst.cu, compiled once per problem kind and kernel family so that
// nvcc runs them in parallel).  The launch entry points declared at the end
// are defined in ridc_dispatch.cuh and explicitly instantiated per kind.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include "ridc_device.cuh"
#include "ridc_tma.cuh"
#include "ridc_chunk.cuh"
#include "ridc_resident.cuh"
#include "ridc_levels.cuh"
#include "ridc_febe_carry.cuh"
#include "ridc_sweep.cuh"
#include "ridc_sweep2d.cuh"

namespace ridc {

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
    ChunkLayout lay;           // padded row layout (ghost columns)
    int row0;                  // first computed row (1 for a row shard with ghost rows 0 and ny-1)
    const ChunkGeo* cgeo;      // per-segment item geometry
};

struct TickParams {
    int nact;
    int level[kMaxLevels];
    long long target[kMaxLevels];
    DevSolve sv;             // factors of this launch's shifted solve (RIDC: ep.sv; ARK: per stage)
    const StepItem* pre;     // precomputed item descriptors (ARK stages), or null: build_item
};

__device__ __forceinline__ long long slot_index(const EngineParams& ep, int lev, long long s, long long off = -1)
{
    RIDC_CHECK(lev >= 0 && lev < ep.levels && ep.cap[lev] > 0 && s >= 0);
    return ((off < 0 ? ep.off[lev] : off) + s) % ep.cap[lev];
}

__device__ __forceinline__ double* ring_slot(const EngineParams& ep, int lev, long long s,
                                             long long off = -1)
{
    return ep.ring[lev] + slot_index(ep, lev, s, off) * ep.Vs;
}

// Window assembly for (level j, target t): _window_span / _orient /
// _WeightTables.for_step (engine.py:124-157) with the lag terms of
// _correct_core (engine.py:179-181) folded into the node coefficients.
__device__ inline void build_item(const EngineParams& ep, int j, long long t, StepItem& it, long long off = -1)
{
    it.level = j;
    it.target = t;
    it.vec[0] = ring_slot(ep, j, t - 1, off);
    it.vlev[0] = j;
    it.vslot[0] = slot_index(ep, j, t - 1, off);
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
            it.vlev[nn] = j - 1;
            it.vslot[nn] = slot_index(ep, j - 1, s, off);
            it.ca[nn] = 0.0;
            it.cs[nn] = w[a] - (a == i_new ? ep.dt : 0.0);
            it.cn[nn] = w[a] - (a == i_old ? ep.dt : 0.0);
            ++nn;
        }
    }
    it.nnodes = nn;
    it.out = ring_slot(ep, j, t, off);
    it.out2 = ep.mirror ? ep.mirror + ((ep.mirror_off + t) % ep.mirror_cap) * ep.Vs : nullptr;
    // whole-line items store their row with one bulk tensor store (the level's ring map)
    it.omap1 = ep.mirror ? 0 : j + 1;
    it.opad = 0;
    it.oslot = slot_index(ep, j, t, off);
}

// Item i of a tick -> (level slot, tile): tile = i % tiles, slot = (i / tiles
// + tile) % nact.  A bijection (each tile meets every slot once), and a CTA
// taking items b, b + grid, ... gets a mix of levels: with the plain
// slot = i % nact a CTA would run the same level for every one of its items
// whenever the grid is a multiple of nact, and the top level's CTAs ((j+2)
// nodes per item) would set the tick time.
__device__ __forceinline__ void item_of(int i, int tiles, int nact, int& slot, int& tile)
{
    tile = i % tiles;
    slot = (i / tiles + tile) % nact;
}

// The production tick kernel: persistent CTAs of NT compute threads; thread
// 0 doubles as the TMA producer (ridc_chunk.cuh).  Items of the tick are
// dealt round-robin over the CTAs (item_of).  MODE is
// the solve mode all segments share (0 truncated, 1 cyclic whole line, 2
// Dirichlet whole line), or -1 to dispatch per segment -- one mode per
// kernel keeps the hot loop small in the instruction cache.
template <int KIND, int NT, int ROWS, int NSTAGE, int MODE, int KC>
__global__ void __launch_bounds__(NT, ROWS == 3 && NSTAGE == 1 ? 2 : 1)
    k_tick_chunk(EngineParams ep, TickParams tp, int ipl, const __grid_constant__ TmapSet tm)
{
    using L = ChunkSmem<NT, ROWS, NSTAGE, KC>;
    extern __shared__ __align__(1024) char smraw[];
    char* stage = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
    double* edge = reinterpret_cast<double*>(stage + L::OFF_EDGE);
    uint64_t* full = reinterpret_cast<uint64_t*>(stage + L::OFF_BAR);
    uint64_t* empty = full + NSTAGE;
    // one descriptor per active level (shared by all its tiles), after the stages
    StepItem* items = reinterpret_cast<StepItem*>(stage + L::BYTES);
    __shared__ Aff swarp[2 * (NT / 32) + 1];
    const int total = tp.nact * ipl;
    const DevSolve& sv = tp.sv;
    // phase trace (RIDC_PHASE_TIMING): CTA 0 / thread 0 globaltimer at entry, after the
    // grid dependency wait and at exit, row = target & 7 of the first active level
    long long* tdbg = (sv.dbg && blockIdx.x == 0 && threadIdx.x == 0) ? sv.dbg + (tp.target[0] & 7) * 16 : nullptr;
    auto gtime = [] {
        unsigned long long g;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
        return (long long)g;
    };
    if (tdbg) tdbg[10] = gtime();
    long long* cdbg = (sv.dbg && threadIdx.x == 0 && tp.target[0] == 100 && blockIdx.x < 1024)
                          ? sv.dbg + 128 + 4 * blockIdx.x : nullptr;
    if (cdbg) cdbg[0] = gtime();
    const int nseg = sv.nseg, ny = ep.pb.ny;
    // programmatic dependent launch: let the next tick's grid get scheduled now;
    // its CTAs run this prologue as SMs free up and wait (below) before reading
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    static_assert(sizeof(StepItem) % 8 == 0, "StepItem is copied as 8-byte words");
    if (tp.pre) {   // precomputed descriptors (ARK stages); the step number comes per launch
        for (int k = threadIdx.x; k < tp.nact * (int)(sizeof(StepItem) / 8); k += blockDim.x)
            reinterpret_cast<long long*>(items)[k] = reinterpret_cast<const long long*>(tp.pre)[k];
        __syncthreads();
        if (threadIdx.x < tp.nact) items[threadIdx.x].target = tp.target[threadIdx.x];
    } else if (threadIdx.x < tp.nact) {
        build_item(ep, tp.level[threadIdx.x], tp.target[threadIdx.x], items[threadIdx.x]);
    }
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
        int slot, tile;
        item_of(pc.i, ipl, tp.nact, slot, tile);
        const int row = ep.row0 + tile / nseg, seg = tile - (tile / nseg) * nseg;
        const StepItem& it = items[slot];
        issue_chunk_node<NT, ROWS, NSTAGE, KC>(tm, it.vlev[pc.a], it.vslot[pc.a], row, ny, ep.lay.gpr,
                                           ep.lay.gdata, ep.cgeo[seg], stage + (size_t)s * L::STAGE,
                                           &full[s]);
        if (++pc.a == it.nnodes) { pc.a = 0; pc.i += gridDim.x; }
        ++pc.n;
    };
    // every global read of ring data and every global write happens after the
    // previous tick's grid completed: thread 0 waits before its first load,
    // everyone else reads / writes only after that load's barrier
    if (threadIdx.x == 0) {
        asm volatile("griddepcontrol.wait;" ::: "memory");
        if (tdbg) tdbg[11] = gtime();
        if (cdbg) cdbg[1] = gtime();
        for (int k = 0; k < NSTAGE && pc.i < total; ++k) issue_next(k);
    }
    // after load n was released from stage s: wait for every warp, then load n + NSTAGE into s
    auto refill = [&](long long n, int s) {
        if (pc.i >= total) return;
        mbar_wait(&empty[s], (uint32_t)((n / NSTAGE) & 1));
        issue_next(s);
    };
    long long n = 0;
    int ino = 0;
    const FastLane fl = fast_lane<KC>(sv);
    for (int i = blockIdx.x; i < total; i += gridDim.x, ++ino) {
        int slot, tile;
        item_of(i, ipl, tp.nact, slot, tile);
        const int row = ep.row0 + tile / nseg, seg = tile - (tile / nseg) * nseg;
        const ChunkGeo cg = ep.cgeo[seg];
        switch (MODE >= 0 ? MODE : cg.mode) {
        case 0:
            chunk_item<KIND, NT, ROWS, NSTAGE, 0, KC>(ep.pb, sv, ep.lay, tm, items[slot], cg, row, stage, edge,
                                                  full, empty, n, refill, swarp, ep.err, ino, fl);
            break;
        case 1:
            chunk_item<KIND, NT, ROWS, NSTAGE, 1, KC>(ep.pb, sv, ep.lay, tm, items[slot], cg, row, stage, edge,
                                                  full, empty, n, refill, swarp, ep.err, ino, fl);
            break;
        default:
            chunk_item<KIND, NT, ROWS, NSTAGE, 2, KC>(ep.pb, sv, ep.lay, tm, items[slot], cg, row, stage, edge,
                                                  full, empty, n, refill, swarp, ep.err, ino, fl);
        }
        // 1-D: no barrier here; the next item writes `edge` / the scan scratch
        // only after this item's store barrier, which follows its last reads of
        // both. 2-D keeps it: without it the C3 x-line tick measured 115 -> 135 us
        // (the warps drift apart and the two co-resident CTAs' loads collide).
        if constexpr (ROWS == 3) csync<NT>();
    }
    // the bulk tensor stores of the last items complete before the grid does
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    if (tdbg) tdbg[12] = gtime();
    if (cdbg) cdbg[2] = gtime();
}

template <int KIND, int NT, int KMAX>
__global__ void __launch_bounds__(NT) k_item(DevProblem pb, DevSolve sv, StepItem it,
                                             unsigned long long* err)
{
    extern __shared__ double sbuf[];
    __shared__ Aff swarp[2 * (NT / 32) + 1];
    process_item<KIND, NT, KMAX>(pb, sv, it, blockIdx.x, sbuf, swarp, err);
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

inline LaunchCfg pick_cfg(int Q)
{
    LaunchCfg c;
    if (Q <= 128 * 8) { c.id = 0; c.nt = 128; c.kmax = 8; }
    else if (Q <= 256 * 8) { c.id = 1; c.nt = 256; c.kmax = 8; }
    else { c.id = 2; c.nt = 512; c.kmax = 8; }
    const int cap = c.nt * c.kmax;
    c.smem = (size_t)(cap + cap / 16 + 1) * sizeof(double);
    return c;
}

// ---- chunk tick kernel configurations (NT threads x 16 points, ROWS staged
// rows per node, NSTAGE stages); many warps per SM hide the fp64 / shared
// memory latencies of the scans.
struct ChunkCfg {
    int id;
    int nt, rows, nstage;
    int kc;     // points per thread (16: one group per thread; 8: two threads per group)
    size_t smem;
    int mode;   // common segment mode (k_tick_chunk MODE), -1 mixed
};

#define RIDC_CHUNK_CONFIGS(X) \
    X(0, 64, 1, 4, 16)        \
    X(1, 128, 1, 4, 16)       \
    X(2, 256, 1, 4, 16)       \
    X(3, 512, 1, 3, 16)       \
    X(4, 64, 3, 3, 16)        \
    X(5, 128, 3, 3, 16)       \
    X(6, 512, 3, 2, 8)        \
    X(7, 256, 3, 1, 16)

template <int NT, int ROWS, int NSTAGE, int KC>
ChunkCfg chunk_cfg_make(int id)
{
    ChunkCfg c;
    c.id = id;
    c.nt = NT;
    c.rows = ROWS;
    c.nstage = NSTAGE;
    c.kc = KC;
    c.smem = ChunkSmem<NT, ROWS, NSTAGE, KC>::BYTES + 1024;   // + 1 KiB for the 1024-B alignment
    c.mode = -1;
    return c;
}

// 128-byte groups (16 points) one item of this configuration stages per row
inline int chunk_groups(const ChunkCfg& c) { return c.nt * c.kc / 16; }

// the configuration with this id, as listed in RIDC_CHUNK_CONFIGS
inline ChunkCfg chunk_cfg_of_id(int id)
{
#define RIDC_CFG_OF(ID, NT, ROWS, NSTAGE, KC) \
    if (id == ID) return chunk_cfg_make<NT, ROWS, NSTAGE, KC>(ID);
    RIDC_CHUNK_CONFIGS(RIDC_CFG_OF)
#undef RIDC_CFG_OF
    return chunk_cfg_make<512, 1, 3, 16>(3);
}

// CTAs of the tick kernel per SM.  1-D: one (4096-point items at two CTAs per
// SM measured 1.7-2x slower than 8192-point items at one: twice the halo
// overhead).  2-D single-stage config: two when both fit the shared memory,
// so one CTA's x-line solve overlaps the other's row loads.
inline int chunk_ctas_per_sm(const ChunkCfg& c, int nact = kMaxLevels)
{
    if (c.rows == 3 && c.nstage == 1 && 2 * (c.smem + (size_t)nact * sizeof(StepItem) + 1024) <= 228 * 1024)
        return 2;
    return 1;
}

// 2-D lines of 4096: the single-stage 256 x 16 config (id 7, same 256 groups
// per item as id 6, so the same tiling and tensor maps) when two CTAs of it
// fit an SM with `max_nact` item descriptors: one CTA's x-line solve then
// overlaps the other's row loads (C3 FEBE 150 -> 119 us/tick, C4 703 -> 446).
// With many levels per tick the descriptors crowd it to one CTA per SM and
// the double-buffered 512 x 8 config (id 6) is faster.
inline void prefer_two_per_sm(ChunkCfg& c, int max_nact)
{
    if (c.id != 6) return;
    ChunkCfg t = chunk_cfg_of_id(7);
    t.mode = c.mode;
    if (chunk_ctas_per_sm(t, max_nact) == 2) c = t;
}

// smallest config whose NT*16 points cover `points` (the item's staged range)
inline ChunkCfg pick_chunk(int kind, int points)
{
    const bool two_d = kind == ADV_DIFF_2D || kind == RD_2D;
    if (two_d) {
        if (points <= 64 * 16) return chunk_cfg_of_id(4);
        if (points <= 128 * 16) return chunk_cfg_of_id(5);
        return chunk_cfg_of_id(6);   // 512 threads x 8 points: 16 warps per 4096-point line
    }
    if (points <= 64 * 16) return chunk_cfg_of_id(0);
    if (points <= 128 * 16) return chunk_cfg_of_id(1);
    if (points <= 256 * 16) return chunk_cfg_of_id(2);
    return chunk_cfg_of_id(3);
}

inline int chunk_points_max(int kind)
{
    if (kind == ADV_DIFF_2D || kind == RD_2D) return 256 * 16;
    return 512 * 16;
}

// ---- resident level march (ridc_levels.cuh): every lane a group of nseg CTAs
constexpr int kResStages = 2;

}  // namespace ridc

#include "ridc_sweep2d_levels.cuh"
#include "ridc_sweep_levels.cuh"
#include "ridc_carry_levels.cuh"
#include "ridc_carry_res2.cuh"
#include "ridc_carry_res2w.cuh"

namespace ridc {

// ---- launch entry points, one instantiation per problem kind (ridc_inst.cu)
template <int KIND>
cudaError_t launch_chunk_k(const ChunkCfg& c, int grid, cudaStream_t st, const EngineParams& ep,
                           const TickParams& tp, int ipl, const TmapSet& tm);
template <int KIND>
cudaError_t launch_item_k(const LaunchCfg& c, int items, cudaStream_t st, const DevProblem& pb,
                          const DevSolve& sv, const StepItem& it, unsigned long long* err);
template <int KIND>
cudaError_t resident_k(int nt, int mode, bool launch, int grid, cudaStream_t st, const ResidentParams& rp,
                       int* per_sm);
template <int KIND>
cudaError_t febe_carry_k(bool launch, int grid, int nt, cudaStream_t st, const CarryParams& cp, int* per_sm);
template <int KIND>
cudaError_t febe_wcarry_k(bool launch, int k, int grid, int nt, cudaStream_t st, const CarryParams& cp, int* per_sm);
template <int KIND>
cudaError_t sweep_k(int nt, int grid, cudaStream_t st, const SweepParams& sp, const TmapSet& tm, long long off,
                    long long target);
template <int KIND>
cudaError_t sweep2d_k(int nt, int grid, cudaStream_t st, const Sweep2DParams& sp, const TmapSet& tm, long long off,
                      long long target);
template <int KIND>
cudaError_t sweep_levels_k(int grid, cudaStream_t st, const EngineParams& ep, const TickParams& tp,
                           const SweepParams& sp, const TmapSet& tm);
template <int KIND>
cudaError_t carry_res2_k(bool launch, int grid, int nt, cudaStream_t st, const CarryRes2Params& cp, int* per_sm);
template <int KIND>
cudaError_t carry_res2w_k(bool launch, int grid, cudaStream_t st, const CarryRes2Params& cp, int* per_sm);
template <int KIND>
cudaError_t carry_levels_k(int grid, int wpc, int k, cudaStream_t st, const EngineParams& ep, const TickParams& tp,
                           const CarryLevParams& cp, const TmapSet& tm, unsigned tick);
template <int KIND>
cudaError_t sweep2d_levels_k(int nt, int grid, cudaStream_t st, const EngineParams& ep, const TickParams& tp,
                             const SweepLevParams& sp, const TmapSet& tm);
template <int KIND, bool SYS>
cudaError_t levels_k(int nt, int mode, bool launch, int grid, cudaStream_t st, const LevelsParams& lp,
                     const TmapSet& tm, int* per_sm, bool dense);

}  // namespace ridc
