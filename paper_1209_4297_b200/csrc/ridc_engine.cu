// ridc_engine.cu -- kernels + host runtime behind include/ridc_b200.h (sm_100a).
//
// Single-device engine: every tick of the lagged pipeline is ONE kernel launch
// covering all active levels (levels are independent within a tick:
// level j at tick k computes step k - j(j+1)/2, reading only data published
// in earlier ticks, engine.py:363-371), and the whole run (all restart
// intervals, all ticks) is captured once into a CUDA graph at create time
// (the analogue of _prepare's pre-factorisation, engine.py:465-473).
//
// Single level (RIDC order 1, FEBE) on 1-D lines whose segments fit one CTA
// each: one cooperative launch marches every step with the state held in
// registers (ridc_resident.cuh); only segment edges go through L2.
//
// Several levels on 1-D lines whose levels x segments fit the SMs: one
// cooperative launch per restart interval, every level a CTA group, the
// lagged pipeline between them driven by per-segment flags
// (ridc_levels.cuh); the one-level-per-GPU pipeline ranks (ridc_pipe_*) run
// the same kernel with one level each, flags and stores over NVLink.
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

#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3: ranges cost nothing unless a tool attaches

#include "../../include/ridc_b200.h"
#include "ridc_kernels.cuh"
#include "ridc_sweep_warp.cuh"
#include "ridc_carry_levels.cuh"

using namespace ridc;

namespace {

thread_local std::string g_last_error;

// NVTX range over a host entry point (the phases a profiler timeline shows:
// create / graph capture / march / pipeline interval / shards / ARK)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

int env_int(const char* name, int def)
{
    const char* e = getenv(name);
    const int v = e ? atoi(e) : def;
    return v > 0 ? v : def;
}

// top-ring slots while the trajectory is streamed to host memory
constexpr long long kTrajDepth = 8;

// phase-trace buffer (RIDC_PHASE_TIMING): 8 rows x 16 stamps of CTA 0, then per
// CTA (entry, wait-done, exit) globaltimer of tick target 100
constexpr int kDbgWords = 128 + 4 * 1024;

// state (plain [ny][nx]) -> slot 0 of every level ring, padded layout with ghosts
// (engine.py:357-360: step 0 = initial data on every level)
__global__ void k_seed_chunk(const double* __restrict__ src, EngineParams ep, long long off)
{
    const int nx = ep.pb.nx, ny = ep.pb.ny, GW = ep.lay.GW, P = ep.lay.P;
    const long long tot = (long long)ny * P;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < tot;
         i += (long long)gridDim.x * blockDim.x) {
        const int r = (int)(i / P), c = (int)(i - (long long)r * P) - GW;
        double v = 0.0;
        if (c >= 0 && c < nx) v = src[(size_t)r * nx + c];
        else if (ep.pb.periodic && c >= -GW && c < nx + GW) v = src[(size_t)r * nx + ((c + nx) % nx)];
        for (int j = 0; j < ep.levels; ++j)
            if (ep.ring[j]) ring_slot(ep, j, 0, off)[i] = v;
    }
}

__global__ void k_bump_epoch(unsigned* e) { *e += 1u; }

// Wait on the device until *flag >= want: the consumer side of a watermark
// written by a producer on ANOTHER device where the stream wait cannot flush
// remote writes (CU_DEVICE_ATTRIBUTE_CAN_FLUSH_REMOTE_WRITES = 0).  The
// system-scope acquire orders the producer's earlier peer stores (made
// visible by the fence before its stream write of the watermark) before
// every later kernel of this stream.  A wait beyond spin_limit cycles sets
// *abort and returns (the host reports PipelineProtocolError).
__global__ void k_wait_flag(const unsigned long long* flag, unsigned long long want, unsigned* abort,
                            long long spin_limit)
{
    if (threadIdx.x != 0) return;
    const long long t0 = clock64();
    unsigned long long v;
    for (;;) {
        asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flag) : "memory");
        if (v >= want) return;
        if (clock64() - t0 > spin_limit || *(volatile unsigned*)abort) {
            atomicExch(abort, 1u);
            return;
        }
        __nanosleep(200);
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

cudaError_t launch_chunk(int kind, const ChunkCfg& c, int grid, cudaStream_t st, const EngineParams& ep,
                         const TickParams& tp, int ipl, const TmapSet& tm)
{
    switch (kind) {
    case ADV_DIFF_1D: return launch_chunk_k<ADV_DIFF_1D>(c, grid, st, ep, tp, ipl, tm);
    case BURGERS_1D: return launch_chunk_k<BURGERS_1D>(c, grid, st, ep, tp, ipl, tm);
    case RD_1D: return launch_chunk_k<RD_1D>(c, grid, st, ep, tp, ipl, tm);
    case ADV_DIFF_2D: return launch_chunk_k<ADV_DIFF_2D>(c, grid, st, ep, tp, ipl, tm);
    case RD_2D: return launch_chunk_k<RD_2D>(c, grid, st, ep, tp, ipl, tm);
    }
    return cudaErrorInvalidValue;
}

// launch == false: occupancy query into *per_sm (blocks per SM)
cudaError_t resident_dispatch(int kind, int nt, int mode, bool launch, int grid, cudaStream_t st,
                              const ResidentParams& rp, int* per_sm)
{
    switch (kind) {
    case ADV_DIFF_1D: return resident_k<ADV_DIFF_1D>(nt, mode, launch, grid, st, rp, per_sm);
    case BURGERS_1D: return resident_k<BURGERS_1D>(nt, mode, launch, grid, st, rp, per_sm);
    case RD_1D: return resident_k<RD_1D>(nt, mode, launch, grid, st, rp, per_sm);
    default: return cudaErrorInvalidValue;
    }
}

// launch == false: occupancy query into *per_sm.  sys: flags at system scope
// (levels on different GPUs), else GPU scope (every level on this device).
// dense: the two-CTAs-per-SM variant of the 4096-point items (single GPU only)
cudaError_t levels_dispatch(int kind, int nt, int mode, bool launch, int grid, cudaStream_t st,
                            const LevelsParams& lp, const TmapSet& tm, int* per_sm, bool sys, bool dense = false)
{
#define RIDC_LEV_KIND(K)                                                                   \
    case K:                                                                                \
        return sys ? levels_k<K, true>(nt, mode, launch, grid, st, lp, tm, per_sm, false)   \
                   : levels_k<K, false>(nt, mode, launch, grid, st, lp, tm, per_sm, dense);
    switch (kind) {
        RIDC_LEV_KIND(ADV_DIFF_1D)
        RIDC_LEV_KIND(BURGERS_1D)
        RIDC_LEV_KIND(RD_1D)
    default: return cudaErrorInvalidValue;
    }
#undef RIDC_LEV_KIND
}

cudaError_t launch_item(int kind, const LaunchCfg& c, int items, cudaStream_t st,
                        const DevProblem& pb, const DevSolve& sv, const StepItem& it,
                        unsigned long long* err)
{
    switch (kind) {
    case ADV_DIFF_1D: return launch_item_k<ADV_DIFF_1D>(c, items, st, pb, sv, it, err);
    case BURGERS_1D: return launch_item_k<BURGERS_1D>(c, items, st, pb, sv, it, err);
    case RD_1D: return launch_item_k<RD_1D>(c, items, st, pb, sv, it, err);
    case ADV_DIFF_2D: return launch_item_k<ADV_DIFF_2D>(c, items, st, pb, sv, it, err);
    case RD_2D: return launch_item_k<RD_2D>(c, items, st, pb, sv, it, err);
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
    double r = 0;
    LaunchCfg cfg;             // register-path (single-op) launch
    // engine (chunk layout)
    ChunkCfg ccfg;
    ChunkLayout lay;
    std::vector<ChunkGeo> cgeo;
    std::string err;
};

// Factors of (I - coeff * cdx * D_xx): limits, Dirichlet pivot tables, carry powers.
void make_factors(const DevProblem& pb, double coeff, SolveSetup& ss)
{
    const double r = coeff * pb.cdx;
    ss.r = r;
    DevSolve& sv = ss.sv;
    memset(&sv, 0, sizeof sv);
    const double b = 1.0 + 2.0 * r;
    const double s = std::sqrt(1.0 + 4.0 * r);
    sv.lam = 2.0 * r / (b + s);
    sv.g = 2.0 / (b + s);
    ss.tab.clear();
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
            zf[e] = acc;
        }
    };
    fill_zf(sv.zf4, 4);
    fill_zf(sv.zf8, 8);
    fill_zf(sv.zf16, 16);
    // M^(2^i) for the chunk-carry scans (fast_solve): repeated squaring of lam^K
    auto fill_mp = [&](double* mp, int K) {
        mp[0] = sv.pw[K - 1];
        for (int i = 1; i < 10; ++i) mp[i] = mp[i - 1] * mp[i - 1];
    };
    fill_mp(sv.mp8, 8);
    fill_mp(sv.mp16, 16);
}

// truncation halo: lam^H <= 2^-60 relative to the recurrence magnitude
int halo_of(double lam)
{
    return lam > 0.0 ? (int)std::ceil(60.0 * std::log(2.0) / -std::log(lam)) + 1 : 0;
}

// Register-path tiling for the single operators (ridc_op_*): whole lines up
// to kCap-2 points, else truncated segments.
int make_solve(const DevProblem& pb, double coeff, int cap, int /*balance_items*/, int /*nsm*/,
               SolveSetup& ss)
{
    make_factors(pb, coeff, ss);
    DevSolve& sv = ss.sv;
    if (pb.nx + 2 <= cap) {
        sv.nseg = 1;
        sv.tile = pb.nx;
        sv.halo = 0;
        ss.cfg = pick_cfg(pb.nx + 2);
        return RIDC_OK;
    }
    const int H = halo_of(sv.lam);
    const int Tmax = cap - 2 - 2 * H;
    if (Tmax < 256) {
        char buf[256];
        snprintf(buf, sizeof buf,
                 "stiffness r=%.4g needs a truncation halo of %d points; the segmented "
                 "line solve supports at most %d (use fewer points or a smaller dt)",
                 ss.r, H, (cap - 2 - 256) / 2);
        ss.err = buf;
        return RIDC_E_CONFIG;
    }
    sv.halo = H;
    sv.tile = Tmax;
    sv.nseg = (pb.nx + Tmax - 1) / Tmax;
    sv.tile = (pb.nx + sv.nseg - 1) / sv.nseg;
    ss.cfg = pick_cfg(cap);
    return RIDC_OK;
}

int floor_div(int a, int b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }

// Engine tiling in chunk layout (ridc_chunk.cuh).  Tiling depends only on
// the problem and dt (never on levels or devices), so every level computes
// bitwise the same states on one GPU and in the multi-GPU pipeline.
// Segment count balances `items_per_row_set` x nseg items over nsm CTAs.
int make_chunk_solve(const DevProblem& pb, double coeff, int nsm, SolveSetup& ss)
{
    make_factors(pb, coeff, ss);
    DevSolve& sv = ss.sv;
    const int nx = pb.nx;
    const int pmax = chunk_points_max(pb.kind);
    const bool whole = ((nx + 15) / 16) * 16 <= pmax;
    int H = 0, nseg = 1, T = nx;
    if (!whole) {
        H = halo_of(sv.lam);
        const int Tmax = pmax - 2 * H - 2 - 32;   // group alignment slack
        if (Tmax < 256) {
            char buf[256];
            snprintf(buf, sizeof buf,
                     "stiffness r=%.4g needs a truncation halo of %d points; the segmented "
                     "line solve supports at most %d (use fewer points or a smaller dt)",
                     ss.r, H, (pmax - 2 - 32 - 256) / 2);
            ss.err = buf;
            return RIDC_E_CONFIG;
        }
        const int n0 = (nx + Tmax - 1) / Tmax;
        int nbest = n0;
        long long best = LLONG_MAX;
        for (int n = n0; n <= 4 * n0; ++n) {
            const int Tn = (nx + n - 1) / n;
            const long long items = (long long)pb.ny * n;
            const long long per = (items + nsm - 1) / nsm;
            const long long cost = per * (Tn + 2LL * H + 2 + 512);
            if (cost < best) { best = cost; nbest = n; }
        }
        T = (nx + nbest - 1) / nbest;
        nseg = (nx + T - 1) / T;
    }
    sv.halo = H;
    sv.tile = T;
    sv.nseg = nseg;
    // ghost columns: periodic segments read up to H+1 (+15 alignment) beyond the line
    const int GW = whole ? 16 : 16 * ((H + 1 + 15 + 15) / 16);
    if (!whole && GW > nx) {
        ss.err = "truncation halo longer than the line";
        return RIDC_E_CONFIG;
    }
    ss.lay.GW = GW;
    ss.lay.P = 16 * ((nx + 2 * GW + 15) / 16);
    ss.lay.gpr = ss.lay.P / 16;
    ss.lay.gdata = GW / 16;
    ss.cgeo.clear();
    int maxng = 0;
    for (int seg = 0; seg < nseg; ++seg) {
        ChunkGeo cg;
        cg.c0 = seg * T;
        cg.tlen = std::min(T, nx - cg.c0);
        if (whole) {
            cg.g0 = 0;
            cg.ng = (nx + 15) / 16;
            cg.s_end = nx;
            cg.mode = pb.periodic ? 1 : 2;
        } else {
            int lo = cg.c0 - H - 1, hi = cg.c0 + cg.tlen + H + 1;
            bool exact_l = false, exact_r = false;
            if (!pb.periodic) {
                if (lo <= 0) { lo = 0; exact_l = true; }
                if (hi >= nx) { hi = nx; exact_r = true; }
            }
            cg.g0 = floor_div(lo, 16);
            const int g1 = floor_div(hi + 15, 16);
            cg.ng = g1 - cg.g0;
            cg.s_end = exact_r ? nx - 16 * cg.g0 : 16 * cg.ng;
            const bool in_tab = sv.ntab > 0 && 16 * cg.g0 < sv.ntab;
            cg.mode = (exact_l || exact_r || in_tab) ? 2 : 0;
        }
        maxng = std::max(maxng, cg.ng);
        ss.cgeo.push_back(cg);
    }
    ss.ccfg = pick_chunk(pb.kind, 16 * maxng);
    ss.ccfg.mode = ss.cgeo[0].mode;
    for (const ChunkGeo& g : ss.cgeo)
        if (g.mode != ss.ccfg.mode) ss.ccfg.mode = -1;
    if (pb.periodic && ss.ccfg.mode < 0) {
        ss.err = "internal: periodic line with mixed segment modes";
        return RIDC_E_CONFIG;
    }
    if (!pb.periodic && ss.ccfg.mode != 2) ss.ccfg.mode = -1;
    if (maxng > chunk_groups(ss.ccfg)) {
        ss.err = "internal: item larger than the chunk kernel";
        return RIDC_E_CONFIG;
    }
    return RIDC_OK;
}

// Resident level march geometry (ridc_levels.cuh): the producer segments
// whose tiles (or periodic ghost copies) a consumer segment's staged columns
// read, the converse, the edge width pushed through the halo mailbox and the
// common segment mode.  false: the line does not qualify.
struct ResGeo {
    std::vector<int> deps, readers;   // [nseg][kResDeps], -1 padded
    int edge_w = 0;
    int mode = -1;
};

bool res_geometry(const DevProblem& pb, const SolveSetup& ss, ResGeo& g)
{
    const int nseg = ss.sv.nseg, nx = pb.nx;
    if (!(pb.kind == ADV_DIFF_1D || pb.kind == BURGERS_1D || pb.kind == RD_1D) || pb.ny != 1) return false;
    if (ss.ccfg.rows != 1 || ss.ccfg.kc != kChunk || (int)ss.cgeo.size() != nseg) return false;
    int ext = 0;
    for (const ChunkGeo& c : ss.cgeo) {
        ext = std::max(ext, c.c0 - 16 * c.g0);
        ext = std::max(ext, 16 * (c.g0 + c.ng) - (c.c0 + c.tlen));
    }
    const int W = std::max(ext, ss.lay.GW);
    for (const ChunkGeo& c : ss.cgeo)
        if (nseg > 1 && (ext >= c.tlen || W >= c.tlen)) return false;
    std::vector<int> owner(nx, -1);
    for (int s = 0; s < nseg; ++s)
        for (int c = ss.cgeo[s].c0; c < ss.cgeo[s].c0 + ss.cgeo[s].tlen; ++c) owner[c] = s;
    g.deps.assign((size_t)nseg * kResDeps, -1);
    g.readers.assign((size_t)nseg * kResDeps, -1);
    std::vector<int> nr(nseg, 0);
    for (int k = 0; k < nseg; ++k) {
        const ChunkGeo& c = ss.cgeo[k];
        int nd = 0;
        for (int x = 16 * c.g0; x < 16 * (c.g0 + c.ng); ++x) {
            int col = x;
            if (pb.periodic) col = ((x % nx) + nx) % nx;
            else if (col < 0 || col >= nx) continue;
            const int o = owner[col];
            if (o < 0) return false;
            bool seen = false;
            for (int q = 0; q < nd; ++q) seen |= g.deps[k * kResDeps + q] == o;
            if (seen) continue;
            if (nd == kResDeps) return false;
            g.deps[k * kResDeps + nd++] = o;
            if (nr[o] == kResDeps) return false;
            g.readers[o * kResDeps + nr[o]++] = k;
        }
    }
    g.edge_w = W;
    g.mode = ss.cgeo[0].mode;
    for (const ChunkGeo& c : ss.cgeo)
        if (c.mode != g.mode) g.mode = -1;
    return true;
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
    long long V = 0;           // points per state
    long long Vs = 0;          // ring slot stride: ny padded rows of P doubles
    int nsm = 148;             // CTAs per tick launch
    double* d_weights = nullptr;
    double* d_tab = nullptr;
    ChunkGeo* d_cgeo = nullptr;
    long long* d_dbg = nullptr;
    double* d_ring[kMaxLevels] = {};
    long long cap[kMaxLevels] = {};
    double* d_y0 = nullptr;
    unsigned long long* d_err = nullptr;
    EngineParams ep;
    TmapSet tm;
    std::vector<int> steady_off, startup_off;
    cudaGraphExec_t gexec = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    long long launches = 0;
    long long ring_vectors = 0;
    // resident single-level march (ridc_resident.cuh)
    // trajectory streaming (§8f rank 3): the top ring keeps kTrajDepth slots and
    // every step is drained to pinned host memory by a copy stream
    bool traj_stream = false;
    cudaStream_t cstream = nullptr;
    double* h_traj = nullptr;      // pinned (steps+1) x V
    cudaEvent_t ev_prod = nullptr;
    std::vector<cudaEvent_t> ev_copy;
    bool resident = false;
    int res_mode = -1;             // common segment mode of the resident kernel (-1: mixed)
    unsigned* d_flags = nullptr;   // the watchdog abort word
    uint4* d_mail = nullptr;       // tagged mailbox lines (2 parities x Vs)
    unsigned tag_next = 1;         // next run's epoch
    ResidentParams rp;
    // resident level march (ridc_levels.cuh): levels >= 2 on a 1-D line, one
    // co-resident CTA group per level, device-side flags between the levels
    bool reslev = false;
    bool reslev_dense = false;   // two CTAs per SM (4096-point items)
    int reslev_mode = -1;
    double* d_inbox[kMaxLevels] = {};   // level j's inbox: level j-1's states (j >= 1)
    long long in_cap = 0;
    unsigned long long* d_lflags = nullptr;   // pub [L][nseg], then rel [L][nseg]
    uint4* d_lmail = nullptr;                 // L x 2 parities x Vs tagged lines
    LevelLane* d_lanes = nullptr;
    int* d_geo = nullptr;                     // deps [nseg][4], then readers [nseg][4]
    TmapSet tm_in;
    LevelsParams lp;
    unsigned long long lepoch = 0;
    // carry-exchange FEBE march (ridc_febe_carry.cuh): periodic RD lines, one tile per SM
    bool carry = false;
    bool carry_warp = false;   // k_febe_wcarry: 512-point chunks, one per warp (cparams.T = warps per CTA)
    int carry_wk = 16;         // its points per lane (16 or 32)
    int carry_nt = 0;
    CarryParams cparams;
    uint4* d_cmail = nullptr;
    // streaming FEBE sweep (ridc_sweep.cuh): long periodic RD lines, one launch per step
    bool sweep = false;
    int sweep_nt = 512;
    SweepParams sparams;
    TmapSet tm_sweep;
    // 2-D streaming FEBE sweep (ridc_sweep2d.cuh): every row read once per step
    bool sweep2d = false;
    int sweep2d_nt = 256;
    int sweep2d_grid = 0;
    Sweep2DParams s2params;
    // 1-D level sweep (ridc_sweep_levels.cuh): the ticks of levels >= 2 on long RD lines
    bool sweeplev1 = false;
    // 2-D level sweep (ridc_sweep2d_levels.cuh): the ticks of levels >= 2 on 2-D grids
    bool sweeplev = false;
    int sweeplev_nt = 256;
    int sweeplev_grid = 0;
    SweepLevParams slparams;
    TmapSet tm_lev;
    std::vector<double> h_weights;   // the packed quadrature tables (host copy)
    std::vector<int> h_steady_off;
    // resident RIDC-2 (ridc_carry_res2.cuh): one cooperative launch per interval
    bool carryres = false;
    bool cr_warp = false;   // k_carry_res2w: 512-point chunks, one per warp (cr_nt: the grid)
    int cr_nt = 0;
    CarryRes2Params crparams;
    uint4* d_crmail = nullptr;
    // carry-exchange level tick (ridc_carry_levels.cuh): RIDC p >= 2 on RD lines of <= 14 x SMs x 512 points
    bool carrylev = false;
    int cl_grid = 0, cl_wpc = 0, cl_k = 16;
    CarryLevParams clparams;
    TmapSet tm_cl;
    uint4* d_clx = nullptr;
    unsigned* d_clepoch = nullptr;
    bool fell_back = false;        // a resident march was replaced by the tick graph at run time
    double watchdog = 30.0;        // seconds per in-kernel neighbour wait (ridc_set_watchdog)
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

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link).
typedef CUresult (*PfnEncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                   CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                   CUtensorMapFloatOOBfill);

PfnEncodeTiled encode_tiled()
{
    static PfnEncodeTiled f = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return (PfnEncodeTiled) nullptr;
        return reinterpret_cast<PfnEncodeTiled>(p);
    }();
    return f;
}

// A ring of `cap` slots as a 3-D tensor {16 doubles, Vs/16 groups, cap slots},
// boxes of BR groups, 128-byte swizzle (ridc_chunk.cuh).
int make_ring_map(CUtensorMap* map, double* base, long long Vs, long long cap, int ng, std::string* err)
{
    PfnEncodeTiled enc = encode_tiled();
    if (!enc) return fail(err, RIDC_E_CUDA, "cuTensorMapEncodeTiled unavailable");
    const int BR = ng < 256 ? ng : 256;   // ChunkSmem::BR
    cuuint64_t dims[3] = {16, (cuuint64_t)(Vs / 16), (cuuint64_t)cap};
    cuuint64_t strides[2] = {128, (cuuint64_t)Vs * 8};
    cuuint32_t box[3] = {16, (cuuint32_t)BR, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        char buf[96];
        snprintf(buf, sizeof buf, "cuTensorMapEncodeTiled failed (%d)", (int)r);
        return fail(err, RIDC_E_CUDA, buf);
    }
    return RIDC_OK;
}

EngineParams interval_params(ridc_ctx* c, int interval)
{
    EngineParams ep = c->ep;
    for (int j = 0; j < c->levels; ++j) ep.off[j] = 0;
    if (c->flags & RIDC_RECORD_TRAJECTORY) ep.off[c->levels - 1] = (long long)interval * c->per;
    return ep;
}

const double* final_slot(ridc_ctx* c, int level)
{
    if (c->resident) return c->d_ring[0] + (c->steps % c->cap[0]) * c->Vs;   // one launch, global steps
    if (c->reslev || c->carryres) return c->d_ring[level] + c->Vs;               // slot 1: the final tile
    EngineParams ep = interval_params(c, c->restarts - 1);
    return ep.ring[level] + ((ep.off[level] + c->per) % ep.cap[level]) * c->Vs;
}

// padded ring slot -> plain [ny][nx]
cudaError_t copy_out(ridc_ctx* c, double* dst, const double* slot, cudaMemcpyKind kind, long long nslots = 1)
{
    const ChunkLayout& L = c->ss.lay;
    return cudaMemcpy2DAsync(dst, (size_t)c->pb.nx * sizeof(double), slot + L.GW, (size_t)L.P * sizeof(double),
                             (size_t)c->pb.nx * sizeof(double), (size_t)c->pb.ny * nslots, kind, c->stream);
}

// Capture the whole run: per interval one seed + one launch per tick.
int capture_graph(ridc_ctx* c)
{
    NvtxRange nvtx_("ridc.capture_graph");
    const int L = c->levels;
    const int items = c->pb.ny * c->ss.sv.nseg;
    cudaGraph_t graph = nullptr;
    CUDA_TRY(&c->err, cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    long long launches = 0;
    cudaError_t le = cudaSuccess;
    // trajectory streaming: after the top level writes global step g into slot
    // g % cap, the copy stream drains it to row g of the pinned host buffer;
    // the tick that reuses the slot waits for that copy
    const long long tcap = c->cap[L - 1];
    auto drain = [&](long long g, const double* slot) {
        if (!c->traj_stream || le != cudaSuccess) return;
        const ChunkLayout& Ly = c->ss.lay;
        if ((le = cudaEventRecord(c->ev_prod, c->stream)) != cudaSuccess) return;
        if ((le = cudaStreamWaitEvent(c->cstream, c->ev_prod, 0)) != cudaSuccess) return;
        le = cudaMemcpy2DAsync(c->h_traj + (size_t)g * c->V, (size_t)c->pb.nx * sizeof(double), slot + Ly.GW,
                               (size_t)Ly.P * sizeof(double), (size_t)c->pb.nx * sizeof(double), (size_t)c->pb.ny,
                               cudaMemcpyDeviceToHost, c->cstream);
        if (le == cudaSuccess) le = cudaEventRecord(c->ev_copy[g % tcap], c->cstream);
    };
    auto slot_free = [&](long long g) {   // before the top level writes global step g
        if (c->traj_stream && le == cudaSuccess && g >= tcap)
            le = cudaStreamWaitEvent(c->stream, c->ev_copy[g % tcap], 0);
    };
    for (int r = 0; r < c->restarts && le == cudaSuccess; ++r) {
        EngineParams ep = interval_params(c, r);
        if (r == 0) {
            if (c->carrylev) {   // a fresh tag epoch for the exchange lines of this run
                k_bump_epoch<<<1, 1, 0, c->stream>>>(c->d_clepoch);
                le = cudaGetLastError();
                ++launches;
            }
            const int sb = (int)std::min<long long>((c->Vs + 255) / 256, 148 * 8);
            k_seed_chunk<<<sb, 256, 0, c->stream>>>(c->d_y0, ep, -1);
            le = cudaGetLastError();
            ++launches;
            drain(0, ep.ring[L - 1] + (ep.off[L - 1] % tcap) * c->Vs);   // trajectory row 0: the initial state
        } else {
            // next interval's state0 = the top level's final: plain copy through d_y0
            EngineParams prev = interval_params(c, r - 1);
            const int top = L - 1;
            const double* src = prev.ring[top] + ((prev.off[top] + c->per) % prev.cap[top]) * c->Vs;
            le = copy_out(c, c->d_y0 + c->V, src, cudaMemcpyDeviceToDevice);
            const int sb = (int)std::min<long long>((c->Vs + 255) / 256, 148 * 8);
            if (le == cudaSuccess) {
                k_seed_chunk<<<sb, 256, 0, c->stream>>>(c->d_y0 + c->V, ep, -1);
                le = cudaGetLastError();
            }
            ++launches;
        }
        for (long long k = 1; k <= c->ticks && le == cudaSuccess; ++k) {
            TickParams tp;
            memset(&tp, 0, sizeof tp);
            tp.sv = ep.sv;
            for (int j = 0; j < L; ++j) {
                const long long t = k - delay(j);
                if (t >= 1 && t <= c->per) {
                    tp.level[tp.nact] = j;
                    tp.target[tp.nact] = t;
                    ++tp.nact;
                }
            }
            if (tp.nact == 0) continue;
            const long long ttop = k - delay(L - 1);   // the top level's target this tick
            const bool top_active = ttop >= 1 && ttop <= c->per;
            if (top_active) slot_free((long long)r * c->per + ttop);
            if (le != cudaSuccess) break;
            if (c->carrylev)   // 1-D levels: one chunk per warp, carries exchanged between chunks
                le = carry_levels_k<RD_1D>(c->cl_grid, c->cl_wpc, c->cl_k, c->stream, ep, tp, c->clparams, c->tm_cl,
                                           (unsigned)((long long)r * c->ticks + k));
            else if (c->sweeplev1)   // 1-D levels: every SM sweeps its range for each active level
                le = sweep_levels_k<RD_1D>(c->nsm, c->stream, ep, tp, c->sparams, c->tm_lev);
            else if (c->sweeplev)   // 2-D levels: every CTA sweeps its row block for each active level
                le = c->pb.kind == ADV_DIFF_2D
                         ? sweep2d_levels_k<ADV_DIFF_2D>(c->sweeplev_nt, c->sweeplev_grid, c->stream, ep, tp,
                                                         c->slparams, c->tm_lev)
                         : sweep2d_levels_k<RD_2D>(c->sweeplev_nt, c->sweeplev_grid, c->stream, ep, tp, c->slparams,
                                                   c->tm_lev);
            else if (c->sweep2d)   // 2-D FEBE: every CTA sweeps its row block, each row read once
                le = c->pb.kind == ADV_DIFF_2D
                         ? sweep2d_k<ADV_DIFF_2D>(c->sweep2d_nt, c->sweep2d_grid, c->stream,
                                                  c->s2params, c->tm_sweep, ep.off[0], tp.target[0])
                         : sweep2d_k<RD_2D>(c->sweep2d_nt, c->sweep2d_grid, c->stream, c->s2params,
                                            c->tm_sweep, ep.off[0], tp.target[0]);
            else if (c->sweep)   // FEBE on a long periodic line: every SM sweeps its range
                le = sweep_k<RD_1D>(c->sweep_nt, c->nsm, c->stream, c->sparams, c->tm_sweep,
                                    ep.off[0], tp.target[0]);
            else
                le = launch_chunk(c->pb.kind, c->ss.ccfg,
                                  std::min(c->nsm * chunk_ctas_per_sm(c->ss.ccfg, tp.nact), tp.nact * items),
                                  c->stream, ep, tp, items, c->tm);
            ++launches;
            if (top_active)
                drain((long long)r * c->per + ttop,
                      ep.ring[L - 1] + ((ep.off[L - 1] + ttop) % tcap) * c->Vs);
        }
    }
    if (c->traj_stream && le == cudaSuccess) {   // rejoin the copy stream
        if ((le = cudaEventRecord(c->ev_prod, c->cstream)) == cudaSuccess)
            le = cudaStreamWaitEvent(c->stream, c->ev_prod, 0);
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

// One resident level-march launch per restart interval (ridc_levels.cuh):
// seed every level's own slot 0 and inbox slot 0 with the interval's state0,
// march, then the top level's final becomes the next state0.
// false in *fell_back: the cooperative launch could not get the SMs.
int march_reslev(ridc_ctx* c, bool* fell_back)
{
    *fell_back = false;
    const int L = c->levels, nseg = c->ss.sv.nseg;
    if ((unsigned long long)c->tag_next + (unsigned long long)c->restarts * (c->per + 1) + 2 >= 0xffffffffull) {
        if (c->d_lmail)
            CUDA_TRY(&c->err, cudaMemsetAsync(c->d_lmail, 0, (size_t)L * 2 * c->Vs * sizeof(uint4), c->stream));
        c->tag_next = 1;
    }
    CUDA_TRY(&c->err, cudaMemsetAsync(c->d_flags, 0, sizeof(unsigned), c->stream));
    const int sb = (int)std::min<long long>((c->Vs + 255) / 256, 148 * 8);
    for (int r = 0; r < c->restarts; ++r) {
        const double* src = c->d_y0;
        if (r > 0) {
            CUDA_TRY(&c->err, copy_out(c, c->d_y0 + c->V, final_slot(c, L - 1), cudaMemcpyDeviceToDevice));
            src = c->d_y0 + c->V;
        }
        EngineParams sp;
        memset(&sp, 0, sizeof sp);
        sp.pb = c->pb;
        sp.lay = c->ss.lay;
        sp.levels = L;
        for (int j = 0; j < L; ++j) {
            sp.ring[j] = c->d_ring[j];
            sp.cap[j] = c->cap[j];
        }
        k_seed_chunk<<<sb, 256, 0, c->stream>>>(src, sp, -1);
        CUDA_TRY(&c->err, cudaGetLastError());
        for (int j = 0; j < L; ++j) {
            sp.ring[j] = c->d_inbox[j];
            sp.cap[j] = c->in_cap;
        }
        k_seed_chunk<<<sb, 256, 0, c->stream>>>(src, sp, -1);
        CUDA_TRY(&c->err, cudaGetLastError());
        LevelsParams lp = c->lp;
        lp.epoch = ++c->lepoch;
        lp.tag0 = c->tag_next;
        c->tag_next += (unsigned)c->per + 1;
        const cudaError_t le = levels_dispatch(c->pb.kind, c->ss.ccfg.nt, c->reslev_mode, true, L * nseg,
                                               c->stream, lp, c->tm_in, nullptr, false, c->reslev_dense);
        if (le == cudaErrorCooperativeLaunchTooLarge && r == 0) {
            cudaGetLastError();
            *fell_back = true;
            return RIDC_OK;
        }
        CUDA_TRY(&c->err, le);
    }
    return RIDC_OK;
}

// The resident RIDC-2 march (ridc_carry_res2.cuh): one cooperative launch per
// restart interval from that interval's state0; the top level's final (ring
// slot 1) becomes the next state0.  false in *fell_back: no co-residency.
int march_carryres(ridc_ctx* c, bool* fell_back)
{
    *fell_back = false;
    const int nseg = c->crparams.nseg;
    if ((unsigned long long)c->tag_next + (unsigned long long)c->restarts * (c->per + 3) + 2 >= 0xffffffffull) {
        CUDA_TRY(&c->err, cudaMemsetAsync(c->d_crmail, 0, (size_t)(4 * 4 + 4 * 2) * nseg * sizeof(uint4), c->stream));
        c->tag_next = 1;
    }
    CUDA_TRY(&c->err, cudaMemsetAsync(c->d_flags, 0, sizeof(unsigned), c->stream));
    for (int r = 0; r < c->restarts; ++r) {
        const double* src = c->d_y0;
        if (r > 0) {
            CUDA_TRY(&c->err, copy_out(c, c->d_y0 + c->V, final_slot(c, c->levels - 1), cudaMemcpyDeviceToDevice));
            src = c->d_y0 + c->V;
        }
        CarryRes2Params cp = c->crparams;
        cp.src = src;
        cp.tag0 = c->tag_next;
        c->tag_next += (unsigned)c->per + 3;   // ticks 1 .. per + 2
        const cudaError_t le = c->cr_warp ? carry_res2w_k<RD_1D>(true, c->cr_nt, c->stream, cp, nullptr)
                                          : carry_res2_k<RD_1D>(true, nseg, c->cr_nt, c->stream, cp, nullptr);
        if (le == cudaErrorCooperativeLaunchTooLarge && r == 0) {
            cudaGetLastError();
            *fell_back = true;
            return RIDC_OK;
        }
        CUDA_TRY(&c->err, le);
    }
    return RIDC_OK;
}

int march(ridc_ctx* c, double* wall_seconds)
{
    NvtxRange nvtx_("ridc.march");
    CUDA_TRY(&c->err, cudaMemsetAsync(c->d_err, 0xff, sizeof(unsigned long long), c->stream));
    if (c->carryres) {
        CUDA_TRY(&c->err, cudaEventRecord(c->ev0, c->stream));
        bool fb = false;
        int rc = march_carryres(c, &fb);
        if (rc) return rc;
        if (fb) {   // the SMs are shared right now: the tick kernel's graph for good
            c->carryres = false;
            c->fell_back = true;
            if ((rc = capture_graph(c)) != RIDC_OK) return rc;
        }
    }
    if (c->reslev) {
        CUDA_TRY(&c->err, cudaEventRecord(c->ev0, c->stream));
        bool fb = false;
        int rc = march_reslev(c, &fb);
        if (rc) return rc;
        if (fb) {   // the SMs are shared right now: the tick kernel's graph for good
            c->reslev = false;
            c->fell_back = true;
            if ((rc = capture_graph(c)) != RIDC_OK) return rc;
        }
    }
    if (c->resident) {
        const int nseg = c->ss.sv.nseg;
        // each run tags its mailbox lines with a fresh epoch (no per-run clearing)
        if ((unsigned long long)c->tag_next + c->steps + 2 >= 0xffffffffull) {
            CUDA_TRY(&c->err, cudaMemsetAsync(c->d_mail, 0, 2 * (size_t)c->Vs * sizeof(uint4), c->stream));
            c->tag_next = 1;
        }
        if (c->carry && (unsigned long long)c->tag_next + c->steps + 2 >= 0xffffffffull) {
            CUDA_TRY(&c->err, cudaMemsetAsync(c->d_cmail, 0, (size_t)4 * c->cparams.nseg * sizeof(uint4), c->stream));
            c->tag_next = 1;
        }
        c->rp.tag0 = c->tag_next;
        c->cparams.tag0 = c->tag_next;
        c->tag_next += (unsigned)c->steps + 1;
        CUDA_TRY(&c->err, cudaMemsetAsync(c->d_flags, 0, sizeof(unsigned), c->stream));
        CUDA_TRY(&c->err, cudaEventRecord(c->ev0, c->stream));
        EngineParams ep = interval_params(c, 0);
        const int sb = (int)std::min<long long>((c->Vs + 255) / 256, 148 * 8);
        k_seed_chunk<<<sb, 256, 0, c->stream>>>(c->d_y0, ep, -1);
        CUDA_TRY(&c->err, cudaGetLastError());
        const cudaError_t le =
            c->carry_warp ? febe_wcarry_k<RD_1D>(true, c->carry_wk, (c->cparams.nseg + c->cparams.T - 1) / c->cparams.T,
                                                 c->carry_nt, c->stream, c->cparams, nullptr)
            : c->carry ? febe_carry_k<RD_1D>(true, c->cparams.nseg, c->carry_nt, c->stream, c->cparams, nullptr)
                     : resident_dispatch(c->pb.kind, c->ss.ccfg.nt, c->res_mode, true, nseg, c->stream, c->rp,
                                         nullptr);
        if (le == cudaErrorCooperativeLaunchTooLarge) {
            // the SMs are shared with other work right now: fall back (for good) to
            // the tick kernel's graph, which needs no co-residency
            cudaGetLastError();
            c->resident = false;
            c->carry = false;
            c->carry_warp = false;
            c->fell_back = true;
            int rc = capture_graph(c);
            if (rc) return rc;
        } else {
            CUDA_TRY(&c->err, le);
        }
    }
    if (!c->resident && !c->reslev && !c->carryres) {
        if (c->carrylev) CUDA_TRY(&c->err, cudaMemsetAsync(c->d_flags, 0, sizeof(unsigned), c->stream));
        CUDA_TRY(&c->err, cudaEventRecord(c->ev0, c->stream));
        CUDA_TRY(&c->err, cudaGraphLaunch(c->gexec, c->stream));
    }
    CUDA_TRY(&c->err, cudaEventRecord(c->ev1, c->stream));
    CUDA_TRY(&c->err, cudaEventSynchronize(c->ev1));
    if (wall_seconds) {
        float ms = 0.f;
        CUDA_TRY(&c->err, cudaEventElapsedTime(&ms, c->ev0, c->ev1));
        *wall_seconds = ms * 1e-3;
    }
    if (c->resident || c->reslev || c->carrylev || c->carryres) {
        unsigned ab = 0;
        CUDA_TRY(&c->err, cudaMemcpy(&ab, c->d_flags, sizeof ab, cudaMemcpyDeviceToHost));
        if (ab) return fail(&c->err, RIDC_E_PROTOCOL, "resident march: a neighbour segment wait timed out");
    }
    return check_err_word(c);
}

// Carry-exchange FEBE march (ridc_febe_carry.cuh): RIDC order 1 on a periodic
// reaction-diffusion line of a multiple of 16 points, one tile per SM (<= 8192
// points, >= 2 carry reaches + a warp).  *ok = false: the line does not qualify.
int setup_carry(ridc_ctx* c, bool* ok)
{
    *ok = false;
    const DevProblem& pb = c->pb;
    if (pb.kind != RD_1D || pb.ny != 1 || (pb.nx & 15) || c->levels != 1) return RIDC_OK;
    if (getenv("RIDC_NO_CARRY") && atoi(getenv("RIDC_NO_CARRY")) > 0) return RIDC_OK;
    const double lam = c->ss.sv.lam;
    const int hc = halo_of(lam);
    const int nx = pb.nx;
    int per_sm = 0;
    CarryParams cp;
    memset(&cp, 0, sizeof cp);
    cudaError_t oe = febe_carry_k<RD_1D>(false, 0, kCarryMaxNT, c->stream, cp, &per_sm);
    if (oe != cudaSuccess || per_sm < 1) {
        cudaGetLastError();
        return RIDC_OK;
    }
    int nseg = 0, T = 0, nt = 0;
    // lines of 512-point (or 1024-point) chunks: one chunk per warp, warps
    // coupled through shared memory within a CTA (k_febe_wcarry: no block
    // barriers); RIDC_NO_WCARRY=1 keeps the tile march (A/B)
    bool warp_chunks = false;
    int wk = 0;   // points per lane of the warp march
    {
        const bool off = getenv("RIDC_NO_WCARRY") && atoi(getenv("RIDC_NO_WCARRY")) > 0;
        const int kmin = env_int("RIDC_WCARRY_K", 16) >= 32 ? 32 : 16;   // RIDC_WCARRY_K=32: A/B
        for (int k : {16, 32}) {
            if (k < kmin) continue;
            const int ch = 32 * k, nchunk = nx / ch;
            int wps = 0;
            if (off || nx % ch || nchunk < 2 || nchunk > kWCarryMaxWarps * c->nsm || hc > ch) continue;
            const int grid = std::min(c->nsm, nchunk);
            const int wpc = (nchunk + grid - 1) / grid;
            if (febe_wcarry_k<RD_1D>(false, k, 0, 32 * wpc, c->stream, cp, &wps) == cudaSuccess &&
                wps * c->nsm >= (nchunk + wpc - 1) / wpc) {
                warp_chunks = true;
                wk = k;
                T = wpc;              // the warp march reads T as warps per CTA ...
                nseg = nchunk;        // ... and nseg as the line's chunks
                nt = 32 * wpc;
            }
            cudaGetLastError();
            if (warp_chunks) break;
        }
    }
    if (!warp_chunks) {
        // as many tiles as SMs (each tile a multiple of 16 points), fewer if a tile
        // would be shorter than two carry reaches + one warp of chunks
        for (int n = c->nsm; n >= 2; --n) {
            const int t = 16 * ((nx + 16 * n - 1) / (16 * n));
            const int ns = (nx + t - 1) / t;
            const int tlast = nx - (ns - 1) * t;
            if (t > 16 * kCarryMaxNT) break;                     // longer tiles than a CTA holds
            if (ns >= 2 && t >= 2 * hc + 512 && tlast >= 2 * hc + 512) { nseg = ns; T = t; break; }
        }
        if (nseg < 2) return RIDC_OK;
        nt = 32 * ((T / 16 + 31) / 32);
    }
    CUDA_TRY(&c->err, cudaMalloc(&c->d_cmail, (size_t)2 * 2 * nseg * sizeof(uint4)));
    CUDA_TRY(&c->err, cudaMemset(c->d_cmail, 0, (size_t)2 * 2 * nseg * sizeof(uint4)));
    if (!c->d_flags) CUDA_TRY(&c->err, cudaMalloc(&c->d_flags, sizeof(unsigned)));
    cp.pb = pb;
    cp.lam = lam;
    const double g = c->ss.sv.g, dt = c->dt;
    cp.aa = g * (1.0 + dt * pb.rho);   // g (u + dt rho u (1 - u)) = (aa + bb u) u
    cp.bb = -(g * dt * pb.rho);
    cp.inv1ml2 = 1.0 / (1.0 - lam * lam);
    for (int e = 0; e < 16; ++e) {
        cp.pw[e] = c->ss.sv.pw[e];
        cp.zf[e] = c->ss.sv.zf16[e];
    }
    for (int i = 0; i < 10; ++i) cp.mp[i] = c->ss.sv.mp16[i];
    if (wk == 32) {   // the 32-point tables (fill_zf / fill_mp of make_factors for K = 32)
        for (int e = 0; e < 32; ++e) cp.pw[e] = c->ss.sv.pw[e];
        for (int e = 0; e < 32; ++e) {
            double acc = 0.0;
            for (int k = 31; k >= e; --k) acc = acc * lam + cp.pw[k];
            cp.zf[e] = acc;
        }
        cp.mp[0] = cp.pw[31];
        for (int i = 1; i < 10; ++i) cp.mp[i] = cp.mp[i - 1] * cp.mp[i - 1];
    }
    cp.ring = c->d_ring[0];
    cp.cap = c->cap[0];
    cp.Vs = c->Vs;
    cp.GW = c->ss.lay.GW;
    cp.T = T;
    cp.nx = nx;
    cp.nseg = nseg;
    cp.hc = hc;
    cp.mail = c->d_cmail;
    cp.steps = c->steps;
    cp.per = c->per;
    cp.full_every = (c->flags & RIDC_RECORD_TRAJECTORY) ? 1 : 0;
    cp.err = c->d_err;
    cp.abort = c->d_flags;
    cp.spin_limit = (long long)(c->watchdog * 2.0e9);
    cp.exp = env_int("RIDC_WC_EXP", 0);   // diagnostics: WRONG states, timing only
    c->cparams = cp;
    c->carry = true;
    c->carry_warp = warp_chunks;
    c->carry_wk = wk;
    c->carry_nt = nt;
    c->resident = true;   // the resident FEBE path (final state in ring slot steps % cap)
    c->launches = 2;
    *ok = true;
    return RIDC_OK;
}

// Streaming FEBE sweep (ridc_sweep.cuh): RIDC order 1 on a periodic
// reaction-diffusion line too long to stay resident, a multiple of 16 points,
// at least 1024 points per SM, carry reach <= 512.  Runs inside the captured
// graph (one launch per step) in place of the tick kernel.
int setup_sweep(ridc_ctx* c)
{
    const DevProblem& pb = c->pb;
    if (c->resident || c->levels != 1 || pb.kind != RD_1D || pb.ny != 1 || (pb.nx & 15) ||
        (c->flags & RIDC_TICK_ONLY) || c->ss.sv.nseg < 2)
        return RIDC_OK;
    if (getenv("RIDC_NO_SWEEP") && atoi(getenv("RIDC_NO_SWEEP")) > 0) return RIDC_OK;
    const double lam = c->ss.sv.lam;
    const int hc = halo_of(lam);
    if (hc > 512 || pb.nx < 1024 * c->nsm) return RIDC_OK;
    // one independent sweep per warp (ridc_sweep_warp.cuh) when every warp's
    // range holds a full 512-point chunk; else one sweep per CTA (ridc_sweep.cuh).
    // RIDC_SWEEP_CTA=1 keeps the CTA sweep (A/B).
    const bool cta_only = getenv("RIDC_SWEEP_CTA") && atoi(getenv("RIDC_SWEEP_CTA")) > 0;
    c->sweep_nt = (!cta_only && (long long)pb.nx >= (long long)kWarpChunk * kWarpSweepWarps * c->nsm) ? 32 : 512;
    SweepParams& sp = c->sparams;
    memset(&sp, 0, sizeof sp);
    sp.pb = pb;
    sp.lam = lam;
    const double g = c->ss.sv.g, dt = c->dt;
    sp.aa = g * (1.0 + dt * pb.rho);   // g (u + dt rho u (1 - u)) = (aa + bb u) u
    sp.bb = -(g * dt * pb.rho);
    for (int e = 0; e < 16; ++e) {
        sp.pw[e] = c->ss.sv.pw[e];
        sp.zf[e] = c->ss.sv.zf16[e];
    }
    for (int i = 0; i < 10; ++i) sp.mp[i] = c->ss.sv.mp16[i];
    sp.ring = c->d_ring[0];
    sp.cap = c->cap[0];
    sp.Vs = c->Vs;
    sp.GW = c->ss.lay.GW;
    sp.gpr = c->ss.lay.gpr;
    sp.gdata = c->ss.lay.gdata;
    sp.nx = pb.nx;
    sp.hc = hc;
    sp.per = c->per;
    sp.err = c->d_err;
    sp.g = g;
    memset(&c->tm_sweep, 0, sizeof c->tm_sweep);
    int rc = make_ring_map(&c->tm_sweep.map[0], c->d_ring[0], c->Vs, c->cap[0], c->sweep_nt, &c->err);
    if (rc) return rc;
    c->sweep = true;
    return RIDC_OK;
}

// 2-D streaming FEBE sweep (ridc_sweep2d.cuh): RIDC order 1 on the periodic
// 2-D kinds with x-lines of 16 NT points (NT = 128 / 256 / 512: 2048 / 4096 /
// 8192 columns) and at least two rows per CTA.
int setup_sweep2d(ridc_ctx* c)
{
    const DevProblem& pb = c->pb;
    if (c->levels != 1 || !(pb.kind == ADV_DIFF_2D || pb.kind == RD_2D) || (c->flags & RIDC_TICK_ONLY)) return RIDC_OK;
    if (getenv("RIDC_NO_SWEEP") && atoi(getenv("RIDC_NO_SWEEP")) > 0) return RIDC_OK;
    int nt = 0;
    for (int t : {128, 256, 512})
        if (pb.nx == 16 * t) nt = t;
    if (!nt || pb.ny < 2 * c->nsm * (512 / nt)) return RIDC_OK;
    // the tiling of the engine solves the same shifted operator: take its factors
    SolveSetup fs;
    make_factors(pb, c->dt, fs);
    const double lam = fs.sv.lam, g = fs.sv.g, dt = c->dt;
    Sweep2DParams& sp = c->s2params;
    memset(&sp, 0, sizeof sp);
    sp.pb = pb;
    sp.lam = lam;
    if (pb.kind == RD_2D) {   // (1 + dt rho - 2 dt cdy) w - dt rho w^2, neighbours dt cdy
        sp.c0 = g * (1.0 + dt * pb.rho - 2.0 * dt * pb.cdy);
        sp.c1 = -(g * dt * pb.rho);
        sp.cs = g * dt * pb.cdy;
        sp.cn = g * dt * pb.cdy;
    } else {                  // upwind x / y advection + y-diffusion (eval_point, ridc_device.cuh)
        sp.c0 = g * (1.0 - dt * pb.cax - dt * pb.cay - 2.0 * dt * pb.cdy);
        sp.c1 = g * dt * pb.cax;
        sp.cs = g * dt * (pb.cay + pb.cdy);
        sp.cn = g * dt * pb.cdy;
    }
    double lS = 1.0;   // lam^nx
    for (int i = 0; i < pb.nx; ++i) lS *= lam;
    sp.cyc = 1.0 / (1.0 - lS);
    for (int e = 0; e < 16; ++e) {
        sp.pw[e] = fs.sv.pw[e];
        sp.zf[e] = fs.sv.zf16[e];
    }
    for (int i = 0; i < 10; ++i) sp.mp[i] = fs.sv.mp16[i];
    sp.ring = c->d_ring[0];
    sp.cap = c->cap[0];
    sp.Vs = c->Vs;
    sp.P = c->ss.lay.P;
    sp.GW = c->ss.lay.GW;
    sp.gpr = c->ss.lay.gpr;
    sp.gdata = c->ss.lay.gdata;
    sp.nx = pb.nx;
    sp.ny = pb.ny;
    sp.per = c->per;
    sp.err = c->d_err;
    memset(&c->tm_sweep, 0, sizeof c->tm_sweep);
    int rc = make_ring_map(&c->tm_sweep.map[0], c->d_ring[0], c->Vs, c->cap[0], nt, &c->err);
    if (rc) return rc;
    c->sweep2d_nt = nt;
    // 512 / nt CTAs per SM (RIDC_S2D_CPS overrides: diagnostics)
    c->sweep2d_grid = c->nsm * std::max(1, std::min(512 / nt, env_int("RIDC_S2D_CPS", 512 / nt)));
    c->sweep2d = true;
    return RIDC_OK;
}

// 2-D level sweep (ridc_sweep2d_levels.cuh): RIDC order >= 2 on the periodic
// 2-D kinds with x-lines of 4096 or 8192 points and at least two rows per SM.
int setup_sweep2d_levels(ridc_ctx* c)
{
    const DevProblem& pb = c->pb;
    if (c->levels < 2 || !(pb.kind == ADV_DIFF_2D || pb.kind == RD_2D) || (c->flags & RIDC_TICK_ONLY)) return RIDC_OK;
    if (getenv("RIDC_NO_SWEEP") && atoi(getenv("RIDC_NO_SWEEP")) > 0) return RIDC_OK;
    const int nt = pb.nx == 4096 ? 256 : (pb.nx == 8192 ? 512 : 0);
    if (!nt || pb.ny < 2 * c->nsm) return RIDC_OK;
    SolveSetup fs;
    make_factors(pb, c->dt, fs);
    SweepLevParams& sp = c->slparams;
    memset(&sp, 0, sizeof sp);
    sp.lam = fs.sv.lam;
    sp.g = fs.sv.g;
    double lS = 1.0;   // lam^nx
    for (int i = 0; i < pb.nx; ++i) lS *= sp.lam;
    sp.cyc = 1.0 / (1.0 - lS);
    for (int e = 0; e < 16; ++e) {
        sp.pw[e] = fs.sv.pw[e];
        sp.zf[e] = fs.sv.zf16[e];
    }
    for (int i = 0; i < 10; ++i) sp.mp[i] = fs.sv.mp16[i];
    sp.P = c->ss.lay.P;
    sp.GW = c->ss.lay.GW;
    sp.gpr = c->ss.lay.gpr;
    sp.gdata = c->ss.lay.gdata;
    sp.nx = pb.nx;
    sp.ny = pb.ny;
    memset(&c->tm_lev, 0, sizeof c->tm_lev);
    for (int j = 0; j < c->levels; ++j) {   // every level ring, boxes of 256 groups (4096 points)
        int rc = make_ring_map(&c->tm_lev.map[j], c->d_ring[j], c->Vs, c->cap[j], 256, &c->err);
        if (rc) return rc;
    }
    c->sweeplev_nt = nt;
    // 4096-point rows (256 threads): two CTAs per SM (two row chains per SM
    // hide each other's scan latency; 2 stages each); 8192: one
    c->sweeplev_grid = c->nsm * (nt == 256 && pb.ny >= 4 * c->nsm ? std::max(1, std::min(2, env_int("RIDC_S2L_CPS", 2))) : 1);
    c->sweeplev = true;
    return RIDC_OK;
}

// 1-D level sweep (ridc_sweep_levels.cuh): RIDC order >= 2 on a periodic
// reaction-diffusion line of a multiple of 16 points that the resident level
// march cannot hold, at least 1024 points per SM, carry reach <= 512.
int setup_sweep_levels(ridc_ctx* c)
{
    const DevProblem& pb = c->pb;
    if (c->levels < 2 || c->reslev || pb.kind != RD_1D || pb.ny != 1 || (pb.nx & 15) ||
        (c->flags & RIDC_TICK_ONLY) || c->ss.sv.nseg < 2)
        return RIDC_OK;
    if (getenv("RIDC_NO_SWEEP") && atoi(getenv("RIDC_NO_SWEEP")) > 0) return RIDC_OK;
    const double lam = c->ss.sv.lam;
    const int hc = halo_of(lam);
    // at least three chunks per SM: shorter lines stay L2-resident and the tick
    // kernel is faster there (C2 p = 2 / 4 / 8: 15 / 36 / 90 us per tick against
    // 17 / 46 / 134; 2^22: 0.63-0.77 of HBM against 0.56-0.75; 2^26: 0.89-0.98
    // against 0.60-0.74 -- profiles/r2_sweep_c5_levels.json)
    if (hc > 512 || pb.nx < 3 * kSweepLevMaxChunk * c->nsm || c->ss.lay.GW < 16) return RIDC_OK;
    SweepParams& sp = c->sparams;
    memset(&sp, 0, sizeof sp);
    sp.pb = pb;
    sp.lam = lam;
    sp.g = c->ss.sv.g;
    for (int e = 0; e < 16; ++e) {
        sp.pw[e] = c->ss.sv.pw[e];
        sp.zf[e] = c->ss.sv.zf16[e];
    }
    for (int i = 0; i < 10; ++i) sp.mp[i] = c->ss.sv.mp16[i];
    sp.Vs = c->Vs;
    sp.GW = c->ss.lay.GW;
    sp.gpr = c->ss.lay.gpr;
    sp.gdata = c->ss.lay.gdata;
    sp.nx = pb.nx;
    sp.hc = hc;
    sp.per = c->per;
    sp.err = c->d_err;
    memset(&c->tm_lev, 0, sizeof c->tm_lev);
    for (int j = 0; j < c->levels; ++j) {   // every level ring, boxes of 256 groups (4096 points)
        int rc = make_ring_map(&c->tm_lev.map[j], c->d_ring[j], c->Vs, c->cap[j], 256, &c->err);
        if (rc) return rc;
    }
    c->sweeplev1 = true;
    return RIDC_OK;
}

// Resident RIDC-2 (ridc_carry_res2.cuh): two levels of a periodic
// reaction-diffusion line of a multiple of 16 points held on the SMs, one
// tile per SM (<= 16 x 448 points, >= 2 carry reaches + a warp), no
// trajectory recording (the top level's states never leave the SMs).
int setup_carry_res2(ridc_ctx* c)
{
    const DevProblem& pb = c->pb;
    if (c->levels != 2 || pb.kind != RD_1D || pb.ny != 1 || (pb.nx & 15) ||
        (c->flags & (RIDC_TICK_ONLY | RIDC_RECORD_TRAJECTORY)) || c->traj_stream)
        return RIDC_OK;
    if (getenv("RIDC_NO_CARRYRES") && atoi(getenv("RIDC_NO_CARRYRES")) > 0) return RIDC_OK;
    const double lam = c->ss.sv.lam;
    const int hc = halo_of(lam), nx = pb.nx;
    int nseg = 0, T = 0, nt = 0;
    CarryRes2Params& cp = c->crparams;
    memset(&cp, 0, sizeof cp);
    // one 512-point chunk per warp (k_carry_res2w: no block barriers) where the
    // line divides and 7-warp CTAs fit two per SM; RIDC_RES2_TILE=1 keeps the
    // tile march (A/B)
    bool warp_chunks = false;
    if (nx % 512 == 0 && hc <= 512 && nx / 512 >= 2 && env_int("RIDC_RES2_TILE", 0) == 0) {
        // 7-warp CTAs while one per SM holds the line, else one 14-warp CTA per SM
        // (two 7-warp CTAs per SM measured 7% slower at C2, profiles/r2_res2w.json);
        // RIDC_RES2W_WARPS=7 / 14 forces it (A/B)
        const int nch = nx / 512;
        const int fw = env_int("RIDC_RES2W_WARPS", 0);
        const int wpc = fw == 7 || fw == 14 ? fw : ((nch + kR2wWarps - 1) / kR2wWarps > c->nsm ? 14 : kR2wWarps);
        const int grid = (nch + wpc - 1) / wpc;
        cp.T = wpc;
        int per_sm = 0;
        if (carry_res2w_k<RD_1D>(false, 0, c->stream, cp, &per_sm) == cudaSuccess && per_sm * c->nsm >= grid) {
            warp_chunks = true;
            nseg = nch;           // the warp march reads nseg as the line's chunks ...
            T = wpc;              // ... and T as warps per CTA
            nt = grid;            // cr_nt: its grid
        }
        cudaGetLastError();
    }
    if (!warp_chunks) {
        for (int n = c->nsm; n >= 2; --n) {   // the carry march's tiling, 448 threads at most
            const int t = 16 * ((nx + 16 * n - 1) / (16 * n));
            const int ns = (nx + t - 1) / t;
            const int tlast = nx - (ns - 1) * t;
            if (t > 16 * kRes2MaxNT) break;
            if (ns >= 2 && t >= 2 * hc + 512 && tlast >= 2 * hc + 512) { nseg = ns; T = t; break; }
        }
        if (nseg < 2) return RIDC_OK;
        nt = 32 * ((T / 16 + 31) / 32);
        int per_sm = 0;
        if (carry_res2_k<RD_1D>(false, 0, nt, c->stream, cp, &per_sm) != cudaSuccess || per_sm * c->nsm < nseg) {
            cudaGetLastError();
            return RIDC_OK;
        }
    }
    const size_t mb = (size_t)(4 * 4 + 4 * 2) * nseg * sizeof(uint4);
    CUDA_TRY(&c->err, cudaMalloc(&c->d_crmail, mb));
    CUDA_TRY(&c->err, cudaMemset(c->d_crmail, 0, mb));
    if (!c->d_flags) CUDA_TRY(&c->err, cudaMalloc(&c->d_flags, sizeof(unsigned)));
    const double g = c->ss.sv.g, dt = c->dt;
    cp.lam = lam;
    cp.inv1ml2 = 1.0 / (1.0 - lam * lam);
    cp.aa = g * (1.0 + dt * pb.rho);   // the predictor: g (u + dt rho u (1 - u))
    cp.bb = -(g * dt * pb.rho);
    // the corrector's nodes at steady steps (j = 1: window t, t-1; i_new 0, i_old 1), build_item's coefficients
    const double* w = c->h_weights.data() + c->h_steady_off[1];
    const NodeCoef n0 = node_coef<RD_1D>(pb, 1.0, 0.0, dt);
    const NodeCoef nn = node_coef<RD_1D>(pb, 0.0, w[0] - dt, w[0]);
    const NodeCoef no = node_coef<RD_1D>(pb, 0.0, w[1], w[1] - dt);
    cp.a1 = g * n0.a;
    cp.b1 = g * n0.b;
    cp.an = g * nn.a;
    cp.bn = g * nn.b;
    cp.sn = g * nn.cs * pb.cdx;
    cp.ao = g * no.a;
    cp.bo = g * no.b;
    cp.so = g * no.cs * pb.cdx;
    cp.an2 = cp.an - 2.0 * cp.sn;
    cp.ao2 = cp.ao - 2.0 * cp.so;
    for (int e = 0; e < 16; ++e) {
        cp.pw[e] = c->ss.sv.pw[e];
        cp.zf[e] = c->ss.sv.zf16[e];
    }
    for (int i = 0; i < 10; ++i) cp.mp[i] = c->ss.sv.mp16[i];
    cp.fin0 = c->d_ring[0] + c->Vs + c->ss.lay.GW;   // slot 1 of each level (final_slot)
    cp.fin1 = c->d_ring[1] + c->Vs + c->ss.lay.GW;
    cp.T = T;
    cp.nx = nx;
    cp.nseg = nseg;
    cp.hc = hc;
    cp.mail = c->d_crmail;
    cp.edge = c->d_crmail + 16 * nseg;
    cp.per = c->per;
    cp.err = c->d_err;
    cp.abort = c->d_flags;
    cp.spin_limit = (long long)(c->watchdog * 2.0e9);
    c->cr_nt = nt;
    c->cr_warp = warp_chunks;
    c->carryres = true;
    c->launches = c->restarts;
    return RIDC_OK;
}

// The carry-level tick's per-launch solve constants from a factored shift
// (DevSolve: lam, g and the 16-point tables).  lam = 0, g = 1 (the identity
// "solve" of an ARK final combination) zeroes every carry.
void fill_carry_lev(CarryLevParams& cp, const DevSolve& sv, int k = 16)
{
    cp.lam = sv.lam;
    cp.g = sv.g;
    cp.inv1ml2 = 1.0 / (1.0 - sv.lam * sv.lam);
    cp.zc = sv.lam * cp.inv1ml2;
    for (int e = 0; e < 16; ++e) {
        cp.pw[e] = sv.pw[e];
        cp.zf[e] = sv.zf16[e];
    }
    for (int i = 0; i < 10; ++i) cp.mp[i] = sv.mp16[i];
    if (k == 32) {   // the 32-point tables (make_factors' fill_zf / fill_mp for K = 32)
        for (int e = 0; e < 32; ++e) cp.pw[e] = sv.pw[e];
        for (int e = 0; e < 32; ++e) {
            double acc = 0.0;
            for (int j = 31; j >= e; --j) acc = acc * sv.lam + cp.pw[j];
            cp.zf[e] = acc;
        }
        cp.mp[0] = cp.pw[31];
        for (int i = 1; i < 10; ++i) cp.mp[i] = cp.mp[i - 1] * cp.mp[i - 1];
    }
}

// Points per lane of the carry-level tick for a line of nx points whose
// stiffest shift has carry reach hc: 16 (512-point chunks, <= 14 per CTA) where
// it fits, else 32 (1024-point chunks, <= 7 per CTA); 0: neither.
int carry_lev_k(int nx, int hc, int nsm)
{
    if (nx % 512 == 0 && hc <= 512 && nx / 512 >= 2 && nx / 512 <= ClGeom<16>::WARPS * nsm) return 16;
    if (nx % 1024 == 0 && hc <= 1024 && nx / 1024 >= 2 && nx / 1024 <= ClGeom<32>::WARPS * nsm) return 32;
    return 0;
}

// Carry-exchange level tick (ridc_carry_levels.cuh): RIDC order >= 2 on a
// periodic reaction-diffusion line of a multiple of 512 points, at most
// kClWarps x SMs chunks, carry reach <= 512; one launch per tick in the graph.
// Lines the resident level march holds stay there.
int setup_carry_levels(ridc_ctx* c)
{
    const DevProblem& pb = c->pb;
    if (c->levels < 2 || c->reslev || c->resident || pb.kind != RD_1D || pb.ny != 1 || (pb.nx % 512) ||
        (c->flags & RIDC_TICK_ONLY) || c->ss.lay.GW < 16)
        return RIDC_OK;
    if (getenv("RIDC_NO_CARRYLEV") && atoi(getenv("RIDC_NO_CARRYLEV")) > 0) return RIDC_OK;
    const double lam = c->ss.sv.lam;
    const int hc = halo_of(lam);
    const int k = carry_lev_k(pb.nx, hc, c->nsm);
    if (!k) return RIDC_OK;
    const int nchunk = pb.nx / (32 * k);
    const int grid = std::min(c->nsm, nchunk);
    const int wpc = (nchunk + grid - 1) / grid;
    CarryLevParams& cp = c->clparams;
    memset(&cp, 0, sizeof cp);
    fill_carry_lev(cp, c->ss.sv, k);
    cp.nx = pb.nx;
    cp.GW = c->ss.lay.GW;
    cp.gdata = c->ss.lay.gdata;
    cp.nchunk = nchunk;
    cp.wpc = wpc;
    const size_t xb = (size_t)2 * kMaxLevels * nchunk * sizeof(uint4);
    CUDA_TRY(&c->err, cudaMalloc(&c->d_clx, xb));
    CUDA_TRY(&c->err, cudaMemset(c->d_clx, 0, xb));
    CUDA_TRY(&c->err, cudaMalloc(&c->d_clepoch, sizeof(unsigned)));
    CUDA_TRY(&c->err, cudaMemset(c->d_clepoch, 0, sizeof(unsigned)));
    if (!c->d_flags) CUDA_TRY(&c->err, cudaMalloc(&c->d_flags, sizeof(unsigned)));
    CUDA_TRY(&c->err, cudaMemset(c->d_flags, 0, sizeof(unsigned)));
    cp.xch = c->d_clx;
    cp.epoch = c->d_clepoch;
    cp.ticks = (unsigned)(c->restarts * c->ticks + 1);
    cp.abort = c->d_flags;
    cp.spin_limit = (long long)(c->watchdog * 2.0e9);
    cp.exp = env_int("RIDC_CL_EXP", 0);   // diagnostics: WRONG states, timing only
    memset(&c->tm_cl, 0, sizeof c->tm_cl);
    for (int j = 0; j < c->levels; ++j) {   // every level ring, boxes of one chunk + one group either side
        int rc = make_ring_map(&c->tm_cl.map[j], c->d_ring[j], c->Vs, c->cap[j], kClBoxGroups, &c->err);
        if (rc) return rc;
    }
    c->cl_grid = (nchunk + wpc - 1) / wpc;
    c->cl_wpc = wpc;
    c->cl_k = k;
    c->carrylev = true;
    return RIDC_OK;
}

// Resident single-level march: RIDC order 1 on a 1-D line whose segments fit
// one co-resident CTA each, and whose halos reach only the adjacent segments.
int setup_resident(ridc_ctx* c)
{
    const SolveSetup& ss = c->ss;
    const int nseg = ss.sv.nseg;
    const bool one_d = c->pb.kind == ADV_DIFF_1D || c->pb.kind == BURGERS_1D || c->pb.kind == RD_1D;
    if (c->levels != 1 || !one_d || c->pb.ny != 1 || (c->flags & RIDC_TICK_ONLY) || c->traj_stream)
        return RIDC_OK;
    if (nseg > 1) {   // segmented periodic RD: the carry-exchange march when the line qualifies
        bool ok = false;
        int rc = setup_carry(c, &ok);
        if (rc || ok) return rc;
    }
    if (nseg > c->nsm) return RIDC_OK;
    // whole lines: one CTA marches alone, 2x faster than a launch per step;
    // segmented lines: one co-resident CTA per segment exchanging truncation-halo
    // edges through tagged mailbox lines, ~1.3x faster than the tick kernel (C2)
    // farthest reach of a staged range beyond its tile; every column that close
    // to a tile end is published each step (and at least the periodic ghosts)
    int ext = 0;
    for (const ChunkGeo& g : ss.cgeo) {
        ext = std::max(ext, g.c0 - 16 * g.g0);
        ext = std::max(ext, 16 * (g.g0 + g.ng) - (g.c0 + g.tlen));
    }
    const int W = std::max(ext, ss.lay.GW);
    for (const ChunkGeo& g : ss.cgeo)
        if (nseg > 1 && (ext >= g.tlen || W >= g.tlen)) return RIDC_OK;   // halo spans past a neighbour
    int per_sm = 0;
    ResidentParams& rp = c->rp;
    memset(&rp, 0, sizeof rp);
    int mode = ss.cgeo[0].mode;
    for (const ChunkGeo& g : ss.cgeo)
        if (g.mode != mode) mode = -1;
    c->res_mode = mode;
    const cudaError_t oe = resident_dispatch(c->pb.kind, ss.ccfg.nt, mode, false, 0, c->stream, rp, &per_sm);
    if (oe != cudaSuccess || per_sm * c->nsm < nseg) {
        if (getenv("RIDC_DEBUG"))
            fprintf(stderr, "ridc: resident march unavailable (%s, %d blocks/SM x %d SMs < %d segments)\n",
                    cudaGetErrorString(oe), per_sm, c->nsm, nseg);
        cudaGetLastError();
        return RIDC_OK;
    }
    CUDA_TRY(&c->err, cudaMalloc(&c->d_flags, sizeof(unsigned)));
    if (nseg > 1) {
        CUDA_TRY(&c->err, cudaMalloc(&c->d_mail, 2 * (size_t)c->Vs * sizeof(uint4)));
        CUDA_TRY(&c->err, cudaMemset(c->d_mail, 0, 2 * (size_t)c->Vs * sizeof(uint4)));
    }
    rp.pb = c->pb;
    rp.sv = ss.sv;
    rp.lay = ss.lay;
    rp.cgeo = c->d_cgeo;
    rp.ring = c->d_ring[0];
    rp.cap = c->cap[0];
    rp.Vs = c->Vs;
    rp.dt = c->dt;
    rp.steps = c->steps;
    rp.per = c->per;
    rp.edge_w = W;
    rp.full_every = (c->flags & RIDC_RECORD_TRAJECTORY) ? 1 : 0;
    rp.mail = c->d_mail;
    rp.abort = c->d_flags;
    rp.err = c->d_err;
    rp.spin_limit = (long long)(c->watchdog * 2.0e9);   // clock64 cycles (~2 GHz) per neighbour wait
    rp.dbg = c->d_dbg;
    rp.exp = getenv("RIDC_RES_EXP") ? atoi(getenv("RIDC_RES_EXP")) : 0;   // diagnostics only
    c->resident = true;
    c->launches = 2;
    return RIDC_OK;
}

// Resident level march for levels >= 2 on a 1-D line: every level's segments
// co-resident (L x nseg CTAs, one per SM), no trajectory recording.
int setup_reslev(ridc_ctx* c)
{
    const int L = c->levels, nseg = c->ss.sv.nseg;
    if (L < 2 || (c->flags & (RIDC_TICK_ONLY | RIDC_RECORD_TRAJECTORY)) || c->traj_stream) return RIDC_OK;
    if (getenv("RIDC_NO_RESIDENT_LEVELS") && atoi(getenv("RIDC_NO_RESIDENT_LEVELS")) > 0) return RIDC_OK;
    ResGeo g;
    if (!res_geometry(c->pb, c->ss, g)) return RIDC_OK;
    LevelsParams& lp = c->lp;
    memset(&lp, 0, sizeof lp);
    int per_sm = 0;
    cudaError_t oe = levels_dispatch(c->pb.kind, c->ss.ccfg.nt, g.mode, false, 0, c->stream, lp, c->tm, &per_sm,
                                     false, false);
    c->reslev_dense = false;
    if ((oe != cudaSuccess || per_sm * c->nsm < L * nseg) && c->ss.ccfg.nt == 256) {
        cudaGetLastError();
        oe = levels_dispatch(c->pb.kind, c->ss.ccfg.nt, g.mode, false, 0, c->stream, lp, c->tm, &per_sm, false, true);
        c->reslev_dense = true;
    }
    if (oe != cudaSuccess || per_sm * c->nsm < L * nseg) {
        if (getenv("RIDC_DEBUG"))
            fprintf(stderr, "ridc: resident level march unavailable (%s, %d blocks/SM x %d SMs < %d)\n",
                    cudaGetErrorString(oe), per_sm, c->nsm, L * nseg);
        cudaGetLastError();
        return RIDC_OK;
    }
    c->reslev_mode = g.mode;
    // >= j + 3 for every level (window + deferred publication: deadlock-free), + slack;
    // RIDC_LEVEL_INBOX shrinks it (tests: backpressure on every step)
    c->in_cap = std::max<long long>(env_int("RIDC_LEVEL_INBOX", 16), L + 2);
    memset(&c->tm_in, 0, sizeof c->tm_in);
    for (int j = 1; j < L; ++j) {
        const size_t b = (size_t)c->in_cap * c->Vs * sizeof(double);
        CUDA_TRY(&c->err, cudaMalloc(&c->d_inbox[j], b));
        CUDA_TRY(&c->err, cudaMemset(c->d_inbox[j], 0, b));   // Dirichlet ghosts stay 0
        c->ring_vectors += c->in_cap;
        int rc = make_ring_map(&c->tm_in.map[j], c->d_inbox[j], c->Vs, c->in_cap, chunk_groups(c->ss.ccfg), &c->err);
        if (rc) return rc;
    }
    CUDA_TRY(&c->err, cudaMalloc(&c->d_lflags, (size_t)2 * L * nseg * sizeof(unsigned long long)));
    CUDA_TRY(&c->err, cudaMemset(c->d_lflags, 0, (size_t)2 * L * nseg * sizeof(unsigned long long)));
    if (nseg > 1) {
        CUDA_TRY(&c->err, cudaMalloc(&c->d_lmail, (size_t)L * 2 * c->Vs * sizeof(uint4)));
        CUDA_TRY(&c->err, cudaMemset(c->d_lmail, 0, (size_t)L * 2 * c->Vs * sizeof(uint4)));
    }
    if (!c->d_flags) CUDA_TRY(&c->err, cudaMalloc(&c->d_flags, sizeof(unsigned)));
    CUDA_TRY(&c->err, cudaMalloc(&c->d_geo, 2 * g.deps.size() * sizeof(int)));
    CUDA_TRY(&c->err, cudaMemcpy(c->d_geo, g.deps.data(), g.deps.size() * sizeof(int), cudaMemcpyHostToDevice));
    CUDA_TRY(&c->err, cudaMemcpy(c->d_geo + g.deps.size(), g.readers.data(), g.readers.size() * sizeof(int),
                                 cudaMemcpyHostToDevice));
    unsigned long long* pub = c->d_lflags;
    unsigned long long* rel = c->d_lflags + (size_t)L * nseg;
    std::vector<LevelLane> lanes(L);
    for (int j = 0; j < L; ++j) {
        LevelLane& ln = lanes[j];
        memset(&ln, 0, sizeof ln);
        ln.level = j;
        ln.in_map = j;
        ln.own0 = c->d_ring[j];
        ln.fin = c->d_ring[j] + c->Vs;
        ln.in_off = 0;
        ln.in_cap = c->in_cap;
        ln.in_pub = pub + (size_t)j * nseg;
        ln.in_rel = rel + (size_t)j * nseg;
        if (j < L - 1) {
            ln.out = c->d_inbox[j + 1];
            ln.out_off = 0;
            ln.out_cap = c->in_cap;
            ln.out_pub = pub + (size_t)(j + 1) * nseg;
            ln.out_rel = rel + (size_t)(j + 1) * nseg;
        }
        ln.mail = c->d_lmail ? c->d_lmail + (size_t)j * 2 * c->Vs : nullptr;
    }
    CUDA_TRY(&c->err, cudaMalloc(&c->d_lanes, L * sizeof(LevelLane)));
    CUDA_TRY(&c->err, cudaMemcpy(c->d_lanes, lanes.data(), L * sizeof(LevelLane), cudaMemcpyHostToDevice));
    lp.pb = c->pb;
    lp.sv = c->ss.sv;
    lp.lay = c->ss.lay;
    lp.cgeo = c->d_cgeo;
    lp.lanes = c->d_lanes;
    lp.deps = c->d_geo;
    lp.readers = c->d_geo + g.deps.size();
    lp.weights = c->d_weights;
    for (int j = 0; j < kMaxLevels; ++j) {
        lp.steady_off[j] = c->steady_off[j];
        lp.startup_off[j] = c->startup_off[j];
    }
    lp.dt = c->dt;
    lp.per = c->per;
    lp.Vs = c->Vs;
    lp.edge_w = g.edge_w;
    lp.pub_every = env_int("RIDC_PUB_EVERY", 4);
    lp.err = c->d_err;
    lp.abort = c->d_flags;
    lp.spin_limit = (long long)(c->watchdog * 2.0e9);   // clock64 cycles (~2 GHz) per wait
    c->reslev = true;
    c->launches = 3LL * c->restarts;   // per interval: two seeds + one march
    return RIDC_OK;
}

}  // namespace

extern "C" {

int ridc_create(const ridc_problem* problem, double t_start, double t_end, int32_t levels,
                int64_t steps, int32_t restarts, const double* weights, int64_t nweights,
                int32_t device, uint32_t flags, ridc_ctx** out)
{
    NvtxRange nvtx_("ridc.create");
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
    if ((rc = make_chunk_solve(c->pb, c->dt, c->nsm, c->ss)) != RIDC_OK) {
        c->err = c->ss.err;
        return bail(rc);
    }
    prefer_two_per_sm(c->ss.ccfg, levels);
    c->Vs = (long long)c->pb.ny * c->ss.lay.P;
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
    if (wtotal > 0) c->h_weights.assign(weights, weights + wtotal);
    c->h_steady_off = st;
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
    CTX_TRY(cudaMalloc(&c->d_cgeo, c->ss.cgeo.size() * sizeof(ChunkGeo)));
    CTX_TRY(cudaMemcpy(c->d_cgeo, c->ss.cgeo.data(), c->ss.cgeo.size() * sizeof(ChunkGeo),
                       cudaMemcpyHostToDevice));
    if (getenv("RIDC_PHASE_TIMING") && atoi(getenv("RIDC_PHASE_TIMING")) > 0) {
        CTX_TRY(cudaMalloc(&c->d_dbg, kDbgWords * sizeof(long long)));
        CTX_TRY(cudaMemset(c->d_dbg, 0, kDbgWords * sizeof(long long)));
        c->ss.sv.dbg = c->d_dbg;
    }
    memset(&c->tm, 0, sizeof c->tm);
    if (flags & RIDC_RECORD_TRAJECTORY) {
        // keep the whole trajectory on the device when it fits comfortably, else stream it
        size_t freeb = 0, totalb = 0;
        cudaMemGetInfo(&freeb, &totalb);
        const double traj_bytes = (double)(steps + 1) * (double)c->Vs * sizeof(double);
        const char* e = getenv("RIDC_TRAJ_STREAM");
        c->traj_stream = e ? atoi(e) > 0 : traj_bytes > 0.5 * (double)freeb;
    }
    for (int j = 0; j < levels; ++j) {
        const bool top = j == levels - 1;
        long long cap = top ? 2 : 2LL * j + 3;
        if (top && (flags & RIDC_RECORD_TRAJECTORY)) cap = c->traj_stream ? std::min<long long>(kTrajDepth, steps + 1)
                                                                           : steps + 1;
        c->cap[j] = cap;
        c->ring_vectors += cap;
        // ny padded rows per slot; zeroed once: Dirichlet ghosts stay 0 forever
        CTX_TRY(cudaMalloc(&c->d_ring[j], (size_t)cap * c->Vs * sizeof(double)));
        CTX_TRY(cudaMemset(c->d_ring[j], 0, (size_t)cap * c->Vs * sizeof(double)));
        if ((rc = make_ring_map(&c->tm.map[j], c->d_ring[j], c->Vs, cap, chunk_groups(c->ss.ccfg), &c->err)) != RIDC_OK)
            return bail(rc);
    }
    if (c->traj_stream) {
        if (cudaHostAlloc(&c->h_traj, (size_t)(steps + 1) * c->V * sizeof(double), cudaHostAllocDefault) != cudaSuccess) {
            cudaGetLastError();
            c->h_traj = nullptr;
            c->err = "trajectory needs " + std::to_string((double)(steps + 1) * c->V * 8 / 1e9) +
                     " GB of pinned host memory; allocation failed";
            return bail(RIDC_E_CONFIG);
        }
        CTX_TRY(cudaStreamCreateWithFlags(&c->cstream, cudaStreamNonBlocking));
        CTX_TRY(cudaEventCreateWithFlags(&c->ev_prod, cudaEventDisableTiming));
        c->ev_copy.assign((size_t)c->cap[levels - 1], nullptr);
        for (auto& ev : c->ev_copy) CTX_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    }
    CTX_TRY(cudaMalloc(&c->d_y0, 2 * (size_t)c->V * sizeof(double)));
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
    ep.lay = c->ss.lay;
    ep.cgeo = c->d_cgeo;
    if ((rc = setup_resident(c)) != RIDC_OK) return bail(rc);
    // RIDC-2 on RD lines: both levels per tile (ridc_carry_res2.cuh; 3.1 us per
    // tick at 2^16-2^18 against the resident level march's 5.9-10); other
    // orders: the resident level march where levels x segments fit the SMs
    if (!c->resident && (rc = setup_carry_res2(c)) != RIDC_OK) return bail(rc);
    if (!c->resident && !c->carryres && (rc = setup_reslev(c)) != RIDC_OK) return bail(rc);
    if ((rc = setup_sweep(c)) != RIDC_OK) return bail(rc);
    if ((rc = setup_sweep2d(c)) != RIDC_OK) return bail(rc);
    if ((rc = setup_sweep2d_levels(c)) != RIDC_OK) return bail(rc);
    if (!c->carryres && (rc = setup_carry_levels(c)) != RIDC_OK) return bail(rc);
    if (!c->carrylev && (rc = setup_sweep_levels(c)) != RIDC_OK) return bail(rc);
    if (!c->resident && !c->reslev && !c->carryres && (rc = capture_graph(c)) != RIDC_OK) return bail(rc);
#undef CTX_TRY
    *out = c;
    return RIDC_OK;
}

int ridc_run(ridc_ctx* c, const double* y0_host, double* final_host, double* level_finals_host,
             double* traj_host, double* wall_seconds)
{
    NvtxRange nvtx_("ridc.run");
    if (!c || !y0_host || !final_host) return fail(c ? &c->err : nullptr, RIDC_E_CONFIG, "NULL argument");
    if (traj_host && !(c->flags & RIDC_RECORD_TRAJECTORY))
        return fail(&c->err, RIDC_E_CONFIG, "trajectory requested but not recorded (flags)");
    CUDA_TRY(&c->err, cudaSetDevice(c->device));
    const size_t vb = (size_t)c->V * sizeof(double);
    CUDA_TRY(&c->err, cudaMemcpyAsync(c->d_y0, y0_host, vb, cudaMemcpyHostToDevice, c->stream));
    int rc = march(c, wall_seconds);
    if (rc) return rc;
    CUDA_TRY(&c->err, copy_out(c, final_host, final_slot(c, c->levels - 1), cudaMemcpyDeviceToHost));
    if (level_finals_host)
        for (int j = 0; j < c->levels; ++j)
            CUDA_TRY(&c->err, copy_out(c, level_finals_host + (size_t)j * c->V, final_slot(c, j),
                                       cudaMemcpyDeviceToHost));
    if (traj_host && !c->traj_stream)
        CUDA_TRY(&c->err, copy_out(c, traj_host, c->d_ring[c->levels - 1], cudaMemcpyDeviceToHost,
                                   c->steps + 1));
    CUDA_TRY(&c->err, cudaStreamSynchronize(c->stream));
    if (traj_host && c->traj_stream)   // drained during the march (the graph joins the copy stream)
        memcpy(traj_host, c->h_traj, (size_t)(c->steps + 1) * c->V * sizeof(double));
    return RIDC_OK;
}

int ridc_run_device(ridc_ctx* c, const double* y0_dev, double* final_dev, double* wall_seconds)
{
    NvtxRange nvtx_("ridc.run_device");
    if (!c || !y0_dev || !final_dev) return fail(c ? &c->err : nullptr, RIDC_E_CONFIG, "NULL argument");
    CUDA_TRY(&c->err, cudaSetDevice(c->device));
    const size_t vb = (size_t)c->V * sizeof(double);
    CUDA_TRY(&c->err, cudaMemcpyAsync(c->d_y0, y0_dev, vb, cudaMemcpyDeviceToDevice, c->stream));
    int rc = march(c, wall_seconds);
    if (rc) return rc;
    CUDA_TRY(&c->err, copy_out(c, final_dev, final_slot(c, c->levels - 1), cudaMemcpyDeviceToDevice));
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
    info->tile = c->carry_warp ? 32 * c->carry_wk : c->carry ? c->cparams.T : c->ss.sv.tile;
    info->halo = c->carry ? 0 : c->ss.sv.halo;   // the carry march exchanges carries, not halos
    info->items_per_level = c->carry ? c->cparams.nseg : c->pb.ny * c->ss.sv.nseg;
    info->threads = c->carry ? c->carry_nt : c->ss.ccfg.nt;
    info->ring_vectors = c->ring_vectors;
    info->lambda = c->ss.sv.lam;
    info->r = c->ss.r;
    info->path = c->carry_warp ? RIDC_PATH_WARP_CARRY_FEBE
                 : c->carry ? RIDC_PATH_CARRY_FEBE
                 : (c->sweep && !c->resident) ? (c->sweep_nt == 32 ? RIDC_PATH_SWEEP_WARP_FEBE : RIDC_PATH_SWEEP_FEBE)
                 : c->sweep2d ? RIDC_PATH_SWEEP2D_FEBE
                 : c->sweeplev ? RIDC_PATH_SWEEP2D_LEVELS
                 : c->sweeplev1 ? RIDC_PATH_SWEEP_LEVELS
                 : c->carrylev ? RIDC_PATH_CARRY_LEVELS
                 : c->carryres ? RIDC_PATH_RESIDENT_CARRY_LEVELS
                          : c->resident ? RIDC_PATH_RESIDENT_FEBE
                                        : (c->reslev ? RIDC_PATH_RESIDENT_LEVELS : RIDC_PATH_TICK);
    info->fell_back = c->fell_back ? 1 : 0;
    return RIDC_OK;
}

int ridc_set_watchdog(ridc_ctx* c, double seconds)
{
    if (!c || !(seconds > 0.0)) return fail(c ? &c->err : nullptr, RIDC_E_CONFIG, "watchdog must be positive");
    c->watchdog = seconds;
    c->rp.spin_limit = (long long)(seconds * 2.0e9);
    c->lp.spin_limit = (long long)(seconds * 2.0e9);
    c->cparams.spin_limit = (long long)(seconds * 2.0e9);
    c->crparams.spin_limit = (long long)(seconds * 2.0e9);
    if (c->carrylev && c->clparams.spin_limit != (long long)(seconds * 2.0e9)) {
        // the limit is a kernel parameter of every captured tick: capture again
        c->clparams.spin_limit = (long long)(seconds * 2.0e9);
        CUDA_TRY(&c->err, cudaSetDevice(c->device));
        CUDA_TRY(&c->err, cudaStreamSynchronize(c->stream));
        if (c->gexec) cudaGraphExecDestroy(c->gexec);
        c->gexec = nullptr;
        return capture_graph(c);
    }
    return RIDC_OK;
}

int ridc_destroy(ridc_ctx* c)
{
    if (!c) return RIDC_OK;
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    if (c->gexec) cudaGraphExecDestroy(c->gexec);
    for (int j = 0; j < kMaxLevels; ++j)
        if (c->d_ring[j]) cudaFree(c->d_ring[j]);
    if (c->d_weights) cudaFree(c->d_weights);
    if (c->d_tab) cudaFree(c->d_tab);
    if (c->d_cgeo) cudaFree(c->d_cgeo);
    if (c->d_dbg) cudaFree(c->d_dbg);
    if (c->d_y0) cudaFree(c->d_y0);
    if (c->d_err) cudaFree(c->d_err);
    if (c->d_flags) cudaFree(c->d_flags);
    if (c->d_mail) cudaFree(c->d_mail);
    if (c->d_cmail) cudaFree(c->d_cmail);
    if (c->d_clx) cudaFree(c->d_clx);
    if (c->d_crmail) cudaFree(c->d_crmail);
    if (c->d_clepoch) cudaFree(c->d_clepoch);
    for (int j = 0; j < kMaxLevels; ++j)
        if (c->d_inbox[j]) cudaFree(c->d_inbox[j]);
    if (c->d_lflags) cudaFree(c->d_lflags);
    if (c->d_lmail) cudaFree(c->d_lmail);
    if (c->d_lanes) cudaFree(c->d_lanes);
    if (c->d_geo) cudaFree(c->d_geo);
    if (c->ev0) cudaEventDestroy(c->ev0);
    if (c->ev1) cudaEventDestroy(c->ev1);
    if (c->ev_prod) cudaEventDestroy(c->ev_prod);
    for (cudaEvent_t ev : c->ev_copy)
        if (ev) cudaEventDestroy(ev);
    if (c->cstream) cudaStreamDestroy(c->cstream);
    if (c->h_traj) cudaFreeHost(c->h_traj);
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
    CUDA_TRY(nullptr, cudaMemcpy(out, c->d_dbg, std::min(n, kDbgWords) * sizeof(long long), cudaMemcpyDeviceToHost));
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

// Wait until *flag >= want on stream st.  remote: the value (and the data it
// publishes) is written from another device; the stream wait then needs
// CU_STREAM_WAIT_VALUE_FLUSH so that later work sees the producer's earlier
// remote writes -- or, where the device cannot flush remote writes, an
// in-kernel system-scope acquire poll (k_wait_flag).
cudaError_t wait_value(cudaStream_t st, const unsigned long long* flag, unsigned long long want, bool remote,
                       bool can_flush, unsigned* abort, long long spin_limit)
{
    const DriverOps& ops = driver_ops();
    if (remote && !can_flush) {
        k_wait_flag<<<1, 32, 0, st>>>(flag, want, abort, spin_limit);
        return cudaGetLastError();
    }
    const unsigned flags = CU_STREAM_WAIT_VALUE_GEQ | (remote ? CU_STREAM_WAIT_VALUE_FLUSH : 0);
    return ops.wait(reinterpret_cast<CUstream>(st), (CUdeviceptr)flag, (cuuint64_t)want, flags) == CUDA_SUCCESS
               ? cudaSuccess
               : cudaErrorUnknown;
}

bool device_can_flush_remote(int device)
{
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrCanFlushRemoteWrites, device) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return v != 0;
}

constexpr uint32_t kBlobMagic = 0x52494443u;   // "RIDC"
constexpr size_t kFlagBytes = 4096;            // wm (+0), rel (+8), pub[nseg] (+256), relv[nseg] (+2048), then the inbox ring
constexpr size_t kPubOff = 256, kRelOff = 2048;
// levels x shards words (after relv[kPipeMaxSeg]): global step numbers
constexpr size_t kWInUp = 3840;     // inbox ghost row 0 delivered (by level-1, shard-1)
constexpr size_t kWInDn = 3848;     // inbox ghost row n+1 delivered (by level-1, shard+1)
constexpr size_t kWRelUp = 3856;    // released-below of consumer (level+1, shard-1)
constexpr size_t kWRelDn = 3864;    // released-below of consumer (level+1, shard+1)
constexpr size_t kWGhUp = 3872;     // own ghost row 0 delivered (by level, shard-1)
constexpr size_t kWGhDn = 3880;     // own ghost row n+1 delivered (by level, shard+1)
constexpr size_t kWDoneUp = 3888;   // (level, shard-1) finished step g
constexpr size_t kWDoneDn = 3896;   // (level, shard+1) finished step g
constexpr int kPipeMaxSeg = (int)((kRelOff - kPubOff) / 8);
static_assert(kRelOff + 8 * kPipeMaxSeg <= kWInUp && kWDoneDn + 8 <= kFlagBytes, "mailbox words overlap");

struct PipeBlob {
    uint32_t magic;
    int32_t pid, device, level;
    cudaIpcMemHandle_t handle;
    uint64_t direct;       // mailbox base (valid inside the exporting process)
    int64_t inbox_cap;
    int64_t vs;
    int32_t resident;      // resident level march (device-side flags) vs stream memops
    int32_t shard, nshards, rows;   // row shard of a levels x shards grid (rows: local ny incl. 2 ghost rows)
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
    void* opened[8] = {};
    uint64_t opened_direct[8] = {};
    int32_t opened_pid[8] = {};
    // levels x row shards (ridc_pipe_create_shard): this rank computes level
    // `level` on rows [r0, r0 + nrows) of a gny-row grid, held as a local grid
    // of nrows + 2 rows (ghost rows 0 and nrows + 1); the own ring lives in the
    // mailbox allocation so the neighbour shards can deliver its ghost rows
    int shard = 0, nshards = 1, r0 = 0, nrows = 0, gny = 0;
    double* d_s0 = nullptr;                       // the interval's state0 rows r0-1 .. r0+nrows (local seed)
    double* up_inbox = nullptr;                   // (level+1, shard-1)'s inbox ring
    double* dn_inbox = nullptr;                   // (level+1, shard+1)'s inbox ring
    int up_rows = 0, dn_rows = 0;                 // local rows (ghosts included) of shards s-1 / s+1
    unsigned long long* up_in_wm = nullptr;       // its W_INDN: my first row landed in its ghost row n+1
    unsigned long long* dn_in_wm = nullptr;       // its W_INUP: my last row landed in its ghost row 0
    unsigned long long* prev_up_rel = nullptr;    // (level-1, shard-1)'s W_RELDN: I release my ghost-row-0 slots
    unsigned long long* prev_dn_rel = nullptr;    // (level-1, shard+1)'s W_RELUP
    double* side_up_own = nullptr;                // (level, shard-1)'s own ring
    double* side_dn_own = nullptr;                // (level, shard+1)'s own ring
    unsigned long long* side_up_gh = nullptr;     // its W_GHDN: my first row landed in its ghost row n+1
    unsigned long long* side_dn_gh = nullptr;     // its W_GHUP
    unsigned long long* side_up_done = nullptr;   // its W_DONEDN: I finished step g
    unsigned long long* side_dn_done = nullptr;   // its W_DONEUP
    bool up_remote = false, dn_remote = false;    // the up / down neighbours of the previous level sit on another device
    bool sup_remote = false, sdn_remote = false;  // the same-level neighbours
    double* d_weights = nullptr;
    double* d_tab = nullptr;
    ChunkGeo* d_cgeo = nullptr;
    unsigned long long* d_err = nullptr;
    TmapSet tm;
    std::vector<int> st, su;
    std::map<int, cudaGraphExec_t> graphs;
    long long launches = 0;
    // resident level march (ridc_levels.cuh): one launch per interval, the
    // watermark / release protocol as per-segment flags polled in the kernel
    bool reslev_ok = false, reslev = false;
    int reslev_mode = -1;
    ResGeo rgeo;
    int* d_geo = nullptr;
    uint4* d_lmail = nullptr;
    unsigned* d_abort = nullptr;
    LevelLane* d_lanes = nullptr;   // one per interval (filled at connect)
    unsigned long long* in_rel = nullptr;    // producer's relv (peer)
    unsigned long long* out_pub = nullptr;   // consumer's pub (peer)
    unsigned long long lepoch = 0;
    unsigned tag_next = 1;
    bool prev_remote = false;   // the producer (level - 1) sits on another device
    bool can_flush = false;     // this device can flush remote writes after a stream wait
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
    ep.lay = p->ss.lay;
    ep.cgeo = p->d_cgeo;
    if (p->nshards > 1) ep.row0 = 1;   // rows 1..nrows; rows 0 and nrows + 1 are the neighbours' ghosts
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
            if (wait_value(p->stream, p->wm, (unsigned long long)need, p->prev_remote, p->can_flush, p->d_abort,
                           (long long)(p->watchdog * 2.0e9)) != cudaSuccess)
                return pipe_fail(p, RIDC_E_CUDA, "watermark wait failed");
        }
        if (j < top) {
            const long long need_rel = g0 + t - p->next_cap + 1;
            if (need_rel > 0 &&
                ops.wait(cs, (CUdeviceptr)p->rel, (cuuint64_t)need_rel, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
                return pipe_fail(p, RIDC_E_CUDA, "cuStreamWaitValue64 (release) failed");
        }
        TickParams tp;
        memset(&tp, 0, sizeof tp);
        tp.sv = ep.sv;
        tp.nact = 1;
        tp.level[0] = j;
        tp.target[0] = t;
        cudaError_t le = launch_chunk(p->pb.kind, p->ss.ccfg, std::min(p->nsm * chunk_ctas_per_sm(p->ss.ccfg, 1), items),
                                      p->stream, ep, tp, items,
                                      p->tm);
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

// One interval of a levels x shards rank (stream memops only).  Per step t
// (global step g): wait for the window -- my inbox interior from (j-1, s) and
// its ghost rows 0 / n+1 from (j-1, s-1) / (j-1, s+1) -- for my own ghost rows
// of step g-1 from (j, s-1) / (j, s+1), and for ring space at my three
// consumers; run the tick kernel on my rows (storing into (j+1, s)'s inbox);
// then deliver: my first / last row into the same-level neighbours' own ring
// (once they finished step g-1) and into the diagonal consumers' inbox ghost
// rows, raise every watermark, report step g done and release the producers'
// slots below my next window (LevelBuffer's protocol, engine.py:284-331, per
// neighbour).
int pipe_enqueue_shard(ridc_pipe* p, int interval, long long* launches)
{
    const DriverOps& ops = driver_ops();
    const int j = p->level, top = p->levels - 1;
    const long long g0 = (long long)interval * p->per;
    const EngineParams ep = pipe_params(p, g0);
    const int items = p->nrows * p->ss.sv.nseg;
    CUstream cs = reinterpret_cast<CUstream>(p->stream);
    const long long spin = (long long)(p->watchdog * 2.0e9);
    const size_t P = (size_t)p->ss.lay.P, rowb = P * sizeof(double);
    const size_t Vs = (size_t)p->Vs;
    const size_t vs_up = (size_t)p->up_rows * P, vs_dn = (size_t)p->dn_rows * P;
    auto word = [&](size_t off) { return reinterpret_cast<unsigned long long*>(p->mailbox + off); };
    auto wait = [&](const unsigned long long* f, long long v, bool remote) {
        return wait_value(p->stream, f, (unsigned long long)v, remote, p->can_flush, p->d_abort, spin) == cudaSuccess;
    };
    auto write = [&](unsigned long long* f, long long v) {
        return ops.write(cs, (CUdeviceptr)f, (cuuint64_t)v, CU_STREAM_WRITE_VALUE_DEFAULT) == CUDA_SUCCESS;
    };
    auto copy_row = [&](double* dst, const double* src) {
        return cudaMemcpyAsync(dst, src, rowb, cudaMemcpyDefault, p->stream) == cudaSuccess;
    };
    long long n = 0;
    for (long long t = 1; t <= p->per; ++t) {
        const long long g = g0 + t;
        if (j > 0) {
            const long long need = g0 + (t < j ? j : t);
            if (!wait(p->wm, need, p->prev_remote) || !wait(word(kWInUp), need, p->up_remote) ||
                !wait(word(kWInDn), need, p->dn_remote))
                return pipe_fail(p, RIDC_E_CUDA, "watermark wait failed");
        }
        if (t > 1 && (!wait(word(kWGhUp), g - 1, p->sup_remote) || !wait(word(kWGhDn), g - 1, p->sdn_remote)))
            return pipe_fail(p, RIDC_E_CUDA, "ghost-row wait failed");
        if (j < top) {
            const long long need_rel = g - p->next_cap + 1;
            if (need_rel > 0 && (!wait(p->rel, need_rel, false) || !wait(word(kWRelUp), need_rel, false) ||
                                 !wait(word(kWRelDn), need_rel, false)))
                return pipe_fail(p, RIDC_E_CUDA, "release wait failed");
        }
        TickParams tp;
        memset(&tp, 0, sizeof tp);
        tp.sv = ep.sv;
        tp.nact = 1;
        tp.level[0] = j;
        tp.target[0] = t;
        cudaError_t le = launch_chunk(p->pb.kind, p->ss.ccfg, std::min(p->nsm * chunk_ctas_per_sm(p->ss.ccfg, 1), items),
                                      p->stream, ep, tp, items, p->tm);
        if (le != cudaSuccess) return pipe_fail(p, RIDC_E_CUDA, std::string("tick launch: ") + cudaGetErrorString(le));
        ++n;
        const double* mine = p->own + (g % 2) * Vs;
        const double* first = mine + P, *last = mine + (size_t)p->nrows * P;
        // my boundary rows -> the same-level neighbours' own slot of step g (their ghost rows),
        // once each finished step g-1 (its last read of that slot's old content)
        if (t > 1 && (!wait(word(kWDoneUp), g - 1, p->sup_remote) || !wait(word(kWDoneDn), g - 1, p->sdn_remote)))
            return pipe_fail(p, RIDC_E_CUDA, "neighbour progress wait failed");
        if (!copy_row(p->side_up_own + (g % 2) * vs_up + (size_t)(p->up_rows - 1) * P, first) ||
            !copy_row(p->side_dn_own + (g % 2) * vs_dn, last) || !write(p->side_up_gh, g) || !write(p->side_dn_gh, g))
            return pipe_fail(p, RIDC_E_CUDA, "ghost-row delivery failed");
        if (j < top) {   // the diagonal consumers' inbox ghost rows, then every consumer's watermark
            const long long slot = g % p->next_cap;
            if (!copy_row(p->up_inbox + slot * vs_up + (size_t)(p->up_rows - 1) * P, first) ||
                !copy_row(p->dn_inbox + slot * vs_dn, last) || !write(p->up_in_wm, g) || !write(p->dn_in_wm, g) ||
                !write(p->next_wm, g))
                return pipe_fail(p, RIDC_E_CUDA, "inbox ghost-row delivery failed");
        }
        if (!write(p->side_up_done, g) || !write(p->side_dn_done, g))
            return pipe_fail(p, RIDC_E_CUDA, "progress write failed");
        if (j > 0) {
            const long long below = g0 + std::max(0LL, t + 1 - j);
            if (!write(p->prev_rel, below) || !write(p->prev_up_rel, below) || !write(p->prev_dn_rel, below))
                return pipe_fail(p, RIDC_E_CUDA, "release write failed");
        }
    }
    *launches = n;
    return RIDC_OK;
}

}  // namespace

extern "C" {

int64_t ridc_pipe_handle_bytes(void) { return (int64_t)sizeof(PipeBlob); }

static int pipe_create(const ridc_problem* gproblem, double t_start, double t_end, int32_t levels,
                       int64_t steps, int32_t restarts, const double* weights, int64_t nweights,
                       int32_t level, int32_t shard, int32_t nshards, int32_t device, int32_t inbox_capacity,
                       double watchdog_seconds, ridc_pipe** out)
{
    if (!out) return pipe_fail(nullptr, RIDC_E_CONFIG, "out is NULL");
    *out = nullptr;
    int rc = validate_problem(gproblem);
    if (rc) return rc;
    // a row shard computes its rows of the global grid as a local grid with one
    // ghost row per side (the tiling along x depends on nx and dt only)
    ridc_problem sub = *gproblem;
    int r0 = 0, nrows = gproblem->ny;
    if (nshards > 1) {
        if (gproblem->kind != RIDC_ADV_DIFF_2D && gproblem->kind != RIDC_REACTION_DIFFUSION_2D)
            return pipe_fail(nullptr, RIDC_E_CONFIG, "row shards need a 2-D kind (explicit in y)");
        if (nshards > gproblem->ny) return pipe_fail(nullptr, RIDC_E_CONFIG, "need 2 <= shards <= ny");
        if (shard < 0 || shard >= nshards) return pipe_fail(nullptr, RIDC_E_CONFIG, "shard out of range");
        r0 = (int)((long long)gproblem->ny * shard / nshards);
        nrows = (int)((long long)gproblem->ny * (shard + 1) / nshards) - r0;
        sub.ny = nrows + 2;
    }
    const ridc_problem* problem = &sub;
    if (levels < 1 || levels > kMaxLevels) return pipe_fail(nullptr, RIDC_E_CONFIG, "levels must be in 1..12");
    if (level < 0 || level >= levels) return pipe_fail(nullptr, RIDC_E_CONFIG, "level out of range");
    if (steps < 1 || restarts < 1 || steps % restarts)
        return pipe_fail(nullptr, RIDC_E_CONFIG, "steps must be a positive multiple of restarts");
    const long long per = steps / restarts;
    if (per < delay(levels) + 1) return pipe_fail(nullptr, RIDC_E_CONFIG, "restart interval shorter than the pipeline fill");
    if (!(t_start < t_end)) return pipe_fail(nullptr, RIDC_E_CONFIG, "need t_start < t_end");
    if (level > 0 && inbox_capacity > 0 && inbox_capacity < level + 3) {
        char buf[160];
        snprintf(buf, sizeof buf, "inbox_capacity %d too small for level %d: its window needs %d slots and "
                                  "the deferred publication 2 more (>= %d)", inbox_capacity, level, level + 1,
                 level + 3);
        return pipe_fail(nullptr, RIDC_E_CONFIG, buf);
    }
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
    p->shard = nshards > 1 ? shard : 0;
    p->nshards = nshards > 1 ? nshards : 1;
    p->r0 = r0;
    p->nrows = nrows;
    p->gny = gproblem->ny;
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
    // default: the greedy schedule's window (2j+5) + 8 slots of run-ahead, so a
    // producer rarely blocks on its consumer's release (or publishes early for it)
    p->inbox_cap = inbox_capacity > 0 ? inbox_capacity : 2LL * level + 13;
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
    if ((rc = make_chunk_solve(p->pb, p->dt, p->nsm, p->ss)) != RIDC_OK) {
        p->err = p->ss.err;
        return bail(rc);
    }
    prefer_two_per_sm(p->ss.ccfg, levels);   // the single-device engine's choice: bitwise the same states
    p->Vs = (long long)p->pb.ny * p->ss.lay.P;
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
    P_TRY(cudaMalloc(&p->d_cgeo, p->ss.cgeo.size() * sizeof(ChunkGeo)));
    P_TRY(cudaMemcpy(p->d_cgeo, p->ss.cgeo.data(), p->ss.cgeo.size() * sizeof(ChunkGeo), cudaMemcpyHostToDevice));
    P_TRY(cudaMalloc(&p->d_err, sizeof(unsigned long long)));
    P_TRY(cudaMalloc(&p->d_abort, sizeof(unsigned)));
    P_TRY(cudaMemset(p->d_abort, 0, sizeof(unsigned)));
    p->can_flush = device_can_flush_remote(device);
    // mailbox: flags, then the inbox ring (cap slots of ny padded rows); zeroed: Dirichlet ghosts
    // (a row shard's own 2-slot ring follows the inbox ring in the same
    // allocation: its neighbour shards deliver the own ghost rows through it)
    const size_t ring_bytes = (size_t)p->inbox_cap * p->Vs * sizeof(double);
    const size_t own_bytes = p->nshards > 1 ? (size_t)2 * p->Vs * sizeof(double) : 0;
    P_TRY(cudaMalloc(&p->mailbox, kFlagBytes + ring_bytes + own_bytes));
    P_TRY(cudaMemset(p->mailbox, 0, kFlagBytes + ring_bytes + own_bytes));
    p->wm = reinterpret_cast<unsigned long long*>(p->mailbox);
    p->rel = reinterpret_cast<unsigned long long*>(p->mailbox + 8);
    p->inbox = reinterpret_cast<double*>(p->mailbox + kFlagBytes);
    if (p->nshards > 1) {
        p->own = reinterpret_cast<double*>(p->mailbox + kFlagBytes + ring_bytes);
        P_TRY(cudaMalloc(&p->d_s0, (size_t)p->V * sizeof(double)));
    } else {
        P_TRY(cudaMalloc(&p->own_base, ((size_t)2 * p->Vs + 2 * p->V) * sizeof(double)));
        P_TRY(cudaMemset(p->own_base, 0, (size_t)2 * p->Vs * sizeof(double)));
        p->own = p->own_base;
    }
    memset(&p->tm, 0, sizeof p->tm);
    if ((rc = make_ring_map(&p->tm.map[level], p->own, p->Vs, 2, chunk_groups(p->ss.ccfg), &p->err)) != RIDC_OK)
        return bail(rc);
    if (level > 0 &&
        (rc = make_ring_map(&p->tm.map[level - 1], p->inbox, p->Vs, p->inbox_cap, chunk_groups(p->ss.ccfg), &p->err)) != RIDC_OK)
        return bail(rc);
    // resident level march: 1-D lines whose segments fit one co-resident CTA each
    if (levels >= 2 && p->nshards == 1 && p->ss.sv.nseg <= kPipeMaxSeg && res_geometry(p->pb, p->ss, p->rgeo) &&
        !(getenv("RIDC_NO_RESIDENT_LEVELS") && atoi(getenv("RIDC_NO_RESIDENT_LEVELS")) > 0)) {
        LevelsParams lp;
        memset(&lp, 0, sizeof lp);
        int per_sm = 0;
        const cudaError_t oe = levels_dispatch(p->pb.kind, p->ss.ccfg.nt, p->rgeo.mode, false, 0, p->stream, lp,
                                               p->tm, &per_sm, true);
        if (oe == cudaSuccess && per_sm * p->nsm >= p->ss.sv.nseg) {
            p->reslev_ok = p->reslev = true;
            p->reslev_mode = p->rgeo.mode;
            const int nseg = p->ss.sv.nseg;
            const std::vector<int>& d = p->rgeo.deps;
            P_TRY(cudaMalloc(&p->d_geo, 2 * d.size() * sizeof(int)));
            P_TRY(cudaMemcpy(p->d_geo, d.data(), d.size() * sizeof(int), cudaMemcpyHostToDevice));
            P_TRY(cudaMemcpy(p->d_geo + d.size(), p->rgeo.readers.data(), d.size() * sizeof(int),
                             cudaMemcpyHostToDevice));
            P_TRY(cudaMalloc(&p->d_lanes, (size_t)restarts * sizeof(LevelLane)));
            if (nseg > 1) {
                P_TRY(cudaMalloc(&p->d_lmail, 2 * (size_t)p->Vs * sizeof(uint4)));
                P_TRY(cudaMemset(p->d_lmail, 0, 2 * (size_t)p->Vs * sizeof(uint4)));
            }
        }
        cudaGetLastError();
    }
#undef P_TRY
    *out = p;
    return RIDC_OK;
}

int ridc_pipe_create(const ridc_problem* problem, double t_start, double t_end, int32_t levels,
                     int64_t steps, int32_t restarts, const double* weights, int64_t nweights,
                     int32_t level, int32_t device, int32_t inbox_capacity, double watchdog_seconds,
                     ridc_pipe** out)
{
    return pipe_create(problem, t_start, t_end, levels, steps, restarts, weights, nweights, level, 0, 1, device,
                       inbox_capacity, watchdog_seconds, out);
}

int ridc_pipe_create_shard(const ridc_problem* problem, double t_start, double t_end, int32_t levels,
                           int64_t steps, int32_t restarts, const double* weights, int64_t nweights,
                           int32_t level, int32_t shard, int32_t nshards, int32_t device,
                           int32_t inbox_capacity, double watchdog_seconds, ridc_pipe** out)
{
    if (nshards < 2) return pipe_fail(nullptr, RIDC_E_CONFIG, "need 2 <= shards <= ny");
    return pipe_create(problem, t_start, t_end, levels, steps, restarts, weights, nweights, level, shard, nshards,
                       device, inbox_capacity, watchdog_seconds, out);
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
    b.resident = p->reslev ? 1 : 0;
    b.shard = p->shard;
    b.nshards = p->nshards;
    b.rows = (int32_t)p->pb.ny;
    PIPE_TRY(p, cudaSetDevice(p->device));
    PIPE_TRY(p, cudaIpcGetMemHandle(&b.handle, p->mailbox));
    memcpy(blob, &b, sizeof b);
    return RIDC_OK;
}

static int open_blob(ridc_pipe* p, const void* blob, int want_level, char** base, int slot, long long* cap,
                     int* device)
{
    PipeBlob b;
    memcpy(&b, blob, sizeof b);
    if (b.magic != kBlobMagic || b.level != want_level || b.vs != p->Vs)
        return pipe_fail(p, RIDC_E_PROTOCOL, "pipeline handle from an incompatible rank");
    if ((b.resident != 0) != p->reslev)
        return pipe_fail(p, RIDC_E_CONFIG, "neighbour ranks disagree on the resident level march "
                                           "(ridc_pipe_set_resident before ridc_pipe_export on every rank)");
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
    *device = b.device;
    return RIDC_OK;
}

// A neighbour of a levels x shards rank: (want_level, want_shard) of the same
// grid.  Handles already opened by this rank (the two diagonal neighbours are
// one rank when there are two shards) are reused.
static int open_blob_shard(ridc_pipe* p, const void* blob, int want_level, int want_shard, int slot,
                           PipeBlob* out, char** base)
{
    PipeBlob b;
    memcpy(&b, blob, sizeof b);
    if (b.magic != kBlobMagic || b.level != want_level || b.shard != want_shard || b.nshards != p->nshards ||
        b.resident != 0 || b.vs != (int64_t)b.rows * p->ss.lay.P)
        return pipe_fail(p, RIDC_E_PROTOCOL, "levels x shards handle from an incompatible rank");
    if (b.pid == (int32_t)getpid()) {
        *base = reinterpret_cast<char*>((uintptr_t)b.direct);
        if (b.device != p->device) {
            cudaError_t e = cudaDeviceEnablePeerAccess(b.device, 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
                return pipe_fail(p, RIDC_E_CUDA, std::string("peer access: ") + cudaGetErrorString(e));
            cudaGetLastError();
        }
    } else {
        for (int k = 0; k < slot; ++k)   // same handle as an earlier neighbour
            if (p->opened[k] && p->opened_direct[k] == b.direct && p->opened_pid[k] == b.pid) {
                *base = reinterpret_cast<char*>(p->opened[k]);
                *out = b;
                return RIDC_OK;
            }
        void* ptr = nullptr;
        PIPE_TRY(p, cudaIpcOpenMemHandle(&ptr, b.handle, cudaIpcMemLazyEnablePeerAccess));
        p->opened[slot] = ptr;
        p->opened_direct[slot] = b.direct;
        p->opened_pid[slot] = b.pid;
        *base = reinterpret_cast<char*>(ptr);
    }
    *out = b;
    return RIDC_OK;
}

int ridc_pipe_connect_shard(ridc_pipe* p, const void* const* blobs)
{
    if (!p || !blobs) return pipe_fail(p, RIDC_E_CONFIG, "NULL argument");
    if (p->nshards < 2) return pipe_fail(p, RIDC_E_CONFIG, "not a row-shard rank (ridc_pipe_connect)");
    PIPE_TRY(p, cudaSetDevice(p->device));
    const int j = p->level, top = p->levels - 1, S = p->nshards;
    const int su = (p->shard + S - 1) % S, sd = (p->shard + 1) % S;
    for (int k = 0; k < 8; ++k) {
        const bool want = k < 3 ? j > 0 : k < 6 ? j < top : true;
        if (want != (blobs[k] != nullptr))
            return pipe_fail(p, RIDC_E_CONFIG, "shard rank needs exactly its existing neighbours");
    }
    int rc;
    PipeBlob b;
    char* base = nullptr;
    if (j > 0) {
        // (j-1, s): my inbox interior; its release counter
        if ((rc = open_blob_shard(p, blobs[0], j - 1, p->shard, 0, &b, &base)) != RIDC_OK) return rc;
        p->prev_remote = b.device != p->device;
        p->prev_rel = reinterpret_cast<unsigned long long*>(base + 8);
        // (j-1, s-1) delivers my inbox ghost row 0 (its last row); I release to its W_RELDN
        if ((rc = open_blob_shard(p, blobs[1], j - 1, su, 1, &b, &base)) != RIDC_OK) return rc;
        p->up_remote = b.device != p->device;
        p->prev_up_rel = reinterpret_cast<unsigned long long*>(base + kWRelDn);
        // (j-1, s+1) delivers my inbox ghost row n+1 (its first row); I release to its W_RELUP
        if ((rc = open_blob_shard(p, blobs[2], j - 1, sd, 2, &b, &base)) != RIDC_OK) return rc;
        p->dn_remote = b.device != p->device;
        p->prev_dn_rel = reinterpret_cast<unsigned long long*>(base + kWRelUp);
    }
    if (j < top) {
        if ((rc = open_blob_shard(p, blobs[3], j + 1, p->shard, 3, &b, &base)) != RIDC_OK) return rc;
        p->next_wm = reinterpret_cast<unsigned long long*>(base);
        p->next_inbox = reinterpret_cast<double*>(base + kFlagBytes);
        p->next_cap = b.inbox_cap;
        if ((rc = open_blob_shard(p, blobs[4], j + 1, su, 4, &b, &base)) != RIDC_OK) return rc;
        if (b.inbox_cap != p->next_cap) return pipe_fail(p, RIDC_E_CONFIG, "consumer shards disagree on inbox capacity");
        p->up_inbox = reinterpret_cast<double*>(base + kFlagBytes);
        p->up_in_wm = reinterpret_cast<unsigned long long*>(base + kWInDn);
        if ((rc = open_blob_shard(p, blobs[5], j + 1, sd, 5, &b, &base)) != RIDC_OK) return rc;
        if (b.inbox_cap != p->next_cap) return pipe_fail(p, RIDC_E_CONFIG, "consumer shards disagree on inbox capacity");
        p->dn_inbox = reinterpret_cast<double*>(base + kFlagBytes);
        p->dn_in_wm = reinterpret_cast<unsigned long long*>(base + kWInUp);
    }
    // (j, s-1) / (j, s+1): own ghost rows both ways, and step-done counters
    if ((rc = open_blob_shard(p, blobs[6], j, su, 6, &b, &base)) != RIDC_OK) return rc;
    p->sup_remote = b.device != p->device;
    p->side_up_own = reinterpret_cast<double*>(base + kFlagBytes + (size_t)b.inbox_cap * b.vs * sizeof(double));
    p->side_up_gh = reinterpret_cast<unsigned long long*>(base + kWGhDn);
    p->side_up_done = reinterpret_cast<unsigned long long*>(base + kWDoneDn);
    p->up_rows = b.rows;   // shard s-1's local rows (its ranks of every level)
    if ((rc = open_blob_shard(p, blobs[7], j, sd, 7, &b, &base)) != RIDC_OK) return rc;
    p->sdn_remote = b.device != p->device;
    p->side_dn_own = reinterpret_cast<double*>(base + kFlagBytes + (size_t)b.inbox_cap * b.vs * sizeof(double));
    p->side_dn_gh = reinterpret_cast<unsigned long long*>(base + kWGhUp);
    p->side_dn_done = reinterpret_cast<unsigned long long*>(base + kWDoneUp);
    p->dn_rows = b.rows;
    return RIDC_OK;
}

int ridc_pipe_reset(ridc_pipe* p)
{
    if (!p) return pipe_fail(nullptr, RIDC_E_CONFIG, "NULL pipe");
    PIPE_TRY(p, cudaSetDevice(p->device));
    PIPE_TRY(p, cudaStreamSynchronize(p->stream));
    PIPE_TRY(p, cudaMemset(p->mailbox, 0, kFlagBytes));
    return RIDC_OK;
}

int ridc_pipe_connect(ridc_pipe* p, const void* prev_blob, const void* next_blob)
{
    if (!p) return pipe_fail(nullptr, RIDC_E_CONFIG, "NULL pipe");
    if (p->nshards > 1) return pipe_fail(p, RIDC_E_CONFIG, "row-shard rank: use ridc_pipe_connect_shard");
    PIPE_TRY(p, cudaSetDevice(p->device));
    const int j = p->level, top = p->levels - 1;
    if ((j > 0) != (prev_blob != nullptr) || (j < top) != (next_blob != nullptr))
        return pipe_fail(p, RIDC_E_CONFIG, "level needs exactly its existing neighbours");
    int rc;
    long long cap = 0;
    char* base = nullptr;
    if (prev_blob) {
        int pdev = p->device;
        if ((rc = open_blob(p, prev_blob, j - 1, &base, 0, &cap, &pdev)) != RIDC_OK) return rc;
        p->prev_remote = pdev != p->device;
        p->prev_rel = reinterpret_cast<unsigned long long*>(base + 8);
        p->in_rel = reinterpret_cast<unsigned long long*>(base + kRelOff);
    }
    if (next_blob) {
        int ndev = p->device;
        if ((rc = open_blob(p, next_blob, j + 1, &base, 1, &cap, &ndev)) != RIDC_OK) return rc;
        p->next_wm = reinterpret_cast<unsigned long long*>(base);
        p->next_inbox = reinterpret_cast<double*>(base + kFlagBytes);
        p->next_cap = cap;
        p->out_pub = reinterpret_cast<unsigned long long*>(base + kPubOff);
    }
    if (p->reslev) {   // one lane per interval: slots and offsets follow the global step numbers
        std::vector<LevelLane> lanes(p->restarts);
        for (int r = 0; r < p->restarts; ++r) {
            const long long g0 = (long long)r * p->per;
            LevelLane& ln = lanes[r];
            memset(&ln, 0, sizeof ln);
            ln.level = j;
            ln.in_map = j > 0 ? j - 1 : 0;
            ln.own0 = p->own + (g0 % 2) * p->Vs;
            ln.fin = p->own + ((g0 + p->per) % 2) * p->Vs;
            ln.in_off = g0;
            ln.in_cap = p->inbox_cap;
            ln.in_pub = reinterpret_cast<unsigned long long*>(p->mailbox + kPubOff);
            ln.in_rel = p->in_rel;
            ln.out = j < top ? p->next_inbox : nullptr;
            ln.out_off = g0;
            ln.out_cap = p->next_cap;
            ln.out_pub = p->out_pub;
            ln.out_rel = reinterpret_cast<unsigned long long*>(p->mailbox + kRelOff);
            ln.mail = p->d_lmail;
        }
        PIPE_TRY(p, cudaMemcpy(p->d_lanes, lanes.data(), lanes.size() * sizeof(LevelLane), cudaMemcpyHostToDevice));
    }
    return RIDC_OK;
}

int ridc_pipe_run_interval(ridc_pipe* p, int32_t interval, const double* state0_dev, double* final_dev,
                           double* wall_seconds)
{
    NvtxRange nvtx_("ridc.pipe_interval");
    if (!p || !state0_dev || !final_dev) return pipe_fail(p, RIDC_E_CONFIG, "NULL argument");
    if (interval < 0 || interval >= p->restarts) return pipe_fail(p, RIDC_E_CONFIG, "interval out of range");
    const int j = p->level, top = p->levels - 1;
    if ((j > 0 && !p->prev_rel) || (j < top && !p->next_inbox) || (p->nshards > 1 && !p->side_up_own))
        return pipe_fail(p, RIDC_E_CONFIG, "pipeline rank not connected");
    PIPE_TRY(p, cudaSetDevice(p->device));
    const long long g0 = (long long)interval * p->per;
    if (p->nshards > 1) {
        // a row shard seeds from global rows r0-1 .. r0+nrows (periodic in y)
        const size_t rb = (size_t)p->pb.nx * sizeof(double);
        for (int lr = 0; lr < p->nrows + 2; ++lr) {
            const int gr = ((p->r0 - 1 + lr) % p->gny + p->gny) % p->gny;
            PIPE_TRY(p, cudaMemcpyAsync(p->d_s0 + (size_t)lr * p->pb.nx, state0_dev + (size_t)gr * p->pb.nx, rb,
                                        cudaMemcpyDeviceToDevice, p->stream));
        }
        state0_dev = p->d_s0;
    }
    // seed: step g0 of my own ring and of my inbox is the interval's state0
    // (plain state -> padded rows with periodic ghosts)
    EngineParams ep = pipe_params(p, g0);
    {
        EngineParams sp = ep;
        for (int k = 0; k < kMaxLevels; ++k) sp.ring[k] = nullptr;
        sp.ring[j] = ep.ring[j];
        if (j > 0) sp.ring[j - 1] = ep.ring[j - 1];
        const int sb = (int)std::min<long long>((p->Vs + 255) / 256, 148 * 8);
        k_seed_chunk<<<sb, 256, 0, p->stream>>>(state0_dev, sp, g0);
        PIPE_TRY(p, cudaGetLastError());
    }
    PIPE_TRY(p, cudaMemsetAsync(p->d_err, 0xff, sizeof(unsigned long long), p->stream));
    PIPE_TRY(p, cudaMemsetAsync(p->d_abort, 0, sizeof(unsigned), p->stream));
    PIPE_TRY(p, cudaEventRecord(p->ev0, p->stream));
    // the interval's ops: captured into a graph on first use (memops included)
    auto it = p->graphs.find(interval);
    long long launches = 0;
    if (p->reslev) {
        const int nseg = p->ss.sv.nseg;
        if (p->tag_next + (unsigned long long)p->per + 2 >= 0xffffffffull) {
            if (p->d_lmail) PIPE_TRY(p, cudaMemsetAsync(p->d_lmail, 0, 2 * (size_t)p->Vs * sizeof(uint4), p->stream));
            p->tag_next = 1;
        }
        LevelsParams lp;
        memset(&lp, 0, sizeof lp);
        lp.pb = p->pb;
        lp.sv = p->ss.sv;
        lp.lay = p->ss.lay;
        lp.cgeo = p->d_cgeo;
        lp.lanes = p->d_lanes + interval;
        lp.deps = p->d_geo;
        lp.readers = p->d_geo + p->rgeo.deps.size();
        lp.weights = p->d_weights;
        for (int k = 0; k < kMaxLevels; ++k) {
            lp.steady_off[k] = p->st[k];
            lp.startup_off[k] = p->su[k];
        }
        lp.dt = p->dt;
        lp.per = p->per;
        lp.Vs = p->Vs;
        lp.epoch = ++p->lepoch;   // every rank runs its intervals in the same order: epochs agree
        lp.tag0 = p->tag_next;
        p->tag_next += (unsigned)p->per + 1;
        lp.edge_w = p->rgeo.edge_w;
        lp.pub_every = env_int("RIDC_PUB_EVERY", 4);
        lp.err = p->d_err;
        lp.abort = p->d_abort;
        lp.spin_limit = (long long)(p->watchdog * 2.0e9);
        const cudaError_t le = levels_dispatch(p->pb.kind, p->ss.ccfg.nt, p->reslev_mode, true, nseg, p->stream,
                                               lp, p->tm, nullptr, true);
        if (le != cudaSuccess)
            return pipe_fail(p, RIDC_E_CUDA, std::string("resident level march launch: ") + cudaGetErrorString(le));
        launches = 1;
    } else if (it == p->graphs.end()) {
        cudaGraph_t graph = nullptr;
        cudaGraphExec_t exec = nullptr;
        bool captured = false;
        if (cudaStreamBeginCapture(p->stream, cudaStreamCaptureModeThreadLocal) == cudaSuccess) {
            int rc = p->nshards > 1 ? pipe_enqueue_shard(p, interval, &launches) : pipe_enqueue(p, interval, &launches);
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
            int rc = p->nshards > 1 ? pipe_enqueue_shard(p, interval, &launches)
                                    : pipe_enqueue(p, interval, &launches);   // direct enqueue fallback
            if (rc) return rc;
        }
    } else {
        PIPE_TRY(p, cudaGraphLaunch(it->second, p->stream));
        launches = p->per;
    }
    p->launches = launches;
    {
        const ChunkLayout& Ly = p->ss.lay;
        const double* fin = ep.ring[j] + ((ep.off[j] + p->per) % 2) * p->Vs;
        const int r_first = p->nshards > 1 ? 1 : 0, nr = p->nshards > 1 ? p->nrows : (int)p->pb.ny;
        PIPE_TRY(p, cudaMemcpy2DAsync(final_dev, (size_t)p->pb.nx * sizeof(double), fin + (size_t)r_first * Ly.P + Ly.GW,
                                      (size_t)Ly.P * sizeof(double), (size_t)p->pb.nx * sizeof(double),
                                      (size_t)nr, cudaMemcpyDeviceToDevice, p->stream));
    }
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
    {   // in-kernel waits (resident march, or k_wait_flag on a remote producer) that timed out
        unsigned ab = 0;
        PIPE_TRY(p, cudaMemcpy(&ab, p->d_abort, sizeof ab, cudaMemcpyDeviceToHost));
        if (ab) {
            char buf[160];
            snprintf(buf, sizeof buf, "pipeline made no progress within %gs; waiting levels: %d@interval%d",
                     p->watchdog, j, interval);
            return pipe_fail(p, RIDC_E_PROTOCOL, buf);
        }
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
    info->kernel_launches = p->reslev ? 1 : p->per;   /* per interval */
    info->tile = p->ss.sv.tile;
    info->halo = p->ss.sv.halo;
    info->items_per_level = p->pb.ny * p->ss.sv.nseg;
    info->threads = p->ss.ccfg.nt;
    info->ring_vectors = 2 + (p->level > 0 ? p->inbox_cap : 0);
    info->lambda = p->ss.sv.lam;
    info->r = p->ss.r;
    info->path = p->reslev ? RIDC_PATH_RESIDENT_LEVELS : RIDC_PATH_TICK;
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
    if (p->d_s0) cudaFree(p->d_s0);
    if (p->d_weights) cudaFree(p->d_weights);
    if (p->d_tab) cudaFree(p->d_tab);
    if (p->d_cgeo) cudaFree(p->d_cgeo);
    if (p->d_err) cudaFree(p->d_err);
    if (p->d_geo) cudaFree(p->d_geo);
    if (p->d_lmail) cudaFree(p->d_lmail);
    if (p->d_abort) cudaFree(p->d_abort);
    if (p->d_lanes) cudaFree(p->d_lanes);
    if (p->ev0) cudaEventDestroy(p->ev0);
    if (p->ev1) cudaEventDestroy(p->ev1);
    if (p->stream) cudaStreamDestroy(p->stream);
    delete p;
    return RIDC_OK;
}

int ridc_pipe_set_resident(ridc_pipe* p, int32_t enable)
{
    if (!p) return pipe_fail(nullptr, RIDC_E_CONFIG, "NULL pipe");
    p->reslev = enable && p->reslev_ok;
    return RIDC_OK;
}

int ridc_pipe_resident(const ridc_pipe* p) { return p && p->reslev ? 1 : 0; }

const char* ridc_pipe_last_error(const ridc_pipe* p)
{
    if (p && !p->err.empty()) return p->err.c_str();
    return g_last_error.c_str();
}

}  // extern "C"

// ================================================================ ARK (IMEX) steps
//
// The paper's comparators (steppers.ark_step / integrate_ark, steppers.py:122-155;
// tableaus.py imex3/imex4) on the same device machinery as the RIDC levels.
// Stage i's right-hand side  y_n + dt sum_{j<i} (aI_ij f^S(Y_j) + aE_ij f^N(Y_j))
// (kernels.stage_accumulate, kernels.py:149-158) is exactly a window item:
// node Y_j with weights (ca, cs, cn) = (j == 0 ? 1 : 0, dt aI_ij, dt aE_ij),
// f^S / f^N recomputed from the stored stage states by the stencils; the
// stage solve (I - aI_ii dt L_S) uses that stage's own factors (identity
// factors lam = 0, g = 1 when aI_ii = 0 and for the final combination).
// One tiling serves every stage: it is built for the largest shift, whose
// truncation halo bounds all the others.  One tick-kernel launch per stage,
// the whole march captured in one CUDA graph.

namespace {

struct ArkSolve {
    DevSolve sv;
    double* d_tab = nullptr;
};

}  // namespace

struct ridc_ark_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    DevProblem pb;
    SolveSetup ss;             // tiling + layout (largest shift)
    int nsm = 148;
    int stages = 0;
    long long steps = 0;
    double dt = 0;
    long long V = 0, Vs = 0, cap = 0;
    double* d_ring = nullptr;  // slots: y (2, alternating by step parity), stage states Y_i at 2 + i
    ChunkGeo* d_cgeo = nullptr;
    StepItem* d_items = nullptr;   // [parity][item]
    int nitems = 0;
    std::vector<ArkSolve> solves;  // per item
    double* d_y0 = nullptr;
    unsigned long long* d_err = nullptr;
    EngineParams ep;
    TmapSet tm;
    cudaGraphExec_t gexec = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    long long launches = 0;
    // the carry-exchange tick for every stage (periodic RD lines of 512-point chunks)
    bool carrylev = false;
    int cl_grid = 0, cl_wpc = 0, cl_k = 16;
    std::vector<CarryLevParams> clp;   // per item: the stage's solve
    TmapSet tm_cl;
    uint4* d_clx = nullptr;
    unsigned* d_clepoch = nullptr;
    unsigned* d_abort = nullptr;
    double watchdog = 30.0;
    std::string err;
};

namespace {

int ark_fail(ridc_ark_ctx* a, int code, const std::string& m) { return fail(a ? &a->err : nullptr, code, m); }

// Identity "solve": lam = 0, g = 1 makes both recurrences and every carry exact copies.
DevSolve identity_solve(const DevSolve& tiling)
{
    DevSolve sv;
    memset(&sv, 0, sizeof sv);
    sv.lam = 0.0;
    sv.g = 1.0;
    sv.halo = tiling.halo;
    sv.tile = tiling.tile;
    sv.nseg = tiling.nseg;
    return sv;
}

}  // namespace

extern "C" {

int ridc_ark_create(const ridc_problem* problem, double t_start, double t_end, int64_t steps, int32_t stages,
                    const double* a_implicit, const double* a_explicit, const double* b_implicit,
                    const double* b_explicit, int32_t device, ridc_ark_ctx** out)
{
    if (!out) return fail(nullptr, RIDC_E_CONFIG, "out is NULL");
    *out = nullptr;
    int rc = validate_problem(problem);
    if (rc) return rc;
    if (steps < 1) return fail(nullptr, RIDC_E_CONFIG, "steps must be positive");
    if (!(t_start < t_end)) return fail(nullptr, RIDC_E_CONFIG, "need t_start < t_end");
    if (stages < 1 || stages + 1 > kMaxNodes)
        return fail(nullptr, RIDC_E_CONFIG, "ARK stage count out of range");
    if (!a_implicit || !a_explicit || !b_implicit || !b_explicit)
        return fail(nullptr, RIDC_E_CONFIG, "NULL tableau");
    const int s = stages;
    for (int i = 0; i < s; ++i)
        for (int j = 0; j < s; ++j) {
            if (j > i && a_implicit[i * s + j] != 0.0)
                return fail(nullptr, RIDC_E_CONFIG, "a_implicit must be lower triangular");
            if (j >= i && a_explicit[i * s + j] != 0.0)
                return fail(nullptr, RIDC_E_CONFIG, "a_explicit must be strictly lower triangular");
        }
    ridc_ark_ctx* a = new ridc_ark_ctx();
    auto bail = [&](int code) {
        std::string m = a->err.empty() ? g_last_error : a->err;
        ridc_ark_destroy(a);
        g_last_error = m;
        return code;
    };
#define ARK_TRY(expr)                                                                        \
    do {                                                                                     \
        cudaError_t _e = (expr);                                                             \
        if (_e != cudaSuccess) {                                                             \
            a->err = std::string(#expr " failed: ") + cudaGetErrorString(_e);               \
            return bail(RIDC_E_CUDA);                                                        \
        }                                                                                    \
    } while (0)
    a->device = device;
    a->pb = make_problem(problem);
    a->stages = s;
    a->steps = steps;
    a->dt = (t_end - t_start) / (double)steps;   // integrate_ark: uniform dt
    a->V = (long long)problem->nx * problem->ny;
    if (cudaSetDevice(device) != cudaSuccess) {
        a->err = "cudaSetDevice failed";
        return bail(RIDC_E_CUDA);
    }
    if (cudaDeviceGetAttribute(&a->nsm, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) a->nsm = 148;
    double amax = 0.0;
    for (int i = 0; i < s; ++i) amax = std::max(amax, a_implicit[i * s + i]);
    if ((rc = make_chunk_solve(a->pb, amax * a->dt, a->nsm, a->ss)) != RIDC_OK) {
        a->err = a->ss.err;
        return bail(rc);
    }
    prefer_two_per_sm(a->ss.ccfg, 1);
    a->Vs = (long long)a->pb.ny * a->ss.lay.P;
    a->cap = 2 + s;
    ARK_TRY(cudaStreamCreateWithFlags(&a->stream, cudaStreamNonBlocking));
    ARK_TRY(cudaEventCreate(&a->ev0));
    ARK_TRY(cudaEventCreate(&a->ev1));
    ARK_TRY(cudaMalloc(&a->d_ring, (size_t)a->cap * a->Vs * sizeof(double)));
    ARK_TRY(cudaMemset(a->d_ring, 0, (size_t)a->cap * a->Vs * sizeof(double)));   // Dirichlet ghosts stay 0
    ARK_TRY(cudaMalloc(&a->d_cgeo, a->ss.cgeo.size() * sizeof(ChunkGeo)));
    ARK_TRY(cudaMemcpy(a->d_cgeo, a->ss.cgeo.data(), a->ss.cgeo.size() * sizeof(ChunkGeo), cudaMemcpyHostToDevice));
    ARK_TRY(cudaMalloc(&a->d_y0, (size_t)a->V * sizeof(double)));
    ARK_TRY(cudaMalloc(&a->d_err, sizeof(unsigned long long)));
    memset(&a->tm, 0, sizeof a->tm);
    if ((rc = make_ring_map(&a->tm.map[0], a->d_ring, a->Vs, a->cap, chunk_groups(a->ss.ccfg), &a->err)) != RIDC_OK)
        return bail(rc);
    EngineParams& ep = a->ep;
    memset(&ep, 0, sizeof ep);
    ep.pb = a->pb;
    ep.sv = a->ss.sv;
    ep.V = a->V;
    ep.Vs = a->Vs;
    ep.dt = a->dt;
    ep.levels = 1;
    ep.ring[0] = a->d_ring;
    ep.cap[0] = a->cap;
    ep.err = a->d_err;
    ep.lay = a->ss.lay;
    ep.cgeo = a->d_cgeo;

    // ---- the items of one step: stages with a nonzero diagonal or i > 0, then the final
    // combination.  Y_0 aliases y_n when aI_00 = 0 (both paper tableaus).
    const bool y0_alias = a_implicit[0] == 0.0;
    auto slot_of_stage = [&](int j, int parity) -> long long { return (j == 0 && y0_alias) ? parity : 2 + j; };
    std::vector<int> item_stage;   // stage index, s = final
    for (int i = (y0_alias ? 1 : 0); i < s; ++i) item_stage.push_back(i);
    item_stage.push_back(s);
    a->nitems = (int)item_stage.size();
    std::vector<StepItem> items(2 * a->nitems);
    for (int parity = 0; parity < 2; ++parity)
        for (int k = 0; k < a->nitems; ++k) {
            const int i = item_stage[k];
            const bool fin = i == s;
            StepItem& it = items[parity * a->nitems + k];
            memset(&it, 0, sizeof it);
            it.level = fin ? 0 : 1;   // non-finite word: the final store of a step reports first
            it.target = 0;            // the step number arrives per launch (TickParams.target)
            int nn = 0;
            auto add = [&](long long slot, double ca, double cs, double cn) {
                it.vec[nn] = a->d_ring + slot * a->Vs;
                it.vlev[nn] = 0;
                it.vslot[nn] = slot;
                it.ca[nn] = ca;
                it.cs[nn] = cs;
                it.cn[nn] = cn;
                ++nn;
            };
            // y_n itself (ca = 1), merged with Y_0's stencil weights when Y_0 aliases it
            const double* rs = fin ? b_implicit : a_implicit + i * s;
            const double* rn = fin ? b_explicit : a_explicit + i * s;
            const int upto = fin ? s : i;
            if (y0_alias) add(parity, 1.0, upto > 0 ? a->dt * rs[0] : 0.0, upto > 0 ? a->dt * rn[0] : 0.0);
            else add(parity, 1.0, 0.0, 0.0);
            for (int j = y0_alias ? 1 : 0; j < upto; ++j)
                if (rs[j] != 0.0 || rn[j] != 0.0) add(slot_of_stage(j, parity), 0.0, a->dt * rs[j], a->dt * rn[j]);
            it.nnodes = nn;
            const long long oslot = fin ? 1 - parity : slot_of_stage(i, parity);
            it.out = a->d_ring + oslot * a->Vs;
            it.out2 = nullptr;
        }
    // ---- per-item solves
    a->solves.resize(a->nitems);
    for (int k = 0; k < a->nitems; ++k) {
        const int i = item_stage[k];
        const double aii = i < s ? a_implicit[i * s + i] : 0.0;
        ArkSolve& as = a->solves[k];
        if (aii == 0.0) {
            as.sv = identity_solve(a->ss.sv);
            continue;
        }
        SolveSetup st;
        make_factors(a->pb, aii * a->dt, st);
        as.sv = st.sv;
        as.sv.halo = a->ss.sv.halo;
        as.sv.tile = a->ss.sv.tile;
        as.sv.nseg = a->ss.sv.nseg;
        if (!st.tab.empty()) {
            ARK_TRY(cudaMalloc(&as.d_tab, st.tab.size() * sizeof(double)));
            ARK_TRY(cudaMemcpy(as.d_tab, st.tab.data(), st.tab.size() * sizeof(double), cudaMemcpyHostToDevice));
            as.sv.tab_m = as.d_tab;
            as.sv.tab_g = as.d_tab + as.sv.ntab;
        }
    }
    ARK_TRY(cudaMalloc(&a->d_items, items.size() * sizeof(StepItem)));
    ARK_TRY(cudaMemcpy(a->d_items, items.data(), items.size() * sizeof(StepItem), cudaMemcpyHostToDevice));

    // ---- the carry-exchange tick (ridc_carry_levels.cuh) for every stage where
    // the line qualifies: periodic RD, 512-point chunks, the stiffest stage's
    // carry reach <= 512
    {
        const bool off = getenv("RIDC_NO_CARRYLEV") && atoi(getenv("RIDC_NO_CARRYLEV")) > 0;
        const int kp = (a->pb.kind == RD_1D && a->pb.ny == 1) ? carry_lev_k(a->pb.nx, halo_of(a->ss.sv.lam), a->nsm) : 0;
        const int nchunk = kp ? a->pb.nx / (32 * kp) : 0;
        if (!off && kp && a->ss.lay.GW >= 16 && (long long)steps * a->nitems < 0x7fffffffLL) {
            a->cl_k = kp;
            const int grid = std::min(a->nsm, nchunk), wpc = (nchunk + grid - 1) / grid;
            const size_t xb = (size_t)2 * kMaxLevels * nchunk * sizeof(uint4);
            ARK_TRY(cudaMalloc(&a->d_clx, xb));
            ARK_TRY(cudaMemset(a->d_clx, 0, xb));
            ARK_TRY(cudaMalloc(&a->d_clepoch, sizeof(unsigned)));
            ARK_TRY(cudaMemset(a->d_clepoch, 0, sizeof(unsigned)));
            ARK_TRY(cudaMalloc(&a->d_abort, sizeof(unsigned)));
            ARK_TRY(cudaMemset(a->d_abort, 0, sizeof(unsigned)));
            a->clp.resize(a->nitems);
            for (int k = 0; k < a->nitems; ++k) {
                CarryLevParams& cp = a->clp[k];
                memset(&cp, 0, sizeof cp);
                fill_carry_lev(cp, a->solves[k].sv, a->cl_k);
                cp.nx = a->pb.nx;
                cp.GW = a->ss.lay.GW;
                cp.gdata = a->ss.lay.gdata;
                cp.nchunk = nchunk;
                cp.wpc = wpc;
                cp.xch = a->d_clx;
                cp.epoch = a->d_clepoch;
                cp.ticks = (unsigned)(steps * a->nitems + 1);
                cp.abort = a->d_abort;
                cp.spin_limit = (long long)(a->watchdog * 2.0e9);
            }
            memset(&a->tm_cl, 0, sizeof a->tm_cl);
            if ((rc = make_ring_map(&a->tm_cl.map[0], a->d_ring, a->Vs, a->cap, kClBoxGroups, &a->err)) != RIDC_OK)
                return bail(rc);
            a->cl_grid = (nchunk + wpc - 1) / wpc;
            a->cl_wpc = wpc;
            a->carrylev = true;
        }
    }

    // ---- capture: seed y_0 into slot 0, then per step one launch per item
    const int tiles = a->pb.ny * a->ss.sv.nseg;
    cudaGraph_t graph = nullptr;
    ARK_TRY(cudaStreamBeginCapture(a->stream, cudaStreamCaptureModeThreadLocal));
    cudaError_t le = cudaSuccess;
    long long launches = 0;
    if (a->carrylev) {   // a fresh tag epoch for the exchange lines of this run
        k_bump_epoch<<<1, 1, 0, a->stream>>>(a->d_clepoch);
        le = cudaGetLastError();
        ++launches;
    }
    const int sb = (int)std::min<long long>((a->Vs + 255) / 256, 148 * 8);
    if (le == cudaSuccess) {
        k_seed_chunk<<<sb, 256, 0, a->stream>>>(a->d_y0, ep, -1);
        le = cudaGetLastError();
    }
    ++launches;
    for (long long n = 0; n < steps && le == cudaSuccess; ++n) {
        const int parity = (int)(n & 1);
        for (int k = 0; k < a->nitems && le == cudaSuccess; ++k) {
            TickParams tp;
            memset(&tp, 0, sizeof tp);
            tp.nact = 1;
            tp.sv = a->solves[k].sv;
            tp.pre = a->d_items + parity * a->nitems + k;
            tp.target[0] = n + 1;
            if (a->carrylev)
                le = carry_levels_k<RD_1D>(a->cl_grid, a->cl_wpc, a->cl_k, a->stream, ep, tp, a->clp[k], a->tm_cl,
                                           (unsigned)(n * a->nitems + k + 1));
            else
                le = launch_chunk(a->pb.kind, a->ss.ccfg, std::min(a->nsm * chunk_ctas_per_sm(a->ss.ccfg, 1), tiles),
                                  a->stream, ep, tp, tiles, a->tm);
            ++launches;
        }
    }
    cudaError_t ce = cudaStreamEndCapture(a->stream, &graph);
    if (le != cudaSuccess) {
        if (graph) cudaGraphDestroy(graph);
        a->err = std::string("ARK launch during capture: ") + cudaGetErrorString(le);
        return bail(RIDC_E_CUDA);
    }
    ARK_TRY(ce);
    cudaError_t ie = cudaGraphInstantiate(&a->gexec, graph, 0);
    cudaGraphDestroy(graph);
    ARK_TRY(ie);
    a->launches = launches;
#undef ARK_TRY
    *out = a;
    return RIDC_OK;
}

static int ark_march(ridc_ark_ctx* a, double* wall_seconds)
{
    CUDA_TRY(&a->err, cudaMemsetAsync(a->d_err, 0xff, sizeof(unsigned long long), a->stream));
    if (a->d_abort) CUDA_TRY(&a->err, cudaMemsetAsync(a->d_abort, 0, sizeof(unsigned), a->stream));
    CUDA_TRY(&a->err, cudaEventRecord(a->ev0, a->stream));
    CUDA_TRY(&a->err, cudaGraphLaunch(a->gexec, a->stream));
    CUDA_TRY(&a->err, cudaEventRecord(a->ev1, a->stream));
    CUDA_TRY(&a->err, cudaEventSynchronize(a->ev1));
    if (wall_seconds) {
        float ms = 0.f;
        CUDA_TRY(&a->err, cudaEventElapsedTime(&ms, a->ev0, a->ev1));
        *wall_seconds = ms * 1e-3;
    }
    if (a->d_abort) {
        unsigned ab = 0;
        CUDA_TRY(&a->err, cudaMemcpy(&ab, a->d_abort, sizeof ab, cudaMemcpyDeviceToHost));
        if (ab) return ark_fail(a, RIDC_E_PROTOCOL, "ARK march: a neighbour chunk's carry wait timed out");
    }
    unsigned long long w = 0;
    CUDA_TRY(&a->err, cudaMemcpy(&w, a->d_err, sizeof w, cudaMemcpyDeviceToHost));
    if (w != ULLONG_MAX) {
        char buf[128];
        snprintf(buf, sizeof buf, "ARK march produced non-finite entries at step %lld", (long long)(w >> 8));
        return ark_fail(a, RIDC_E_NONFINITE, buf);   // steppers.py:153-154
    }
    return RIDC_OK;
}

static const double* ark_final(const ridc_ark_ctx* a) { return a->d_ring + (a->steps & 1) * a->Vs; }

int ridc_ark_run(ridc_ark_ctx* a, const double* y0_host, double* final_host, double* wall_seconds)
{
    NvtxRange nvtx_("ridc.ark_run");
    if (!a || !y0_host || !final_host) return ark_fail(a, RIDC_E_CONFIG, "NULL argument");
    CUDA_TRY(&a->err, cudaSetDevice(a->device));
    CUDA_TRY(&a->err, cudaMemcpyAsync(a->d_y0, y0_host, (size_t)a->V * sizeof(double), cudaMemcpyHostToDevice,
                                      a->stream));
    int rc = ark_march(a, wall_seconds);
    if (rc) return rc;
    const ChunkLayout& L = a->ss.lay;
    CUDA_TRY(&a->err, cudaMemcpy2DAsync(final_host, (size_t)a->pb.nx * sizeof(double), ark_final(a) + L.GW,
                                        (size_t)L.P * sizeof(double), (size_t)a->pb.nx * sizeof(double),
                                        (size_t)a->pb.ny, cudaMemcpyDeviceToHost, a->stream));
    CUDA_TRY(&a->err, cudaStreamSynchronize(a->stream));
    return RIDC_OK;
}

int ridc_ark_run_device(ridc_ark_ctx* a, const double* y0_dev, double* final_dev, double* wall_seconds)
{
    NvtxRange nvtx_("ridc.ark_run_device");
    if (!a || !y0_dev || !final_dev) return ark_fail(a, RIDC_E_CONFIG, "NULL argument");
    CUDA_TRY(&a->err, cudaSetDevice(a->device));
    CUDA_TRY(&a->err, cudaMemcpyAsync(a->d_y0, y0_dev, (size_t)a->V * sizeof(double), cudaMemcpyDeviceToDevice,
                                      a->stream));
    int rc = ark_march(a, wall_seconds);
    if (rc) return rc;
    const ChunkLayout& L = a->ss.lay;
    CUDA_TRY(&a->err, cudaMemcpy2DAsync(final_dev, (size_t)a->pb.nx * sizeof(double), ark_final(a) + L.GW,
                                        (size_t)L.P * sizeof(double), (size_t)a->pb.nx * sizeof(double),
                                        (size_t)a->pb.ny, cudaMemcpyDeviceToDevice, a->stream));
    CUDA_TRY(&a->err, cudaStreamSynchronize(a->stream));
    return RIDC_OK;
}

int ridc_ark_info(const ridc_ark_ctx* a, int64_t* kernel_launches, int32_t* items_per_step)
{
    if (!a) return fail(nullptr, RIDC_E_CONFIG, "NULL argument");
    if (kernel_launches) *kernel_launches = a->launches;
    if (items_per_step) *items_per_step = a->nitems;
    return RIDC_OK;
}

int ridc_ark_path(const ridc_ark_ctx* a)
{
    if (!a) {
        fail(nullptr, RIDC_E_CONFIG, "NULL argument");
        return -1;
    }
    return a->carrylev ? RIDC_PATH_CARRY_LEVELS : RIDC_PATH_TICK;
}

int ridc_ark_destroy(ridc_ark_ctx* a)
{
    if (!a) return RIDC_OK;
    cudaSetDevice(a->device);
    if (a->stream) cudaStreamSynchronize(a->stream);
    if (a->gexec) cudaGraphExecDestroy(a->gexec);
    for (ArkSolve& s : a->solves)
        if (s.d_tab) cudaFree(s.d_tab);
    if (a->d_ring) cudaFree(a->d_ring);
    if (a->d_cgeo) cudaFree(a->d_cgeo);
    if (a->d_items) cudaFree(a->d_items);
    if (a->d_clx) cudaFree(a->d_clx);
    if (a->d_clepoch) cudaFree(a->d_clepoch);
    if (a->d_abort) cudaFree(a->d_abort);
    if (a->d_y0) cudaFree(a->d_y0);
    if (a->d_err) cudaFree(a->d_err);
    if (a->ev0) cudaEventDestroy(a->ev0);
    if (a->ev1) cudaEventDestroy(a->ev1);
    if (a->stream) cudaStreamDestroy(a->stream);
    delete a;
    return RIDC_OK;
}

const char* ridc_ark_last_error(const ridc_ark_ctx* a) { return a ? a->err.c_str() : g_last_error.c_str(); }

}  // extern "C"

// ================================================================ 2-D row shards (§8f rank 4)
//
// The y-direction of the 2-D kinds is explicit (only the x-lines are solved
// implicitly), so a 2-D state splits into row shards that need, per tick, only
// each neighbour's boundary row of every slot just written: shard s owns rows
// [r0, r0 + n) and keeps them as local rows 1..n of an (n + 2)-row layout
// whose rows 0 and n + 1 are ghosts of the neighbours' rows (periodic in y).
// Every level runs on every shard (the shards sit UNDER the levels), the
// tiling in x is the unsharded one, and the y-neighbours carry the same
// values, so a sharded run equals the unsharded engine bitwise.
//
// This group drives S shards on ONE device in lockstep (one graph: per tick
// the S tick launches, then 2 S row copies per active level).  Across GPUs
// the same per-tick boundary-row exchange becomes peer copies / NCCL
// send-recv between neighbouring ranks; that transport is the next step.

struct ridc_shards {
    int device = 0;
    int nshards = 0;
    int levels = 0;
    long long steps = 0, per = 0, ticks = 0;
    int restarts = 0;
    int nx = 0, ny = 0;
    std::vector<ridc_ctx*> sh;
    std::vector<int> r0, n;
    cudaStream_t stream = nullptr;
    cudaGraphExec_t gexec = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    long long launches = 0;
    // multi-stream mode (one stream per shard, possibly one device per shard):
    // per shard a mailbox {got_up, got_dn} = last global tick whose boundary row
    // the upper / lower neighbour has copied into this shard's ghost row
    bool multi = false;
    std::vector<unsigned long long*> mbox;
    std::vector<cudaEvent_t> sev0, sev1;
    double watchdog = 30.0;
    long long epoch = 0;           // mailbox counters of run m start above epoch (no per-run reset)
    std::string err;
};

namespace {

int shard_fail(ridc_shards* g, int code, const std::string& m) { return fail(g ? &g->err : nullptr, code, m); }

// padded row `row` of ring j, slot index `slot` of shard context c
double* shard_row(ridc_ctx* c, int j, long long slot, int row)
{
    return c->d_ring[j] + slot * c->Vs + (size_t)row * c->ss.lay.P;
}

int capture_shards(ridc_shards* g)
{
    const int S = g->nshards, L = g->levels;
    cudaGraph_t graph = nullptr;
    CUDA_TRY(&g->err, cudaStreamBeginCapture(g->stream, cudaStreamCaptureModeThreadLocal));
    cudaError_t le = cudaSuccess;
    long long launches = 0;
    const int sb_max = 148 * 8;
    for (int r = 0; r < g->restarts && le == cudaSuccess; ++r) {
        for (int s = 0; s < S && le == cudaSuccess; ++s) {
            ridc_ctx* c = g->sh[s];
            EngineParams ep = interval_params(c, r);
            const int sb = (int)std::min<long long>((c->Vs + 255) / 256, sb_max);
            if (r == 0) {
                k_seed_chunk<<<sb, 256, 0, g->stream>>>(c->d_y0, ep, -1);
            } else {
                // the top level's final of the previous interval, ghosts included
                // (refreshed by the last tick's exchange)
                EngineParams prev = interval_params(c, r - 1);
                const double* src = prev.ring[L - 1] + ((prev.off[L - 1] + c->per) % prev.cap[L - 1]) * c->Vs;
                const ChunkLayout& Ly = c->ss.lay;
                le = cudaMemcpy2DAsync(c->d_y0 + c->V, (size_t)c->pb.nx * sizeof(double), src + Ly.GW,
                                       (size_t)Ly.P * sizeof(double), (size_t)c->pb.nx * sizeof(double),
                                       (size_t)c->pb.ny, cudaMemcpyDeviceToDevice, g->stream);
                if (le == cudaSuccess) k_seed_chunk<<<sb, 256, 0, g->stream>>>(c->d_y0 + c->V, ep, -1);
            }
            if (le == cudaSuccess) le = cudaGetLastError();
            ++launches;
        }
        for (long long k = 1; k <= g->ticks && le == cudaSuccess; ++k) {
            TickParams tp;
            memset(&tp, 0, sizeof tp);
            for (int j = 0; j < L; ++j) {
                const long long t = k - delay(j);
                if (t >= 1 && t <= g->per) {
                    tp.level[tp.nact] = j;
                    tp.target[tp.nact] = t;
                    ++tp.nact;
                }
            }
            if (tp.nact == 0) continue;
            for (int s = 0; s < S && le == cudaSuccess; ++s) {
                ridc_ctx* c = g->sh[s];
                EngineParams ep = interval_params(c, r);
                tp.sv = ep.sv;
                const int items = g->n[s] * c->ss.sv.nseg;   // owned rows only
                le = launch_chunk(c->pb.kind, c->ss.ccfg,
                                  std::min(c->nsm * chunk_ctas_per_sm(c->ss.ccfg, tp.nact), tp.nact * items), g->stream,
                                  ep, tp, items, c->tm);
                ++launches;
            }
            // boundary rows of every slot written this tick -> the neighbours' ghost rows
            for (int a = 0; a < tp.nact && le == cudaSuccess; ++a) {
                const int j = tp.level[a];
                for (int s = 0; s < S && le == cudaSuccess; ++s) {
                    ridc_ctx* c = g->sh[s];
                    ridc_ctx* up = g->sh[(s + S - 1) % S];
                    ridc_ctx* dn = g->sh[(s + 1) % S];
                    EngineParams ep = interval_params(c, r);
                    const long long slot = (ep.off[j] + tp.target[a]) % ep.cap[j];
                    const size_t rowb = (size_t)c->ss.lay.P * sizeof(double);
                    le = cudaMemcpyAsync(shard_row(up, j, slot, g->n[(s + S - 1) % S] + 1), shard_row(c, j, slot, 1),
                                         rowb, cudaMemcpyDeviceToDevice, g->stream);
                    if (le == cudaSuccess)
                        le = cudaMemcpyAsync(shard_row(dn, j, slot, 0), shard_row(c, j, slot, g->n[s]), rowb,
                                             cudaMemcpyDeviceToDevice, g->stream);
                }
            }
        }
    }
    cudaError_t ce = cudaStreamEndCapture(g->stream, &graph);
    if (le != cudaSuccess) {
        if (graph) cudaGraphDestroy(graph);
        return shard_fail(g, RIDC_E_CUDA, std::string("shard capture: ") + cudaGetErrorString(le));
    }
    CUDA_TRY(&g->err, ce);
    cudaError_t ie = cudaGraphInstantiate(&g->gexec, graph, 0);
    cudaGraphDestroy(graph);
    CUDA_TRY(&g->err, ie);
    g->launches = launches;
    return RIDC_OK;
}

// Multi-stream shard interval (one stream per shard; shards may sit on
// different devices).  Per tick k (global tick G = interval * ticks + k):
//   wait until both neighbours delivered tick G-1 into my ghost rows
//   (cuStreamWaitValue64 on my mailbox), run the tick, copy my boundary rows
//   of every slot just written into the neighbours' ghost rows (peer copies
//   over NVLink across devices), then raise their mailboxes to G.
// A neighbour delivers tick G only after finishing tick G, so when my copy
// of tick G+1 lands in its ghost row of a slot, its last read of that slot's
// old content (at tick G at the latest) is done: skew is at most one tick.
int enqueue_shard(ridc_shards* g, int s, int interval)
{
    // (global tick numbers below are offset by the run epoch)
    const DriverOps& ops = driver_ops();
    if (!ops.wait || !ops.write) return shard_fail(g, RIDC_E_CUDA, "stream memory operations unavailable");
    const int S = g->nshards, L = g->levels;
    ridc_ctx* c = g->sh[s];
    const int su = (s + S - 1) % S, sd = (s + 1) % S;
    ridc_ctx* up = g->sh[su];
    ridc_ctx* dn = g->sh[sd];
    CUstream cs = reinterpret_cast<CUstream>(c->stream);
    CUDA_TRY(&g->err, cudaSetDevice(c->device));
    EngineParams ep = interval_params(c, interval);
    const long long G0 = g->epoch + (long long)interval * g->ticks;
    const int sb = (int)std::min<long long>((c->Vs + 255) / 256, 148 * 8);
    // got_up is written by the upper neighbour's stream, got_dn by the lower's
    // (after their peer copies): remote writers need a flushing wait
    const bool can_flush = device_can_flush_remote(c->device);
    unsigned* abort = reinterpret_cast<unsigned*>(g->mbox[s] + 2);
    const long long spin = (long long)(g->watchdog * 2.0e9);
    auto wait_both = [&](long long G) -> int {
        if (G <= 0) return RIDC_OK;
        if (wait_value(c->stream, g->mbox[s] + 0, (unsigned long long)G, up->device != c->device, can_flush, abort,
                       spin) != cudaSuccess ||
            wait_value(c->stream, g->mbox[s] + 1, (unsigned long long)G, dn->device != c->device, can_flush, abort,
                       spin) != cudaSuccess)
            return shard_fail(g, RIDC_E_CUDA, "shard mailbox wait failed");
        return RIDC_OK;
    };
    int rc;
    if (interval == 0) {
        k_seed_chunk<<<sb, 256, 0, c->stream>>>(c->d_y0, ep, -1);
    } else {
        // the previous interval's top final with ghost rows the neighbours refreshed
        if ((rc = wait_both(G0)) != RIDC_OK) return rc;   // the last tick of the previous interval
        EngineParams prev = interval_params(c, interval - 1);
        const double* src = prev.ring[L - 1] + ((prev.off[L - 1] + c->per) % prev.cap[L - 1]) * c->Vs;
        const ChunkLayout& Ly = c->ss.lay;
        CUDA_TRY(&g->err, cudaMemcpy2DAsync(c->d_y0 + c->V, (size_t)c->pb.nx * sizeof(double), src + Ly.GW,
                                            (size_t)Ly.P * sizeof(double), (size_t)c->pb.nx * sizeof(double),
                                            (size_t)c->pb.ny, cudaMemcpyDeviceToDevice, c->stream));
        k_seed_chunk<<<sb, 256, 0, c->stream>>>(c->d_y0 + c->V, ep, -1);
    }
    CUDA_TRY(&g->err, cudaGetLastError());
    const size_t rowb = (size_t)c->ss.lay.P * sizeof(double);
    for (long long k = 1; k <= g->ticks; ++k) {
        TickParams tp;
        memset(&tp, 0, sizeof tp);
        tp.sv = ep.sv;
        for (int j = 0; j < L; ++j) {
            const long long t = k - delay(j);
            if (t >= 1 && t <= g->per) {
                tp.level[tp.nact] = j;
                tp.target[tp.nact] = t;
                ++tp.nact;
            }
        }
        const long long G = G0 + k;
        if ((k > 1 || interval > 0) && (rc = wait_both(G - 1)) != RIDC_OK) return rc;
        if (tp.nact > 0) {
            const int items = g->n[s] * c->ss.sv.nseg;
            cudaError_t le = launch_chunk(c->pb.kind, c->ss.ccfg,
                                          std::min(c->nsm * chunk_ctas_per_sm(c->ss.ccfg, tp.nact), tp.nact * items),
                                          c->stream, ep, tp, items, c->tm);
            if (le != cudaSuccess) return shard_fail(g, RIDC_E_CUDA, std::string("shard tick: ") + cudaGetErrorString(le));
            for (int a = 0; a < tp.nact; ++a) {
                const int j = tp.level[a];
                const long long slot = (ep.off[j] + tp.target[a]) % ep.cap[j];
                CUDA_TRY(&g->err, cudaMemcpyAsync(shard_row(up, j, slot, g->n[su] + 1), shard_row(c, j, slot, 1), rowb,
                                                  cudaMemcpyDefault, c->stream));
                CUDA_TRY(&g->err, cudaMemcpyAsync(shard_row(dn, j, slot, 0), shard_row(c, j, slot, g->n[s]), rowb,
                                                  cudaMemcpyDefault, c->stream));
            }
        }
        // my rows of tick G are in both neighbours' ghosts (the upper neighbour's
        // lower ghost: its got_dn; the lower neighbour's upper ghost: its got_up)
        if (ops.write(cs, (CUdeviceptr)(g->mbox[su] + 1), (cuuint64_t)G, CU_STREAM_WRITE_VALUE_DEFAULT) != CUDA_SUCCESS ||
            ops.write(cs, (CUdeviceptr)(g->mbox[sd] + 0), (cuuint64_t)G, CU_STREAM_WRITE_VALUE_DEFAULT) != CUDA_SUCCESS)
            return shard_fail(g, RIDC_E_CUDA, "cuStreamWriteValue64 (shard mailbox) failed");
        ++g->launches;
    }
    return RIDC_OK;
}

}  // namespace

extern "C" {

int ridc_shards_destroy(ridc_shards* g)
{
    if (!g) return RIDC_OK;
    cudaSetDevice(g->device);
    if (g->stream) cudaStreamSynchronize(g->stream);
    if (g->gexec) cudaGraphExecDestroy(g->gexec);
    for (size_t s = 0; s < g->mbox.size(); ++s) {
        if (s < g->sh.size() && g->sh[s]) cudaSetDevice(g->sh[s]->device);
        if (g->mbox[s]) cudaFree(g->mbox[s]);
        if (s < g->sev0.size() && g->sev0[s]) cudaEventDestroy(g->sev0[s]);
        if (s < g->sev1.size() && g->sev1[s]) cudaEventDestroy(g->sev1[s]);
    }
    for (ridc_ctx* c : g->sh) ridc_destroy(c);
    if (g->ev0) cudaEventDestroy(g->ev0);
    if (g->ev1) cudaEventDestroy(g->ev1);
    if (g->stream) cudaStreamDestroy(g->stream);
    delete g;
    return RIDC_OK;
}

int ridc_shards_create(const ridc_problem* problem, double t_start, double t_end, int32_t levels, int64_t steps,
                       int32_t restarts, const double* weights, int64_t nweights, int32_t nshards, int32_t device,
                       ridc_shards** out)
{
    if (!out) return fail(nullptr, RIDC_E_CONFIG, "out is NULL");
    *out = nullptr;
    int rc = validate_problem(problem);
    if (rc) return rc;
    if (problem->kind != RIDC_ADV_DIFF_2D && problem->kind != RIDC_REACTION_DIFFUSION_2D)
        return fail(nullptr, RIDC_E_CONFIG, "row shards need a 2-D kind (explicit in y)");
    if (nshards < 2 || nshards > problem->ny) return fail(nullptr, RIDC_E_CONFIG, "need 2 <= shards <= ny");
    ridc_shards* g = new ridc_shards();
    g->device = device;
    g->nshards = nshards;
    g->levels = levels;
    g->steps = steps;
    g->restarts = restarts;
    g->nx = problem->nx;
    g->ny = problem->ny;
    for (int s = 0; s < nshards; ++s) {
        const int a = (int)((long long)problem->ny * s / nshards), b = (int)((long long)problem->ny * (s + 1) / nshards);
        g->r0.push_back(a);
        g->n.push_back(b - a);
        ridc_problem sub = *problem;
        sub.ny = b - a + 2;   // owned rows + one ghost row on each side
        ridc_ctx* c = nullptr;
        rc = ridc_create(&sub, t_start, t_end, levels, steps, restarts, weights, nweights, device, RIDC_TICK_ONLY, &c);
        if (rc) {
            const std::string m = g_last_error;
            ridc_shards_destroy(g);
            g_last_error = m;
            return rc;
        }
        c->ep.row0 = 1;   // compute rows 1..n; rows 0 and n+1 are the neighbours' ghosts
        g->sh.push_back(c);
    }
    g->per = g->sh[0]->per;
    g->ticks = g->sh[0]->ticks;
    auto bail = [&](int code) {
        const std::string m = g->err.empty() ? g_last_error : g->err;
        ridc_shards_destroy(g);
        g_last_error = m;
        return code;
    };
    if (cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreate(&g->ev0) != cudaSuccess || cudaEventCreate(&g->ev1) != cudaSuccess) {
        g->err = "stream / event creation failed";
        return bail(RIDC_E_CUDA);
    }
    if ((rc = capture_shards(g)) != RIDC_OK) return bail(rc);
    *out = g;
    return RIDC_OK;
}

static int shards_run_multi(ridc_shards* g, const double* y0_host, double* final_host, double* wall_seconds)
{
    const size_t rowb = (size_t)g->nx * sizeof(double);
    const int S = g->nshards;
    for (int s = 0; s < S; ++s) {
        ridc_ctx* c = g->sh[s];
        CUDA_TRY(&g->err, cudaSetDevice(c->device));
        for (int lr = 0; lr < g->n[s] + 2; ++lr) {
            const int gr = (g->r0[s] - 1 + lr + g->ny) % g->ny;
            CUDA_TRY(&g->err, cudaMemcpyAsync(c->d_y0 + (size_t)lr * g->nx, y0_host + (size_t)gr * g->nx, rowb,
                                              cudaMemcpyHostToDevice, c->stream));
        }
        CUDA_TRY(&g->err, cudaMemsetAsync(c->d_err, 0xff, sizeof(unsigned long long), c->stream));
        CUDA_TRY(&g->err, cudaMemsetAsync(g->mbox[s] + 2, 0, sizeof(unsigned long long), c->stream));
        CUDA_TRY(&g->err, cudaEventRecord(g->sev0[s], c->stream));
    }
    int rc;
    for (int r = 0; r < g->restarts; ++r)
        for (int s = 0; s < S; ++s)
            if ((rc = enqueue_shard(g, s, r)) != RIDC_OK) return rc;
    for (int s = 0; s < S; ++s) {
        CUDA_TRY(&g->err, cudaSetDevice(g->sh[s]->device));
        CUDA_TRY(&g->err, cudaEventRecord(g->sev1[s], g->sh[s]->stream));
    }
    // watchdog: a shard whose neighbour never delivers turns into PipelineProtocolError
    const auto t0 = std::chrono::steady_clock::now();
    for (int s = 0; s < S; ++s) {
        for (;;) {
            cudaSetDevice(g->sh[s]->device);
            cudaError_t q = cudaEventQuery(g->sev1[s]);
            if (q == cudaSuccess) break;
            if (q != cudaErrorNotReady) return shard_fail(g, RIDC_E_CUDA, cudaGetErrorString(q));
            if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > g->watchdog)
                return shard_fail(g, RIDC_E_PROTOCOL, "row shards made no progress within the watchdog");
            std::this_thread::sleep_for(std::chrono::microseconds(200));
        }
    }
    g->epoch += (long long)g->restarts * g->ticks + 1;
    for (int s = 0; s < S; ++s) {   // an in-kernel mailbox wait that timed out
        unsigned ab = 0;
        CUDA_TRY(&g->err, cudaSetDevice(g->sh[s]->device));
        CUDA_TRY(&g->err, cudaMemcpy(&ab, g->mbox[s] + 2, sizeof ab, cudaMemcpyDeviceToHost));
        if (ab) return shard_fail(g, RIDC_E_PROTOCOL, "row shards made no progress within the watchdog");
    }
    double wall = 0.0;
    for (int s = 0; s < S; ++s) {
        ridc_ctx* c = g->sh[s];
        CUDA_TRY(&g->err, cudaSetDevice(c->device));
        float ms = 0.f;
        CUDA_TRY(&g->err, cudaEventElapsedTime(&ms, g->sev0[s], g->sev1[s]));
        wall = std::max(wall, ms * 1e-3);
        rc = check_err_word(c);
        if (rc) return shard_fail(g, rc, c->err);
        const ChunkLayout& Ly = c->ss.lay;
        const double* fin = final_slot(c, g->levels - 1) + (size_t)1 * Ly.P;
        CUDA_TRY(&g->err, cudaMemcpy2DAsync(final_host + (size_t)g->r0[s] * g->nx, rowb, fin + Ly.GW,
                                            (size_t)Ly.P * sizeof(double), rowb, (size_t)g->n[s],
                                            cudaMemcpyDeviceToHost, c->stream));
        CUDA_TRY(&g->err, cudaStreamSynchronize(c->stream));
    }
    if (wall_seconds) *wall_seconds = wall;
    return RIDC_OK;
}

int ridc_shards_run(ridc_shards* g, const double* y0_host, double* final_host, double* wall_seconds)
{
    NvtxRange nvtx_("ridc.shards_run");
    if (!g || !y0_host || !final_host) return shard_fail(g, RIDC_E_CONFIG, "NULL argument");
    if (g->multi) return shards_run_multi(g, y0_host, final_host, wall_seconds);
    CUDA_TRY(&g->err, cudaSetDevice(g->device));
    const size_t rowb = (size_t)g->nx * sizeof(double);
    const int S = g->nshards;
    // each shard's initial state: its rows plus the wrapped neighbour rows
    for (int s = 0; s < S; ++s) {
        ridc_ctx* c = g->sh[s];
        for (int lr = 0; lr < g->n[s] + 2; ++lr) {
            const int gr = (g->r0[s] - 1 + lr + g->ny) % g->ny;
            CUDA_TRY(&g->err, cudaMemcpyAsync(c->d_y0 + (size_t)lr * g->nx, y0_host + (size_t)gr * g->nx, rowb,
                                              cudaMemcpyHostToDevice, g->stream));
        }
        CUDA_TRY(&g->err, cudaMemsetAsync(c->d_err, 0xff, sizeof(unsigned long long), g->stream));
    }
    CUDA_TRY(&g->err, cudaEventRecord(g->ev0, g->stream));
    CUDA_TRY(&g->err, cudaGraphLaunch(g->gexec, g->stream));
    CUDA_TRY(&g->err, cudaEventRecord(g->ev1, g->stream));
    CUDA_TRY(&g->err, cudaEventSynchronize(g->ev1));
    if (wall_seconds) {
        float ms = 0.f;
        CUDA_TRY(&g->err, cudaEventElapsedTime(&ms, g->ev0, g->ev1));
        *wall_seconds = ms * 1e-3;
    }
    for (int s = 0; s < S; ++s) {
        ridc_ctx* c = g->sh[s];
        int rc = check_err_word(c);
        if (rc) return shard_fail(g, rc, c->err);
        const ChunkLayout& Ly = c->ss.lay;
        const double* fin = final_slot(c, g->levels - 1) + (size_t)1 * Ly.P;   // owned rows 1..n
        CUDA_TRY(&g->err, cudaMemcpy2DAsync(final_host + (size_t)g->r0[s] * g->nx, rowb, fin + Ly.GW,
                                            (size_t)Ly.P * sizeof(double), rowb, (size_t)g->n[s],
                                            cudaMemcpyDeviceToHost, g->stream));
    }
    CUDA_TRY(&g->err, cudaStreamSynchronize(g->stream));
    return RIDC_OK;
}

int ridc_shards_info(const ridc_shards* g, int64_t* kernel_launches)
{
    if (!g) return fail(nullptr, RIDC_E_CONFIG, "NULL argument");
    if (kernel_launches) *kernel_launches = g->launches;
    return RIDC_OK;
}

const char* ridc_shards_last_error(const ridc_shards* g) { return g ? g->err.c_str() : g_last_error.c_str(); }

int ridc_shards_create_multi(const ridc_problem* problem, double t_start, double t_end, int32_t levels,
                             int64_t steps, int32_t restarts, const double* weights, int64_t nweights,
                             int32_t nshards, const int32_t* devices, double watchdog_seconds, ridc_shards** out)
{
    if (!out || !devices) return fail(nullptr, RIDC_E_CONFIG, "NULL argument");
    *out = nullptr;
    int rc = validate_problem(problem);
    if (rc) return rc;
    if (problem->kind != RIDC_ADV_DIFF_2D && problem->kind != RIDC_REACTION_DIFFUSION_2D)
        return fail(nullptr, RIDC_E_CONFIG, "row shards need a 2-D kind (explicit in y)");
    if (nshards < 2 || nshards > problem->ny) return fail(nullptr, RIDC_E_CONFIG, "need 2 <= shards <= ny");
    if (!driver_ops().wait || !driver_ops().write)
        return fail(nullptr, RIDC_E_CUDA, "stream memory operations unavailable");
    ridc_shards* g = new ridc_shards();
    g->multi = true;
    g->device = devices[0];
    g->nshards = nshards;
    g->levels = levels;
    g->steps = steps;
    g->restarts = restarts;
    g->nx = problem->nx;
    g->ny = problem->ny;
    g->watchdog = watchdog_seconds > 0 ? watchdog_seconds : 30.0;
    auto bail = [&](int code) {
        const std::string m = g->err.empty() ? g_last_error : g->err;
        ridc_shards_destroy(g);
        g_last_error = m;
        return code;
    };
    for (int s = 0; s < nshards; ++s) {
        const int a = (int)((long long)problem->ny * s / nshards), b = (int)((long long)problem->ny * (s + 1) / nshards);
        g->r0.push_back(a);
        g->n.push_back(b - a);
        ridc_problem sub = *problem;
        sub.ny = b - a + 2;
        ridc_ctx* c = nullptr;
        rc = ridc_create(&sub, t_start, t_end, levels, steps, restarts, weights, nweights, devices[s], RIDC_TICK_ONLY,
                         &c);
        if (rc) return bail(rc);
        c->ep.row0 = 1;
        g->sh.push_back(c);
        unsigned long long* mb = nullptr;
        cudaEvent_t e0 = nullptr, e1 = nullptr;
        // {got_up, got_dn, abort word of the in-kernel waits, pad}
        if (cudaSetDevice(devices[s]) != cudaSuccess || cudaMalloc(&mb, 4 * sizeof(unsigned long long)) != cudaSuccess ||
            cudaMemset(mb, 0, 4 * sizeof(unsigned long long)) != cudaSuccess || cudaEventCreate(&e0) != cudaSuccess ||
            cudaEventCreate(&e1) != cudaSuccess) {
            g->err = "shard mailbox / event allocation failed";
            return bail(RIDC_E_CUDA);
        }
        g->mbox.push_back(mb);
        g->sev0.push_back(e0);
        g->sev1.push_back(e1);
    }
    // peer access between neighbouring shards on different devices
    for (int s = 0; s < nshards; ++s)
        for (int nb : {(s + nshards - 1) % nshards, (s + 1) % nshards}) {
            if (devices[s] == devices[nb]) continue;
            cudaSetDevice(devices[s]);
            cudaError_t e = cudaDeviceEnablePeerAccess(devices[nb], 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) {
                g->err = std::string("peer access: ") + cudaGetErrorString(e);
                return bail(RIDC_E_CUDA);
            }
            cudaGetLastError();
        }
    g->per = g->sh[0]->per;
    g->ticks = g->sh[0]->ticks;
    *out = g;
    return RIDC_OK;
}

}  // extern "C"
