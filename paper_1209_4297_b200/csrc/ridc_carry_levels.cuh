// ridc_carry_levels.cuh -- the tick of the lagged level pipeline on 1-D
// periodic reaction-diffusion lines of up to 14 x SMs x 512 points (C2:
// 2^20 at p = 2..4; or 7 x SMs x 1024 points for shifts whose carry reach
// exceeds 512), one chunk per warp, no truncation halos.
//
// One launch per pipeline tick (the tick kernel's schedule, engine.py:363-371;
// every level of a tick reads only data published in earlier ticks).  The
// line is cut into 512-point chunks (16 points per lane); warp w of CTA b owns
// chunk b x wpc + w and, for every active level in turn:
//   * folds the level's right-hand side node by node (build_item's node list:
//     the level's own state and its window of level j-1 states with the
//     weights and lag terms of _correct_core, engine.py:124-187), each node
//     chunk TMA-staged once with one group either side for the f^S stencil
//     -- SURVEY.md §8d's 8 (j+3) B/pt per level-j step;
//   * solves (I - dt L_S) x = rhs on its chunk with zero carries at both ends
//     (the two recurrences of ridc_device.cuh as warp scans), and publishes
//     two numbers in the LL line format (ridc_resident.cuh): y at its last
//     point (the forward carry of the chunk to its right) and x at its first
//     point (the backward carry of the chunk to its left);
//   * corrects its chunk with the neighbours' two numbers, exactly as the
//     carry-exchange FEBE march does between its tiles (ridc_febe_carry.cuh):
//       head  x_i += c lam^(i+1) / (1 - lam^2),   c = left chunk's y_end
//       tail  x_i += d lam^(512-i),  d = right chunk's first x + my y_end lam / (1 - lam^2)
//     (terms dropped: lam^512 <= 2^-60 relative, carry reach hc <= 512);
//   * stores the chunk (256-bit stores; the line's end chunks also write the
//     periodic ghost columns the next tick's stencils read).
// Every message depends only on the sender's own fold and solve, so each wait
// is one L2 round trip, and it is taken only after the warp folded and solved
// the NEXT level (a two-level software pipeline), by when the neighbours have
// usually published.  States agree with the tick
// kernel to rounding (different association) and with the oracle at <= 1e-10
// (tests/test_gpu_resident.py, test_gpu_fullsize.py).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "ridc_chunk.cuh"
#include "ridc_device.cuh"
#include "ridc_febe_carry.cuh"
#include "ridc_resident.cuh"
#include "ridc_sweep.cuh"
#include "ridc_tma.cuh"
// EngineParams, TickParams, build_item: ridc_kernels.cuh (which includes this file after them)

namespace ridc {

// K points per lane: 16 (512-point chunks, carry reach <= 512) or 32
// (1024-point chunks, reach <= 1024: stiffer shifts, e.g. imex3's a_ii = 2
// stage at C2)
template <int K> struct ClGeom {
    static constexpr int WARPS = K == 16 ? 14 : 7;   // warps (chunks) per CTA at most (shared memory)
    static constexpr int BOX = 2 * K + 2;            // staged groups per node chunk: 2K + one either side
    static constexpr int STAGE = (BOX * 128 + 1023) / 1024 * 1024;   // bytes, the 1024-byte swizzle atom
};
constexpr int kClWarps = 14;          // warps per CTA at most (K = 16)
constexpr int kClStages = 3;          // TMA stages per warp
constexpr int kClBoxGroups = 34;      // the tensor maps' box (K = 16); K = 32 issues two boxes

struct ClNode {   // one node of one level's fold, coefficients with g folded in
    double ga, gb, gs;
    long long slot;
    int lev;
};

struct ClLevel {
    int nn, node0;   // nodes [node0, node0 + nn) of the node table
    int level;
    long long target;
    double* out;
};

constexpr int kClMaxNodes = kMaxLevels * (kMaxLevels + 3) / 2 + 1;   // sum over levels of (j + 2)

template <int K>
inline size_t carry_levels_smem()
{
    return (size_t)ClGeom<K>::WARPS * kClStages * ClGeom<K>::STAGE + 1024;
}

struct CarryLevParams {
    double lam, g, inv1ml2, zc;   // zc = lam / (1 - lam^2)
    double pw[32];                // lam^(e+1), e < K
    double zf[32];                // forward-carry response of a K-point backward pass
    double mp[10];                // M^(2^i), M = lam^K
    int nx, GW, gdata;
    int nchunk;                   // nx / (32 K)
    int wpc;                      // chunks (warps) per CTA
    uint4* xch;                   // [2][kMaxLevels][nchunk] LL lines: 0 = y_end, 1 = first x
    const unsigned* epoch;        // bumped once per run (the graph's first node)
    unsigned ticks;               // ticks per run: tag = epoch * ticks + tick
    unsigned* abort;
    long long spin_limit;
    int exp;                      // diagnostics (RIDC_CL_EXP): 1 = every CTA exits after the launch prologue
};

template <int KIND, int K>
__global__ void __launch_bounds__(ClGeom<K>::WARPS * 32, 1)
    k_carry_levels(EngineParams ep, TickParams tp, const __grid_constant__ CarryLevParams cp,
                   const __grid_constant__ TmapSet tm, unsigned tick)
{
    static_assert(KIND == RD_1D, "carry-exchange level tick: periodic reaction-diffusion lines");
    static_assert(K == 16 || K == 32, "16 or 32 points per lane");
    constexpr int NS = kClStages, GL = K / 16, CH = 32 * K;   // groups per lane, points per chunk
    constexpr int kClStage = ClGeom<K>::STAGE;
    extern __shared__ __align__(1024) char smraw[];
    char* base = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t s_full[ClGeom<K>::WARPS * NS];
    __shared__ ClLevel s_lev[kMaxLevels];
    __shared__ ClNode s_node[kClMaxNodes];
    __shared__ unsigned s_tag;
    const unsigned FULL = 0xffffffffu;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int chunk = blockIdx.x * cp.wpc + warp;
    const bool active = warp < cp.wpc && chunk < cp.nchunk;
    char* stage = base + (size_t)warp * NS * kClStage;
    uint64_t* full = s_full + warp * NS;
    const int nact = tp.nact;
    const double lam = cp.lam, g = cp.g;

    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    // the fold tables of this tick's items (build_item's nodes, g folded into the
    // coefficients), one thread per active level (before the wait: overlaps the
    // previous tick's tail)
    if (tp.pre) {   // precomputed items (ARK stages: nodes y_n and the earlier stages, steppers.py:122-142)
        if (tid < nact) {
            int nn = 0;
            for (int b = 0; b < tid; ++b) nn += tp.pre[b].nnodes;
            const StepItem& it = tp.pre[tid];
            ClLevel& lv = s_lev[tid];
            lv.level = it.level;
            lv.target = tp.target[tid];
            lv.node0 = nn;
            lv.nn = it.nnodes;
            lv.out = it.out;
            for (int b = 0; b < it.nnodes; ++b) {
                const NodeCoef nc = node_coef<KIND>(ep.pb, it.ca[b], it.cs[b], it.cn[b]);
                s_node[nn + b] = ClNode{g * nc.a, g * nc.b, g * nc.cs * ep.pb.cdx, it.vslot[b], it.vlev[b]};
            }
            RIDC_CHECK(nn + it.nnodes <= kClMaxNodes);
        }
    } else if (tid < nact) {
        const int a = tid;
        int nn = 0;
        for (int b = 0; b < a; ++b) nn += tp.level[b] > 0 ? tp.level[b] + 2 : 1;
        const int j = tp.level[a];
        const long long t = tp.target[a];
        ClLevel& lv = s_lev[a];
        lv.level = j;
        lv.target = t;
        lv.node0 = nn;
        lv.out = ring_slot(ep, j, t);
        const NodeCoef n0 = node_coef<KIND>(ep.pb, 1.0, 0.0, ep.dt);
        s_node[nn++] = ClNode{g * n0.a, g * n0.b, 0.0, slot_index(ep, j, t - 1), j};
        if (j > 0) {
            const bool steady = t >= j;
            const double* w = steady ? ep.weights + ep.steady_off[j]
                                     : ep.weights + ep.startup_off[j] + (t - 1) * (j + 1);
            const int i_new = steady ? 0 : (int)t, i_old = steady ? 1 : (int)t - 1;
            for (int b = 0; b <= j; ++b) {
                const long long s = steady ? t - b : b;
                const NodeCoef nc = node_coef<KIND>(ep.pb, 0.0, w[b] - (b == i_new ? ep.dt : 0.0),
                                                    w[b] - (b == i_old ? ep.dt : 0.0));
                s_node[nn++] = ClNode{g * nc.a, g * nc.b, g * nc.cs * ep.pb.cdx, slot_index(ep, j - 1, s), j - 1};
            }
        }
        lv.nn = nn - lv.node0;
        RIDC_CHECK(nn <= kClMaxNodes);
    }
    if (lane == 0) {
        for (int i = 0; i < NS; ++i) mbar_init(&full[i], 1);
        mbar_fence_init();
    }
    // every read of earlier ticks' states (and of the run epoch) waits for the previous launch
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (tid == 0) s_tag = *(volatile const unsigned*)cp.epoch * cp.ticks + tick;
    __syncthreads();
    if (!active || cp.exp == 1) return;
    const unsigned tag = s_tag;
    const int c0 = chunk * CH;   // data column of my chunk's first point
    const int cl = chunk == 0 ? cp.nchunk - 1 : chunk - 1, cr = chunk == cp.nchunk - 1 ? 0 : chunk + 1;
    RIDC_CHECK(cl >= 0 && cl < cp.nchunk && cr >= 0 && cr < cp.nchunk && c0 + CH <= cp.nx);

    // node loads in fold order (level a, node n), NS stages ahead; lane 0 issues
    const int ntot = s_lev[nact - 1].node0 + s_lev[nact - 1].nn;
    auto issue = [&](int m) {
        const int s = m % NS;
        const ClNode& nd = s_node[m];
        RIDC_CHECK(nd.slot >= 0 && nd.slot < ep.cap[nd.lev]);
        mbar_arrive_expect_tx(&full[s], (uint32_t)(GL * kClBoxGroups * 128));
        for (int b = 0; b < GL; ++b)   // GL boxes of 34 groups: the chunk + one group either side (+ 2 spare)
            tma_load_3d(stage + (size_t)s * kClStage + b * (32 * 128), &tm.map[nd.lev], 0,
                        cp.gdata + c0 / 16 - 1 + 32 * b, (int)nd.slot, &full[s]);
    };
    if (lane == 0)
        for (int m = 0; m < NS && m < ntot; ++m) issue(m);

    // M^lane, M^(31-lane)
    double ml = 1.0, mr = 1.0;
#pragma unroll
    for (int i = 0; i < 5; ++i) {
        if (lane & (1 << i)) ml *= cp.mp[i];
        if ((31 - lane) & (1 << i)) mr *= cp.mp[i];
    }
    bool dead = false;
    // Software pipeline over the tick's levels: phase A of level a (fold, local
    // solve, publish the two carries) runs before phase B of level a - 1 (wait
    // for the neighbours' carries, correct, store), so a neighbour's carries
    // usually arrive while this warp folds the next level.
    double vp[K];          // level a - 1 after phase A
    double yend_p = 0.0;   // its y at my last point (zero carry in)
    for (int a = 0; a <= nact; ++a) {
        double v[K];
        double yend = 0.0;
        if (a < nact) {
            const ClLevel lv = s_lev[a];
            // ---- the right-hand side (g folded), node by node
#pragma unroll
            for (int e = 0; e < K; ++e) v[e] = 0.0;
            for (int m = lv.node0; m < lv.node0 + lv.nn; ++m) {
                const int s = m % NS;
                mbar_wait(&full[s], (uint32_t)((m / NS) & 1));
                const char* st = stage + (size_t)s * kClStage;
                const ClNode nd = s_node[m];
                // my points: staged groups GL lane + 1 ...; neighbours: group GL lane
                // element 15, group GL (lane + 1) + 1 element 0
                const int g0 = GL * lane + 1;
                double wl = lds128(swz(st, g0 - 1, 7)).y;
                double2 w2 = lds128(swz(st, g0, 0));
#pragma unroll
                for (int q = 0; q < K / 2; ++q) {
                    const double2 wn = q + 1 < K / 2 ? lds128(swz(st, g0 + (q + 1) / 8, (q + 1) % 8))
                                                     : make_double2(lds128(swz(st, g0 + GL, 0)).x, 0.0);
                    v[2 * q] = fma(nd.gs, (wl - 2.0 * w2.x) + w2.y, fma(fma(nd.gb, w2.x, nd.ga), w2.x, v[2 * q]));
                    v[2 * q + 1] =
                        fma(nd.gs, (w2.x - 2.0 * w2.y) + wn.x, fma(fma(nd.gb, w2.y, nd.ga), w2.y, v[2 * q + 1]));
                    wl = w2.y;
                    w2 = wn;
                }
                __syncwarp();   // every staged value consumed above: the stage may be refilled
                if (lane == 0 && m + NS < ntot) issue(m + NS);
            }
            // ---- forward: local recurrence, warp scan with a zero carry into the chunk
            double y = 0.0;
#pragma unroll
            for (int e = 0; e < K; ++e) {
                y = fma(lam, y, v[e]);
                v[e] = y;
            }
            const double inc = warp_fwd_incl(cp, y, lane);
            double cf = __shfl_up_sync(FULL, inc, 1);
            if (lane == 0) cf = 0.0;
            yend = __shfl_sync(FULL, inc, 31);   // y at my last point (zero carry in)
            st_line_if(lane == 31, cp.xch + (size_t)a * cp.nchunk + chunk, yend, tag);
            // ---- backward with a zero carry at the chunk end
            double x = 0.0;
#pragma unroll
            for (int e = K - 1; e >= 0; --e) {
                x = fma(lam, x, v[e]);
                v[e] = x;
            }
            const double rinc = warp_bwd_incl(cp, fma(cf, cp.zf[0], x), lane);
            double exr = __shfl_down_sync(FULL, rinc, 1);
            if (lane == 31) exr = 0.0;
#pragma unroll
            for (int e = 0; e < K; ++e) v[e] = fma(exr, cp.pw[K - 1 - e], fma(cf, cp.zf[e], v[e]));
            // my first x (zero carries at both ends)
            st_line_if(lane == 0, cp.xch + (size_t)(kMaxLevels + a) * cp.nchunk + chunk, v[0], tag);
        }
        if (a > 0) {
            // ---- level a - 1: the neighbours' carries (the left chunk's y_end, the
            // right chunk's first x), the corrections, the store
            const int b = a - 1;
            const ClLevel lv = s_lev[b];
            // lane 0 reads the left chunk's y_end, lane 31 the right one's first x:
            // one predicated load each, one vote, a warp-uniform re-poll loop (no
            // divergent branch around the wait, as the warp FEBE march)
            const bool need = lane == 0 || lane == 31;
            const uint4* src = lane == 0 ? cp.xch + (size_t)b * cp.nchunk + cl
                                         : cp.xch + (size_t)(kMaxLevels + b) * cp.nchunk + cr;
            uint4 lw = ld_line_if(need && !dead, src);
            bool ok = !need || dead || (lw.y == tag && lw.w == tag);
            if (!__all_sync(FULL, ok)) {
                const long long t0 = clock64();
                for (unsigned it = 1; !__all_sync(FULL, ok); ++it) {
                    if (!ok) {
                        lw = ld_line_gen(src);
                        ok = lw.y == tag && lw.w == tag;
                        if (!ok && (it & 63u) == 0u &&
                            (clock64() - t0 > cp.spin_limit || *(volatile unsigned*)cp.abort)) {
                            atomicExch(cp.abort, 1u);
                            dead = true;
                            ok = true;
                        }
                    }
                }
            }
            const double lwv = need && !dead ? line_value(lw) : 0.0;
            const double cv = lane == 0 ? lwv : 0.0, dv = lane == 31 ? lwv : 0.0;
            const double c = __shfl_sync(FULL, cv, 0);
            // + the head correction my own y_end causes at the right chunk's first point
            const double d = fma(yend_p, cp.zc, __shfl_sync(FULL, dv, 31));
            const double hm = c * cp.inv1ml2 * ml, tmul = d * mr;
#pragma unroll
            for (int e = 0; e < K; ++e) vp[e] = fma(tmul, cp.pw[K - 1 - e], fma(hm, cp.pw[e], vp[e]));
            double fc0 = 0.0, fc1 = 0.0;   // finite check over K points (chunk_finite)
#pragma unroll
            for (int e = 0; e < K; e += 2) {
                fc0 = fma(vp[e], 0.0, fc0);
                fc1 = fma(vp[e + 1], 0.0, fc1);
            }
            const bool bad = (fc0 + fc1) != (fc0 + fc1);
            // ---- store (+ the periodic ghost copies of the line's end groups)
            double* o = lv.out + cp.GW + c0 + lane * K;
#pragma unroll
            for (int e = 0; e < K; e += 4) stg256(o + e, vp[e], vp[e + 1], vp[e + 2], vp[e + 3]);
            if (chunk == 0 && lane == 0)   // the line's first group -> the right ghost group
#pragma unroll
                for (int e = 0; e < 16; e += 4) stg256(o + cp.nx + e, vp[e], vp[e + 1], vp[e + 2], vp[e + 3]);
            if (chunk == cp.nchunk - 1 && lane == 31)   // its last group -> the left ghost group
#pragma unroll
                for (int e = K - 16; e < K; e += 4) stg256(o - cp.nx + e, vp[e], vp[e + 1], vp[e + 2], vp[e + 3]);
            if (bad) atomicMin(ep.err, err_code(lv.target, lv.level));
        }
        if (a < nact) {
#pragma unroll
            for (int e = 0; e < K; ++e) vp[e] = v[e];
            yend_p = yend;
        }
    }
}

}  // namespace ridc
