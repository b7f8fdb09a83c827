// ridc_sweep_levels.cuh -- the tick of the lagged level pipeline on long 1-D
// periodic reaction-diffusion lines as sweeps (every active level, RIDC p >= 2).
//
// One launch per pipeline tick (the tick kernel's schedule, engine.py:363-371).
// CTA c owns the range [R0, R1) of the line and, for every active level in
// turn, sweeps it chunk by chunk as the FEBE sweep does (ridc_sweep.cuh): the
// forward carry rides along the sweep, a chunk's last hc points wait one
// chunk for the backward carry, the range ends are closed by truncated passes
// of one warp.  The right-hand side of a chunk is folded node by node from the
// level's own state and its window of level j-1 states (build_item's node list
// and weights: _window_span / _orient / the lag terms of _correct_core,
// engine.py:124-187), each node chunk TMA-staged once with one extra group on
// either side for the f^S stencil:
//   rhs = g sum_nodes [ (a + b w) w + cs cdx (w_{c-1} - 2 w_c + w_{c+1}) ]
// (node_coef, ridc_device.cuh).  Each node value is read once per tick and
// each new value written once -- SURVEY.md §8d's 8 (j+3) B/pt for level j --
// where the tick kernel stages every node with truncation halos.  The levels'
// rings keep one group of periodic ghost columns, written by the CTAs owning
// the line's ends.  States agree with the tick kernel to rounding.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "ridc_chunk.cuh"
#include "ridc_device.cuh"
#include "ridc_sweep.cuh"
#include "ridc_tma.cuh"
// EngineParams, TickParams, build_item: ridc_kernels.cuh (which includes this file after them)

namespace ridc {

constexpr int kSweepLevStages = 3;
constexpr int kSweepLevMaxChunk = 8192 - 32;   // chunk + one group either side fits a 512-group box

inline size_t sweep_levels_smem(int nact)
{
    return (size_t)kSweepLevStages * 8192 * sizeof(double) + 2 * kSweepLevStages * 8 + (size_t)nact * sizeof(StepItem) +
           1024;
}

template <int KIND>
__global__ void __launch_bounds__(512, 1)
    k_sweep_levels(EngineParams ep, TickParams tp, const __grid_constant__ SweepParams sp,
                   const __grid_constant__ TmapSet tm)
{
    static_assert(KIND == RD_1D, "1-D level sweep: periodic reaction-diffusion lines");
    constexpr int NT = 512, K = 16, NW = NT / 32, NS = kSweepLevStages;
    constexpr int STAGE = 8192 * 8;   // 512 groups
    extern __shared__ __align__(1024) char smraw[];
    char* stage = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(stage + (size_t)NS * STAGE);
    uint64_t* empty = full + NS;
    StepItem* items = reinterpret_cast<StepItem*>(stage + (size_t)NS * STAGE + 2 * NS * 8);
    __shared__ double sx[2 * NW];
    __shared__ double s_bc[2];
    // per level: the forward carry into R0 and the local x at R1 (truncated passes, launch start)
    __shared__ double s_cin0[kMaxLevels], s_xbl[kMaxLevels];
    __shared__ double s_pend[16 * kSweepPend];
    const unsigned FULL = 0xffffffffu;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int G = gridDim.x, cta = blockIdx.x;
    const int nx = sp.nx;
    const long long n16 = nx / 16;
    const int R0 = 16 * (int)((long long)cta * n16 / G), R1 = 16 * (int)((long long)(cta + 1) * n16 / G);
    const int Lr = R1 - R0;
    const int nch = (Lr + kSweepLevMaxChunk - 1) / kSweepLevMaxChunk;
    const int Cr = 16 * ((Lr + 16 * nch - 1) / (16 * nch));
    const DevProblem& pb = ep.pb;
    const double lam = sp.lam, g = sp.g;

    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (tid < tp.nact) build_item(ep, tp.level[tid], tp.target[tid], items[tid]);
    if (tid == 0) {
        for (int i = 0; i < NS; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], NW);
        }
        mbar_fence_init();
    }
    double ml = 1.0, mr = 1.0, mt = 1.0;
#pragma unroll
    for (int i = 0; i < 10; ++i) {
        if (i < 5 && (lane & (1 << i))) ml *= sp.mp[i];
        if (i < 5 && ((31 - lane) & (1 << i))) mr *= sp.mp[i];
        if (tid & (1 << i)) mt *= sp.mp[i];
    }
    __syncthreads();
    RIDC_CHECK(Lr >= 1024 && Cr <= kSweepLevMaxChunk && (nch - 1) * Cr < Lr && sp.hc <= 512 && sp.GW >= 16);

    // node chunks in the order (level a, chunk i, node n), NS stages ahead
    int pa = 0, pi = 0, pn = 0;
    long long issued = 0;
    auto issue_next = [&]() {   // thread 0
        if (pa >= tp.nact) return;
        const StepItem& it = items[pa];
        const int s = (int)(issued % NS);
        if (issued >= NS) mbar_wait(&empty[s], (uint32_t)(((issued - NS) / NS) & 1));
        const int g0 = sp.gdata + (R0 + pi * Cr) / 16 - 1;   // one group before the chunk
        RIDC_CHECK(it.vslot[pn] >= 0 && it.vslot[pn] < ep.cap[it.vlev[pn]] && g0 >= 0);
        mbar_arrive_expect_tx(&full[s], (uint32_t)STAGE);
        for (int b = 0; b < 2; ++b)
            tma_load_3d(stage + (size_t)s * STAGE + b * 256 * 128, &tm.map[it.vlev[pn]], 0, g0 + b * 256,
                        (int)it.vslot[pn], &full[s]);
        ++issued;
        if (++pn == it.nnodes) {
            pn = 0;
            if (++pi == nch) { pi = 0; ++pa; }
        }
    };
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (tid == 0)
        for (int i = 0; i < NS; ++i) issue_next();

    // the right-hand side (g folded) of 16 points starting at data column c0 of
    // level item `it`, straight from global memory (range-end passes)
    auto rhs16 = [&](const StepItem& it, int c0, double (&r)[K]) {
#pragma unroll
        for (int e = 0; e < K; ++e) r[e] = 0.0;
        for (int n = 0; n < it.nnodes; ++n) {
            const NodeCoef nc = node_coef<KIND>(pb, it.ca[n], it.cs[n], it.cn[n]);
            const double* row = it.vec[n] + sp.GW;
            const double sxx = nc.cs * pb.cdx;
            double wl = __ldcg(row + (c0 - 1 < 0 ? c0 - 1 + nx : (c0 - 1 >= nx ? c0 - 1 - nx : c0 - 1)));
            double w = __ldcg(row + (c0 < 0 ? c0 + nx : (c0 >= nx ? c0 - nx : c0)));
#pragma unroll
            for (int e = 0; e < K; ++e) {
                int cr = c0 + e + 1;
                cr = cr < 0 ? cr + nx : (cr >= nx ? cr - nx : cr);
                const double wr = __ldcg(row + cr);
                r[e] = fma(g, fma(sxx, (wl - 2.0 * w) + wr, fma(fma(nc.b, w, nc.a), w, 0.0)), r[e]);
                wl = w;
                w = wr;
            }
        }
    };

    // ---- range ends of every level, one warp per (level, end), before the sweeps:
    // the forward carry into R0 (a truncated forward pass over the 512 points before
    // it) and the local backward value at R1 (forward from zero over the 512 points
    // after it, then backward from zero); the range's own forward carry into R1 is
    // added at the end: x(R1) = local + y(R1 - 1) lam / (1 - lam^2)
    for (int task = warp; task < 2 * tp.nact; task += NW) {
        const StepItem& it = items[task >> 1];
        double r[K];
        rhs16(it, (task & 1) ? R1 + 16 * lane : R0 - 512 + 16 * lane, r);
        double y = 0.0;
#pragma unroll
        for (int e = 0; e < K; ++e) {
            y = fma(lam, y, r[e]);
            r[e] = y;
        }
        const double inc = warp_fwd_incl(sp, y, lane);
        if (!(task & 1)) {
            if (lane == 31) s_cin0[task >> 1] = inc;
        } else {
            double ex = __shfl_up_sync(FULL, inc, 1);
            if (lane == 0) ex = 0.0;
            double x = 0.0;
#pragma unroll
            for (int e = K - 1; e >= 0; --e) x = fma(lam, x, fma(ex, sp.pw[e], r[e]));
            const double xb = warp_bwd_incl(sp, x, lane);
            if (lane == 0) s_xbl[task >> 1] = xb;
        }
    }
    __syncthreads();
    const double zc = lam / (1.0 - lam * lam);

    long long m = 0;   // node chunks consumed
    for (int a = 0; a < tp.nact; ++a) {
        const StepItem& it = items[a];
        const int nn = it.nnodes;
        double* const udst = it.out + sp.GW;
        double cin = s_cin0[a];
        bool bad = false;
        int pend_col = -1, pend_slot = 0;
        double pend_m = 0.0;
        auto store16 = [&](int col, const double (&w)[K]) {
#pragma unroll
            for (int e = 0; e < K; e += 4) stg256(udst + col + e, w[e], w[e + 1], w[e + 2], w[e + 3]);
            if (col < 16)   // periodic ghost copies of the line's ends (the next tick's stencils)
#pragma unroll
                for (int e = 0; e < K; e += 4) stg256(udst + nx + col + e, w[e], w[e + 1], w[e + 2], w[e + 3]);
            if (col >= nx - 16)
#pragma unroll
                for (int e = 0; e < K; e += 4) stg256(udst - nx + col + e, w[e], w[e + 1], w[e + 2], w[e + 3]);
        };
        auto pend_flush = [&](double d) {
            const double dm = d * pend_m;
            double w[K];
#pragma unroll
            for (int e = 0; e < K; ++e) w[e] = fma(dm, sp.pw[K - 1 - e], s_pend[e * kSweepPend + pend_slot]);
            bad |= !chunk_finite(w);
            store16(pend_col, w);
            pend_col = -1;
        };
        for (int i = 0; i < nch; ++i) {
            const int cbase = R0 + i * Cr;
            const int len = min(Cr, R1 - cbase);
            const int nthr = len / K;
            const bool mine = tid < nthr;
            // ---- the right-hand side, node by node (each node chunk read once)
            double v[K];
#pragma unroll
            for (int e = 0; e < K; ++e) v[e] = 0.0;
            for (int n = 0; n < nn; ++n, ++m) {
                const int s = (int)(m % NS);
                mbar_wait(&full[s], (uint32_t)((m / NS) & 1));
                const char* st = stage + (size_t)s * STAGE;
                const NodeCoef nc = node_coef<KIND>(pb, it.ca[n], it.cs[n], it.cn[n]);
                const double ga = g * nc.a, gb = g * nc.b, gs = g * nc.cs * pb.cdx;
                // my points: staged group tid + 1; neighbours: group tid element 15, group tid + 2 element 0
                double wl = lds128(swz(st, tid, 7)).y;
                double2 w2 = lds128(swz(st, tid + 1, 0));
#pragma unroll
                for (int q = 0; q < K / 2; ++q) {
                    const double2 wn = q + 1 < K / 2 ? lds128(swz(st, tid + 1, q + 1))
                                                     : make_double2(lds128(swz(st, tid + 2 < 512 ? tid + 2 : 511, 0)).x, 0.0);
                    v[2 * q] = fma(gs, (wl - 2.0 * w2.x) + w2.y, fma(fma(gb, w2.x, ga), w2.x, v[2 * q]));
                    v[2 * q + 1] = fma(gs, (w2.x - 2.0 * w2.y) + wn.x, fma(fma(gb, w2.y, ga), w2.y, v[2 * q + 1]));
                    wl = w2.y;
                    w2 = wn;
                }
                __syncwarp();   // every loaded value consumed above: the stage may be refilled
                if (lane == 0) mbar_arrive(&empty[s]);
                if (tid == 0) issue_next();
            }
            // ---- forward: local recurrence, block scan with the chunk's carry-in
            double y = 0.0;
#pragma unroll
            for (int e = 0; e < K; ++e) {
                y = fma(lam, y, v[e]);
                v[e] = y;
            }
            const double bf = mine ? y : 0.0;
            double inc = warp_fwd_incl(sp, bf, lane);
            if (lane == 31) sx[warp] = inc;
            double ex = __shfl_up_sync(FULL, inc, 1);
            if (lane == 0) ex = 0.0;
            __syncthreads();
            double wi = lane < NW ? sx[lane] : 0.0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const double t = __shfl_up_sync(FULL, wi, 1 << q);
                if (lane >= (1 << q)) wi = fma(sp.mp[5 + q], t, wi);
            }
            double cw = __shfl_sync(FULL, wi, warp > 0 ? warp - 1 : 0);
            if (warp == 0) cw = 0.0;
            const double cf = fma(mt, cin, fma(ml, cw, ex));
            const double yend = fma(cf, sp.pw[K - 1], bf);
            // ---- backward with a zero carry at the chunk end
            double x = 0.0;
            if (!mine) {
#pragma unroll
                for (int e = 0; e < K; ++e) v[e] = 0.0;
            }
#pragma unroll
            for (int e = K - 1; e >= 0; --e) {
                x = fma(lam, x, v[e]);
                v[e] = x;
            }
            double rinc = mine ? fma(cf, sp.zf[0], x) : 0.0;
            rinc = warp_bwd_incl(sp, rinc, lane);
            if (lane == 0) sx[NW + warp] = rinc;
            double exr = __shfl_down_sync(FULL, rinc, 1);
            if (lane == 31) exr = 0.0;
            if (tid == nthr - 1) s_bc[0] = yend;
            __syncthreads();
            cin = s_bc[0];
            double wr = lane < NW ? sx[NW + (NW - 1 - lane)] : 0.0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const double t = __shfl_up_sync(FULL, wr, 1 << q);
                if (lane >= (1 << q)) wr = fma(sp.mp[5 + q], t, wr);
            }
            const int rl = NW - 1 - warp;
            double dw = __shfl_sync(FULL, wr, rl > 0 ? rl - 1 : 0);
            if (rl == 0) dw = 0.0;
            const double dc = fma(mr, dw, exr);
#pragma unroll
            for (int e = 0; e < K; ++e) v[e] = fma(dc, sp.pw[K - 1 - e], fma(cf, sp.zf[e], v[e]));
            // ---- the previous chunk's tail: its backward carry is my first point's x
            if (tid == 0) s_bc[1] = v[0];
            __syncthreads();
            if (pend_col >= 0) pend_flush(s_bc[1]);
            if (mine) {
                const int col = cbase + tid * K;
                if (K * (tid + 1) > len - sp.hc) {
                    pend_slot = tid - max(0, (len - sp.hc) / K);
                    RIDC_CHECK(pend_slot >= 0 && pend_slot < kSweepPend);
#pragma unroll
                    for (int e = 0; e < K; ++e) s_pend[e * kSweepPend + pend_slot] = v[e];
                    pend_col = col;
                    pend_m = 1.0;
                    const int q = nthr - 1 - tid;
#pragma unroll
                    for (int b = 0; b < 10; ++b)
                        if (q & (1 << b)) pend_m *= sp.mp[b];
                } else {
                    bad |= !chunk_finite(v);
                    store16(col, v);
                }
            }
        }
        // ---- range end: the backward carry at R1 for the last chunk's tail
        if (pend_col >= 0) pend_flush(fma(cin, zc, s_xbl[a]));
        if (bad) atomicMin(ep.err, err_code(it.target, it.level));
        __syncthreads();   // s_bc / s_pend reused by the next level
    }
}

}  // namespace ridc
