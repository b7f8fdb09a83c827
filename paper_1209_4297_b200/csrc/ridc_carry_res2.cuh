// ridc_carry_res2.cuh -- RIDC-2 (predictor + one corrector) on a periodic
// reaction-diffusion line held on the SMs for a whole restart interval.
//
// The lagged pipeline (engine.py:349-459) with p = 2: at tick k the predictor
// computes step k and the corrector step k - 2 (one more than startup_delay,
// engine.py:50-54: see the tick below), the corrector reading the predictor's
// steps k - 2 and k - 3 (its window, _window_span / _orient, engine.py:124-140;
// _correct_core, :179-187).
// Like the carry-exchange FEBE march (ridc_febe_carry.cuh), the line is one
// tile per SM and every tile solves its own points only; here each thread
// holds 16 points of BOTH levels in registers, so a tick is the FEBE step on
// two interleaved systems -- both recurrences and both block scans share the
// barriers, both carry pairs travel in the same round trip:
//   * the corrector's right-hand side folds its own state (f^N) and the two
//     predictor states with the quadrature weights and lag terms (node_coef,
//     build_item's order of nodes), the f^S stencil of the predictor states
//     read from a shared-memory ring of the predictor's last two steps (point
//     (t, e) at [e][t + 1], conflict-free); the tile-end neighbours come from
//     the neighbour tiles' published end values (LL lines, one per tile end
//     per step);
//   * both levels are solved with zero carries at the tile ends and corrected
//     with the neighbours' y_end / local first x (head: x_i += c lam^(i+1) /
//     (1 - lam^2), tail: x_i += d lam^(T-i); dropped terms below 2^-60).
// One cooperative launch per restart interval; the level finals land in ring
// slot 1 of each level (the resident level march's convention).  States agree
// with the tick kernel to rounding (different association) and with the
// oracle at <= 1e-10 (tests/test_gpu_resident.py).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "ridc_device.cuh"
#include "ridc_febe_carry.cuh"
#include "ridc_resident.cuh"

namespace ridc {

constexpr int kRes2MaxNT = 448;   // 14 warps x 16 points: tiles up to 7168 points

struct CarryRes2Params {
    double lam, inv1ml2;
    double aa, bb;                 // predictor rhs with g folded: (aa + bb u) u
    double a1, b1;                 // corrector own node (ca 1, cs 0, cn dt), g folded
    double an, bn, sn;             // node "new" (predictor step t: cs w0 - dt, cn w0), g folded, sn = g cs cdx
    double ao, bo, so;             // node "old" (predictor step t - 1: cs w1, cn w1 - dt)
    double an2, ao2;               // an - 2 sn, ao - 2 so: the f^S stencil's centre folded into the node's linear term
    double pw[16], zf[16], mp[10];
    const double* src;             // the interval's state0 (plain layout, nx doubles)
    double* fin0;                  // level finals: padded slot + GW (data column 0)
    double* fin1;
    int T, nx, nseg, hc;
    uint4* mail;                   // [4 parities][nseg][4]: y_end level 0, level 1, x_first level 0, level 1
    uint4* edge;                   // [4 parities][nseg][2]: the predictor's first / last point of a step
    unsigned tag0;                 // tick k is tagged tag0 + k
    long long per;                 // steps of the interval (ticks: per + 1)
    unsigned long long* err;
    unsigned* abort;
    long long spin_limit;
};

__device__ __forceinline__ double res2_poll(const uint4* p, unsigned want, const CarryRes2Params& cp, bool& dead)
{
    uint4 v = ld_line(p);
    if (v.y == want && v.w == want) return line_value(v);
    const long long t0 = clock64();
    for (unsigned it = 1; !dead; ++it) {   // the watchdog only every 64 polls
        v = ld_line(p);
        if (v.y == want && v.w == want) return line_value(v);
        if ((it & 63u) == 0u && (clock64() - t0 > cp.spin_limit || *(volatile unsigned*)cp.abort)) {
            atomicExch(cp.abort, 1u);
            dead = true;
        }
    }
    return 0.0;
}

constexpr int kRes2NP = kRes2MaxNT + 2;   // ring row stride (compile-time: the addressing is constant offsets)
inline size_t carry_res2_smem(int) { return (size_t)3 * 16 * kRes2NP * sizeof(double); }

template <int KIND>
__global__ void __launch_bounds__(kRes2MaxNT, 1) k_carry_res2(const __grid_constant__ CarryRes2Params cp)
{
    static_assert(KIND == RD_1D, "resident RIDC-2: periodic reaction-diffusion lines");
    constexpr int K = 16;
    extern __shared__ double ring[];               // [3 slots][16][NP]: predictor steps, [e][thread + 1]
    __shared__ double sx[4 * (kRes2MaxNT / 32)];   // block-scan warp totals: fwd 0, fwd 1, bwd 0, bwd 1
    __shared__ double s_yend[2];
    const unsigned FULL = 0xffffffffu;
    const int NT = blockDim.x, NW = NT >> 5;
    constexpr int NP = kRes2NP;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int k = blockIdx.x, nseg = cp.nseg;
    const int c0 = k * cp.T;
    const int Tk = min(cp.T, cp.nx - c0);
    const int nch = Tk / K;
    const bool mine = tid < nch;
    const int i0 = tid * K;
    const bool head = mine && i0 < cp.hc;
    const bool tail = mine && i0 + K > Tk - cp.hc;
    const bool head_warp = warp * 32 * K < cp.hc;
    const bool tail_warp = (warp * 32 + 31) * K + K > Tk - cp.hc && warp * 32 < nch;
    const bool last = tid == nch - 1;
    RIDC_CHECK(nch <= NT && Tk % K == 0 && Tk >= 2 * cp.hc && c0 + Tk <= cp.nx);
    const int kl = k == 0 ? nseg - 1 : k - 1, kr = k == nseg - 1 ? 0 : k + 1;
    const double lam = cp.lam;

    double Mh = cp.inv1ml2, Mt = 1.0, ml = 1.0, mr = 1.0;
    {
        const int q = mine ? nch - 1 - tid : 0;
#pragma unroll
        for (int i = 0; i < 10; ++i) {
            if (tid & (1 << i)) Mh *= cp.mp[i];
            if (q & (1 << i)) Mt *= cp.mp[i];
        }
#pragma unroll
        for (int i = 0; i < 5; ++i) {
            if (lane & (1 << i)) ml *= cp.mp[i];
            if ((31 - lane) & (1 << i)) mr *= cp.mp[i];
        }
    }
    auto R = [&](int slot, int e, int col) -> double& { return ring[(slot * K + e) * NP + col]; };

    // ---- state0: both levels, and the predictor's step 0 in ring slot 0 (+ its end neighbours)
    double u0[K], u1[K];
    if (mine) {
        load_chunk_cg(cp.src + c0 + i0, u0);
    } else {
#pragma unroll
        for (int e = 0; e < K; ++e) u0[e] = 0.0;
    }
#pragma unroll
    for (int e = 0; e < K; ++e) u1[e] = u0[e];
    if (mine)
#pragma unroll
        for (int e = 0; e < K; ++e) R(0, e, tid + 1) = u0[e];
    if (tid == 0) R(0, K - 1, 0) = __ldcg(cp.src + (c0 == 0 ? cp.nx - 1 : c0 - 1));
    if (last) R(0, 0, nch + 1) = __ldcg(cp.src + (c0 + Tk == cp.nx ? 0 : c0 + Tk));
    bool dead = false;

    // one tick: A0 -- the predictor computes step kk, A1 -- the corrector step kk - 2
    // (a lag of two instead of the tick engine's one: the newest predictor step a
    // fold reads was stored before the LAST tick's barriers, so a tick needs no
    // barrier of its own before the fold; the same level-steps, computed alike).
    // Ring slot of predictor step s: s % 3 (r3 = kk % 3).
    auto tick = [&](long long kk, int r3, auto a0c, auto a1c) {
        constexpr bool A0 = decltype(a0c)::value, A1 = decltype(a1c)::value;
        const unsigned tag = cp.tag0 + (unsigned)kk;
        uint4* box = cp.mail + (size_t)(kk & 3) * 4 * nseg;
        uint4* ebox = cp.edge + (size_t)((kk - 2) & 3) * 2 * nseg;
        const int sn = r3 == 2 ? 0 : r3 + 1, so = r3;   // ring slots: predictor steps kk-2, kk-3 (then kk)
        // the neighbour tiles' end points of predictor step kk-2 (published two ticks ago),
        // kept in the ring's end cells that only threads 0 and nch-1 read
        if (A1) {
            if (tid == 0) R(sn, K - 1, 0) = res2_poll(ebox + 2 * kl + 1, cp.tag0 + (unsigned)(kk - 2), cp, dead);
            if (last) R(sn, 0, nch + 1) = res2_poll(ebox + 2 * kr, cp.tag0 + (unsigned)(kk - 2), cp, dead);
        }
        // ---- right-hand sides (g folded in)
        if (A0) {
#pragma unroll
            for (int e = 0; e < K; ++e) u0[e] = fma(cp.bb, u0[e], cp.aa) * u0[e];
        }
        if (A1) {
            const double* Pn = ring + sn * K * NP + tid + 1;   // point (tid, e) of step kk-2 at Pn[e NP]
            const double* Po = ring + so * K * NP + tid + 1;   // step kk-3
            double nl = Pn[(K - 1) * NP - 1], nc = Pn[0], ol = Po[(K - 1) * NP - 1], oc = Po[0];
#pragma unroll
            for (int e = 0; e < K; ++e) {
                const double nr = e == K - 1 ? Pn[1] : Pn[(e + 1) * NP];
                const double orr = e == K - 1 ? Po[1] : Po[(e + 1) * NP];
                double r = fma(cp.b1, u1[e], cp.a1) * u1[e];
                r = fma(cp.sn, nl + nr, fma(fma(cp.bn, nc, cp.an2), nc, r));   // an2 = an - 2 sn
                r = fma(cp.so, ol + orr, fma(fma(cp.bo, oc, cp.ao2), oc, r));
                u1[e] = r;
                nl = nc; nc = nr; ol = oc; oc = orr;
            }
        }
        if (A1 && !mine) {   // threads past the tile feed zeros into the scans
#pragma unroll
            for (int e = 0; e < K; ++e) u1[e] = 0.0;
        }
        // ---- local forward recurrences (zero carry in)
        double y0 = 0.0, y1 = 0.0;
#pragma unroll
        for (int e = 0; e < K; ++e) {
            if (A0) { y0 = fma(lam, y0, u0[e]); u0[e] = y0; }
            if (A1) { y1 = fma(lam, y1, u1[e]); u1[e] = y1; }
        }
        const double bf0 = mine ? y0 : 0.0, bf1 = mine ? y1 : 0.0;
        double inc0 = bf0, inc1 = bf1;
#pragma unroll
        for (int i = 0; i < 5; ++i) {   // multipliers from the constant bank: no registers held
            const double t0 = A0 ? __shfl_up_sync(FULL, inc0, 1 << i) : 0.0;
            const double t1 = A1 ? __shfl_up_sync(FULL, inc1, 1 << i) : 0.0;
            if (lane >= (1 << i)) {
                if (A0) inc0 = fma(cp.mp[i], t0, inc0);
                if (A1) inc1 = fma(cp.mp[i], t1, inc1);
            }
        }
        if (lane == 31) { sx[warp] = inc0; sx[NW + warp] = inc1; }
        double ex0 = __shfl_up_sync(FULL, inc0, 1), ex1 = __shfl_up_sync(FULL, inc1, 1);
        if (lane == 0) { ex0 = 0.0; ex1 = 0.0; }
        __syncthreads();
        double wi0 = lane < NW ? sx[lane] : 0.0, wi1 = lane < NW ? sx[NW + lane] : 0.0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const double t0 = __shfl_up_sync(FULL, wi0, 1 << i), t1 = __shfl_up_sync(FULL, wi1, 1 << i);
            if (lane >= (1 << i)) { wi0 = fma(cp.mp[5 + i], t0, wi0); wi1 = fma(cp.mp[5 + i], t1, wi1); }
        }
        double cw0 = __shfl_sync(FULL, wi0, warp > 0 ? warp - 1 : 0), cw1 = __shfl_sync(FULL, wi1, warp > 0 ? warp - 1 : 0);
        if (warp == 0) { cw0 = 0.0; cw1 = 0.0; }
        const double cf0 = fma(ml, cw0, ex0), cf1 = fma(ml, cw1, ex1);
        // 1. y at my tile's last point, both levels (the right neighbour's forward carries)
        if (last) {
            const double ye0 = fma(cf0, cp.pw[K - 1], bf0), ye1 = fma(cf1, cp.pw[K - 1], bf1);
            if (!dead) {
                if (A0) st_line(box + 4 * k + 0, ye0, tag);
                if (A1) st_line(box + 4 * k + 1, ye1, tag);
            }
            s_yend[0] = ye0;
            s_yend[1] = ye1;
        }
        // ---- local backward recurrences (zero carry at the tile end)
        double x0 = 0.0, x1 = 0.0;
#pragma unroll
        for (int e = K - 1; e >= 0; --e) {
            if (A0) { x0 = fma(lam, x0, u0[e]); u0[e] = x0; }
            if (A1) { x1 = fma(lam, x1, u1[e]); u1[e] = x1; }
        }
        double rinc0 = mine ? fma(cf0, cp.zf[0], x0) : 0.0, rinc1 = mine ? fma(cf1, cp.zf[0], x1) : 0.0;
#pragma unroll
        for (int i = 0; i < 5; ++i) {
            const double t0 = A0 ? __shfl_down_sync(FULL, rinc0, 1 << i) : 0.0;
            const double t1 = A1 ? __shfl_down_sync(FULL, rinc1, 1 << i) : 0.0;
            if (lane + (1 << i) < 32) {
                if (A0) rinc0 = fma(cp.mp[i], t0, rinc0);
                if (A1) rinc1 = fma(cp.mp[i], t1, rinc1);
            }
        }
        if (lane == 0) { sx[2 * NW + warp] = rinc0; sx[3 * NW + warp] = rinc1; }
        double exr0 = __shfl_down_sync(FULL, rinc0, 1), exr1 = __shfl_down_sync(FULL, rinc1, 1);
        if (lane == 31) { exr0 = 0.0; exr1 = 0.0; }
        __syncthreads();
        double wr0 = lane < NW ? sx[2 * NW + (NW - 1 - lane)] : 0.0, wr1 = lane < NW ? sx[3 * NW + (NW - 1 - lane)] : 0.0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const double t0 = __shfl_up_sync(FULL, wr0, 1 << i), t1 = __shfl_up_sync(FULL, wr1, 1 << i);
            if (lane >= (1 << i)) { wr0 = fma(cp.mp[5 + i], t0, wr0); wr1 = fma(cp.mp[5 + i], t1, wr1); }
        }
        const int rl = NW - 1 - warp;
        double dw0 = __shfl_sync(FULL, wr0, rl > 0 ? rl - 1 : 0), dw1 = __shfl_sync(FULL, wr1, rl > 0 ? rl - 1 : 0);
        if (rl == 0) { dw0 = 0.0; dw1 = 0.0; }
        const double dc0 = fma(mr, dw0, exr0), dc1 = fma(mr, dw1, exr1);
#pragma unroll
        for (int e = 0; e < K; ++e) {
            if (A0) u0[e] = fma(dc0, cp.pw[K - 1 - e], fma(cf0, cp.zf[e], u0[e]));
            if (A1) u1[e] = fma(dc1, cp.pw[K - 1 - e], fma(cf1, cp.zf[e], u1[e]));
        }
        // 2. my first point's LOCAL x, both levels (the left neighbour completes it)
        if (tid == 0 && !dead) {
            if (A0) st_line(box + 4 * k + 2, u0[0], tag);
            if (A1) st_line(box + 4 * k + 3, u1[0], tag);
        }
        // ---- head: the left neighbour's forward carries
        if (head_warp) {
            // lane 0 waits for level 0's line, lane 1 for level 1's, in one loop
            double cv = 0.0;
            if ((A0 && lane == 0) || (A1 && lane == 1)) cv = res2_poll(box + 4 * kl + lane, tag, cp, dead);
            const double ca = __shfl_sync(FULL, cv, 0) * Mh;
            const double cb = __shfl_sync(FULL, cv, 1) * Mh;
            if (head) {
#pragma unroll
                for (int e = 0; e < K; ++e) {
                    if (A0) u0[e] = fma(ca, cp.pw[e], u0[e]);
                    if (A1) u1[e] = fma(cb, cp.pw[e], u1[e]);
                }
            }
        }
        // ---- tail: the right neighbour's backward carries (its local first x + the
        // head correction my own y_end causes there)
        if (tail_warp) {
            double dv = 0.0;
            if ((A0 && lane == 0) || (A1 && lane == 1))
                dv = fma(s_yend[lane] * cp.inv1ml2, cp.pw[0], res2_poll(box + 4 * kr + 2 + lane, tag, cp, dead));
            const double da = __shfl_sync(FULL, dv, 0) * Mt;
            const double db = __shfl_sync(FULL, dv, 1) * Mt;
            if (tail) {
#pragma unroll
                for (int e = 0; e < K; ++e) {
                    if (A0) u0[e] = fma(da, cp.pw[K - 1 - e], u0[e]);
                    if (A1) u1[e] = fma(db, cp.pw[K - 1 - e], u1[e]);
                }
            }
        }
        // ---- finite checks (engine.py:160-164); the predictor's new step into the ring
        // (threads past the tile carry garbage that never leaves them: their scan
        // inputs are masked to zero, they store nothing and publish nothing)
        if (mine) {
            if (A0 && !chunk_finite(u0)) atomicMin(cp.err, err_code(kk, 0));
            if (A1 && !chunk_finite(u1)) atomicMin(cp.err, err_code(kk - 2, 1));
            if (A0) {   // step kk over step kk-3 (read above, before this tick's barriers)
                double* Pw = ring + so * K * NP + tid + 1;
#pragma unroll
                for (int e = 0; e < K; ++e) Pw[e * NP] = u0[e];
            }
        }
        if (A0 && !dead) {   // my tile's end points of predictor step kk (the neighbours' stencils)
            uint4* eb = cp.edge + (size_t)(kk & 3) * 2 * nseg;
            if (tid == 0) st_line(eb + 2 * k, u0[0], tag);
            if (last) st_line(eb + 2 * k + 1, u0[K - 1], tag);
        }
    };

    const std::true_type on;
    const std::false_type off;
#pragma unroll 1
    for (int kk = 1; kk <= 2; ++kk) tick(kk, kk, on, off);
    int r3 = 0;
#pragma unroll 1
    for (long long kk = 3; kk <= cp.per; ++kk) {
        tick(kk, r3, on, on);
        r3 = r3 == 2 ? 0 : r3 + 1;
    }
#pragma unroll 1
    for (long long kk = cp.per + 1; kk <= cp.per + 2; ++kk) tick(kk, (int)(kk % 3), off, on);
    if (mine) {
#pragma unroll
        for (int e = 0; e < K; e += 2) {
            *reinterpret_cast<double2*>(cp.fin0 + c0 + i0 + e) = make_double2(u0[e], u0[e + 1]);
            *reinterpret_cast<double2*>(cp.fin1 + c0 + i0 + e) = make_double2(u1[e], u1[e + 1]);
        }
    }
}

}  // namespace ridc
