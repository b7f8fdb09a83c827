// ridc_sweep_warp.cuh -- streaming FEBE step for long periodic lines, one
// independent sweep per WARP (RIDC order 1, reaction-diffusion, lines of
// >= 512 x 12 x SMs points: C5 2^20 .. 2^26).
//
// One launch per time step (engine.py:167-175 _predict_core over the whole
// line).  Round 2's CTA sweep (ridc_sweep.cuh) lets one 512-thread CTA sweep
// its range in 8192-point chunks; each chunk costs three block barriers and
// two block scans, and ncu shows the SM idling on them (barrier 27%, long_sb
// 19% of stall samples, DRAM 39% of peak at 2^24: profiles/r2_sweep_2p24_ncu.txt).
// Here every warp owns a contiguous sub-range of the line (~N / (12 x 148)
// points) and sweeps it in 512-point chunks (16 points per lane) on its own:
// no block barrier anywhere in the step, twelve independent sweeps per SM
// hide each other's scan latency, and each warp keeps three 4 KB TMA loads in
// flight (144 KB per SM).  384 threads per SM leave 168 registers per thread:
// the chunk in flight and the pending one stay in registers without spills.  Every point is still read once and written once
// (16 B/pt) plus the 2 x 512 points around each sub-range.
//
// The shifted solve (I - dt L_S) x = rhs factors into  y_i = g rhs_i + lam y_{i-1}
// (forward) and  x_i = y_i + lam x_{i+1}  (backward), ridc_device.cuh.  Along a
// warp's sweep:
//   * load 0, the 512 points before the sub-range: a truncated forward pass
//     gives the forward carry into it (cin);
//   * load 1, the 512 points after it: a truncated forward + backward pass
//     with zero carry at its start gives X0; the backward carry at the range
//     end is X0 + y_end lam / (1 - lam^2) once the range's last y is known
//     (the response of x there to a unit forward carry);
//   * loads 2.. are the chunks: the forward carry enters each chunk's warp
//     scan exactly; the backward pass runs with a zero carry at the chunk end
//     and the chunk is kept in registers one iteration, until the next chunk's
//     first x is known (its own carry from two chunks ahead is lam^512 <=
//     2^-60 relative: hc <= 512), then corrected and stored with 256-bit
//     stores.  The last chunk is corrected with the range-end carry first, so
//     it may be short.
// Dropped terms are all below 2^-60 relative (the same truncation as the tick
// kernel's segment halos): the states agree with the tick kernel and the
// CTA sweep to rounding and with the oracle at <= 1e-10
// (tests/test_gpu_fullsize.py C5 sizes).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "ridc_sweep.cuh"

namespace ridc {

constexpr int kWarpSweepStages = 4;
constexpr int kWarpSweepWarps = 12;   // 384-thread CTAs, one per SM (<= 168 registers: no spills)
constexpr int kWarpChunk = 512;       // points per warp chunk (16 per lane)
constexpr size_t warp_sweep_smem()
{
    return (size_t)kWarpSweepWarps * kWarpSweepStages * kWarpChunk * sizeof(double) + 1024;
}

template <int KIND>
__global__ void __launch_bounds__(kWarpSweepWarps * 32, 1)
    k_sweep_febe_warp(const __grid_constant__ SweepParams sp, const __grid_constant__ TmapSet tm, long long off,
                      long long target)
{
    static_assert(KIND == RD_1D, "streaming FEBE sweep: periodic reaction-diffusion lines");
    constexpr int K = 16, NS = kWarpSweepStages, NW = kWarpSweepWarps;
    constexpr uint32_t SB = kWarpChunk * sizeof(double);   // bytes per stage
    extern __shared__ __align__(1024) char smraw[];
    char* base = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t s_full[NW * NS];
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    char* stage = base + (size_t)warp * NS * SB;
    uint64_t* full = s_full + warp * NS;
    const int nx = sp.nx;
    const long long n16 = nx / 16, nwt = (long long)gridDim.x * NW, W = (long long)blockIdx.x * NW + warp;
    const int R0 = 16 * (int)(W * n16 / nwt), R1 = 16 * (int)((W + 1) * n16 / nwt);
    const int nch = (R1 - R0 + kWarpChunk - 1) / kWarpChunk;
    const int nload = nch + 2;
    const long long src = (off + target - 1) % sp.cap, dst = (off + target) % sp.cap;
    RIDC_CHECK(src != dst && R1 - R0 >= kWarpChunk && nx >= 2 * kWarpChunk && sp.hc <= kWarpChunk);
    double* udst = sp.ring + dst * sp.Vs + sp.GW;   // data column 0
    const double lam = sp.lam;

    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (lane == 0) {
        for (int i = 0; i < NS; ++i) mbar_init(&full[i], 1);
        mbar_fence_init();
    }
    // M^lane, M^(31-lane)
    double ml = 1.0, mr = 1.0;
#pragma unroll
    for (int i = 0; i < 5; ++i) {
        if (lane & (1 << i)) ml *= sp.mp[i];
        if ((31 - lane) & (1 << i)) mr *= sp.mp[i];
    }
    // the last chunk: lanes holding points, M^(nthr_last - 1 - lane)
    const int len_last = R1 - R0 - (nch - 1) * kWarpChunk;
    const int nthr_last = len_last / K;
    double mlast = 1.0;
    {
        const int q = nthr_last - 1 - lane;
#pragma unroll
        for (int i = 0; i < 5; ++i)
            if (q >= 0 && (q & (1 << i))) mlast *= sp.mp[i];
    }
    __syncthreads();   // barrier inits visible to every lane and to the TMA unit
    // load m: 0 = the 512 points before R0, 1 = the 512 after R1, 2 + i = chunk i
    auto issue = [&](int m) {   // lane 0
        const int s = m % NS;
        int col = m == 0 ? (R0 == 0 ? nx : R0) - kWarpChunk : m == 1 ? (R1 == nx ? 0 : R1) : R0 + (m - 2) * kWarpChunk;
        mbar_arrive_expect_tx(&full[s], SB);
        tma_load_3d(stage + (size_t)s * SB, &tm.map[0], 0, sp.gdata + col / 16, (int)src, &full[s]);
    };
    // every read of the previous step's state waits for the previous launch
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (lane == 0)
        for (int m = 0; m < NS && m < nload; ++m) issue(m);

    double v[K];
    auto take = [&](int m) {   // my 16 points of load m (swizzled)
        mbar_wait(&full[m % NS], (uint32_t)((m / NS) & 1));
        const char* st = stage + (size_t)(m % NS) * SB;
#pragma unroll
        for (int q = 0; q < K / 2; ++q) {
            const double2 w = lds128(swz(st, lane, q));
            v[2 * q] = w.x;
            v[2 * q + 1] = w.y;
        }
    };
    // forward local recurrence over the rhs (consumes every staged value), then
    // the stage goes back to lane 0 for load m + NS
    auto forward_local = [&](int m) {
        double y = 0.0;
#pragma unroll
        for (int e = 0; e < K; ++e) {
            y = fma(lam, y, sweep_rhs(sp, v[e]));
            v[e] = y;
        }
        __syncwarp();
        if (lane == 0 && m + NS < nload) issue(m + NS);
        return y;
    };

    // ---- load 0: forward carry into R0
    take(0);
    double cin = __shfl_sync(FULL, warp_fwd_incl(sp, forward_local(0), lane), 31);
    // ---- load 1: x at R1 with zero forward carry into it (truncated at 512 points)
    double X0;
    {
        take(1);
        const double yl = forward_local(1);
        const double inc = warp_fwd_incl(sp, yl, lane);
        double ex = __shfl_up_sync(FULL, inc, 1);
        if (lane == 0) ex = 0.0;
        double x = 0.0;
#pragma unroll
        for (int e = K - 1; e >= 0; --e) x = fma(lam, x, fma(ex, sp.pw[e], v[e]));
        X0 = __shfl_sync(FULL, warp_bwd_incl(sp, x, lane), 0);
    }
    const double zc = lam / fma(-lam, lam, 1.0);   // x at R1 per unit forward carry into R1

    bool bad = false;
    double pend[K];
    int pend_col = 0;
    for (int i = 0; i < nch; ++i) {
        const int m = i + 2;
        const bool last = i == nch - 1;
        const int cbase = R0 + i * kWarpChunk;
        const int nthr = last ? nthr_last : 32;
        const bool mine = lane < nthr;
        take(m);
        const double yl = forward_local(m);
        // ---- forward carries: the warp scan with the chunk's carry-in
        const double bf = mine ? yl : 0.0;
        const double inc = warp_fwd_incl(sp, bf, lane);
        double ex = __shfl_up_sync(FULL, inc, 1);
        if (lane == 0) ex = 0.0;
        const double cf = fma(ml, cin, ex);   // carry into my 16 points
        cin = __shfl_sync(FULL, fma(cf, sp.pw[K - 1], bf), nthr - 1);   // y at the chunk's last point
        // ---- backward with a zero carry at the chunk end
        if (!mine) {
#pragma unroll
            for (int e = 0; e < K; ++e) v[e] = 0.0;
        }
        double x = 0.0;
#pragma unroll
        for (int e = K - 1; e >= 0; --e) {
            x = fma(lam, x, v[e]);
            v[e] = x;
        }
        const double rinc = warp_bwd_incl(sp, mine ? fma(cf, sp.zf[0], x) : 0.0, lane);
        double exr = __shfl_down_sync(FULL, rinc, 1);
        if (lane == 31) exr = 0.0;
        if (last) {   // the range-end carry (x at R1) reaches the last chunk before anything reads it
            const double dend = fma(cin, zc, X0);
            exr = fma(dend, mlast, exr);
        }
#pragma unroll
        for (int e = 0; e < K; ++e) v[e] = fma(exr, sp.pw[K - 1 - e], fma(cf, sp.zf[e], v[e]));
        // ---- the previous chunk: its backward carry is my first point's x
        const double d = __shfl_sync(FULL, v[0], 0);
        if (i > 0) {
            const double dm = d * mr;
            double w[K];
#pragma unroll
            for (int e = 0; e < K; ++e) w[e] = fma(dm, sp.pw[K - 1 - e], pend[e]);
            bad |= !chunk_finite(w);
            RIDC_CHECK(pend_col >= R0 && pend_col + K <= R1);
#pragma unroll
            for (int e = 0; e < K; e += 4) stg256(udst + pend_col + e, w[e], w[e + 1], w[e + 2], w[e + 3]);
        }
        if (last) {
            if (mine) {
                const int col = cbase + lane * K;
                RIDC_CHECK(col >= R0 && col + K <= R1);
                bad |= !chunk_finite(v);
#pragma unroll
                for (int e = 0; e < K; e += 4) stg256(udst + col + e, v[e], v[e + 1], v[e + 2], v[e + 3]);
            }
        } else {
#pragma unroll
            for (int e = 0; e < K; ++e) pend[e] = v[e];
            pend_col = cbase + lane * K;
        }
    }
    if (bad) atomicMin(sp.err, err_code((target - 1) % sp.per + 1, 0));
}

}  // namespace ridc
