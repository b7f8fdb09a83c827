// ridc_carry_res2w.cuh -- resident RIDC-2 with one 512-point chunk per WARP
// (both levels), the warp carry march's schedule (ridc_febe_carry.cuh,
// k_febe_wcarry) applied to the lagged two-level pipeline of k_carry_res2.
//
// The tick is k_carry_res2's (engine.py:349-459 with p = 2: at tick k the
// predictor computes step k and the corrector step k - 2 from the predictor's
// steps k - 2 and k - 3; node_coef's coefficients, build_item's node order).
// k_carry_res2 solves a whole tile per CTA with block scans (two block
// barriers per tick: 21% of its stall samples, profiles/r2_res2_c2_ncu.txt).
// Here every warp owns 512 points of both levels and solves them with warp
// scans only; neighbouring chunks are coupled exactly by two carries per
// level per tick (the one-hop rule, y_end and the local first x): tagged lines
// in shared memory between the warps of a CTA, through L2 across CTAs, every
// one-lane store / load predicated and every wait a warp vote (as the warp
// FEBE march).  No block barrier after the start.
//
// The corrector's f^S stencil reads the predictor's steps k - 2 and k - 3 from
// a shared-memory ring (3 slots, point (t, e) at [e][t + 1], k_carry_res2's
// layout) including the neighbour threads' end points.  Across a warp edge the
// ordering comes from the carry lines: the writer lane (lane 31 of the left
// warp, lane 0 of the right one) stores its ring cell at the end of tick k,
// fences (cta) and publishes its tick-(k+1) line; the reader warp waits for
// that line at the end of its tick k + 1, fences and syncs the warp before its
// tick-(k+2) fold (release / acquire, then bar.warp.sync's ordering among the
// lanes: the lane that waited need not be the reading one).  A slot is overwritten (step k over
// step k - 3) only at the end of the writer's tick k, after it has seen the
// reader's tick-k line, which the reader publishes after its tick-k fold.
// Across a CTA edge the end points travel as tagged edge lines
// (k_carry_res2's, two ticks old when read).
// One CTA per SM of 7 or 14 warps (128 registers); states agree with the
// tick kernel to rounding and with k_carry_res2 (tests/test_gpu_resident.py).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "ridc_carry_res2.cuh"
#include "ridc_febe_carry.cuh"

namespace ridc {

constexpr int kR2wWarps = 7;   // warps per CTA while one CTA per SM holds the line; else 14
__host__ __device__ constexpr int r2w_np(int w) { return w * 32 + 2; }   // ring row stride
inline size_t carry_res2w_smem(int w) { return (size_t)3 * 16 * r2w_np(w) * sizeof(double); }

// Wait (one lane or none per call site, every lane of the warp calls it) for a
// tagged line: the first load predicated, then one vote; the re-poll loop is
// warp-uniform.  Returns 0 for lanes without `need` (or after the watchdog).
__device__ __forceinline__ double r2w_wait(bool need, const uint4* p, unsigned want, const CarryRes2Params& cp,
                                           bool& dead)
{
    uint4 v = ld_line_if(need && !dead, p);
    bool ok = !need || dead || (v.y == want && v.w == want);
    if (!__all_sync(0xffffffffu, ok)) {
        const long long t0 = clock64();
        for (unsigned it = 1; !__all_sync(0xffffffffu, ok); ++it) {
            if (!ok) {
                v = ld_line_gen(p);
                ok = v.y == want && v.w == want;
                if (!ok && (it & 63u) == 0u && (clock64() - t0 > cp.spin_limit || *(volatile unsigned*)cp.abort)) {
                    atomicExch(cp.abort, 1u);
                    dead = true;
                    ok = true;
                }
            }
        }
    }
    return need && !dead ? line_value(v) : 0.0;
}

// W: warps per CTA (cp.T); cp.nseg: chunks of the line (512 points);
// cp.mail: [2 parities][nseg][4] lines (y_end level 0, level 1, first x level 0,
// level 1); cp.edge: [4 parities][CTAs][2] (a CTA's first / last predictor point)
template <int KIND, int W>
__global__ void __launch_bounds__(W * 32, W <= 7 ? 2 : 1) k_carry_res2w(const __grid_constant__ CarryRes2Params cp)
{
    static_assert(KIND == RD_1D, "resident RIDC-2: periodic reaction-diffusion lines");
    constexpr int K = 16, CH = 32 * K, NP = r2w_np(W);
    extern __shared__ double ring[];   // [3 slots][16][NP]
    __shared__ uint4 s_line[2][W][4];
    const unsigned FULL = 0xffffffffu;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wpc = cp.T, nch = cp.nseg, ncta = gridDim.x, k = blockIdx.x;
    const int nwk = min(wpc, nch - k * wpc);   // my CTA's warps (chunks)
    if (tid < 2 * W * 4) reinterpret_cast<uint4*>(s_line)[tid] = make_uint4(0u, 0u, 0u, 0u);
    const int chunk = k * wpc + warp;
    const bool active = warp < nwk;
    const int c0 = chunk * CH + lane * K;   // data column of my first point
    const int ntk = nwk * 32;               // my CTA's threads with points
    const int kl = k == 0 ? ncta - 1 : k - 1, kr = k == ncta - 1 ? 0 : k + 1;
    const int cl = chunk == 0 ? nch - 1 : chunk - 1, cr = chunk == nch - 1 ? 0 : chunk + 1;
    const bool left_local = warp > 0, right_local = warp + 1 < nwk;
    const double lam = cp.lam, ilam = 1.0 / lam;
    RIDC_CHECK(nwk >= 1 && wpc == W && cp.hc <= CH && nch * CH == cp.nx);
    auto R = [&](int slot, int e, int col) -> double& { return ring[(slot * K + e) * NP + col]; };

    double ml = 1.0, mr = 1.0;
#pragma unroll
    for (int i = 0; i < 5; ++i) {
        if (lane & (1 << i)) ml *= cp.mp[i];
        if ((31 - lane) & (1 << i)) mr *= cp.mp[i];
    }
    const double xw = ml * cp.inv1ml2 * ilam, zc = lam * cp.inv1ml2, zk = lam * cp.pw[K - 1];

    // ---- state0: both levels, the predictor's step 0 in ring slot 0 (+ the CTA's end neighbours)
    double u0[K], u1[K];
    if (active) {
        load_chunk_cg(cp.src + c0, u0);
#pragma unroll
        for (int e = 0; e < K; ++e) R(0, e, tid + 1) = u0[e];
        if (tid == 0) R(0, K - 1, 0) = __ldcg(cp.src + (c0 == 0 ? cp.nx - 1 : c0 - 1));
        if (tid == ntk - 1) R(0, 0, ntk + 1) = __ldcg(cp.src + (c0 + K == cp.nx ? 0 : c0 + K));
    } else {
#pragma unroll
        for (int e = 0; e < K; ++e) u0[e] = 0.0;
    }
#pragma unroll
    for (int e = 0; e < K; ++e) u1[e] = u0[e];
    __syncthreads();   // the one barrier: ring slot 0 and the zeroed lines
    if (!active) return;
    bool dead = false;

    // two interleaved warp scans with multiplier M = lam^16 from the constant bank
    auto scan_fwd = [&](double& a, double& b, bool ea, bool eb) {
#pragma unroll
        for (int i = 0; i < 5; ++i) {
            const double ta = ea ? __shfl_up_sync(FULL, a, 1 << i) : 0.0;
            const double tb = eb ? __shfl_up_sync(FULL, b, 1 << i) : 0.0;
            if (lane >= (1 << i)) {
                if (ea) a = fma(cp.mp[i], ta, a);
                if (eb) b = fma(cp.mp[i], tb, b);
            }
        }
    };
    auto scan_bwd = [&](double& a, double& b, bool ea, bool eb) {
#pragma unroll
        for (int i = 0; i < 5; ++i) {
            const double ta = ea ? __shfl_down_sync(FULL, a, 1 << i) : 0.0;
            const double tb = eb ? __shfl_down_sync(FULL, b, 1 << i) : 0.0;
            if (lane + (1 << i) < 32) {
                if (ea) a = fma(cp.mp[i], ta, a);
                if (eb) b = fma(cp.mp[i], tb, b);
            }
        }
    };

    // one tick: A0 -- the predictor computes step kk, A1 -- the corrector step kk - 2
    auto tick = [&](long long kk, int r3, auto a0c, auto a1c) {
        constexpr bool A0 = decltype(a0c)::value, A1 = decltype(a1c)::value;
        const unsigned tag = cp.tag0 + (unsigned)kk;
        const int par = (int)(kk & 1);
        uint4* box = cp.mail + (size_t)par * 4 * nch;
        const int sn = r3 == 2 ? 0 : r3 + 1, so = r3;   // ring slots: predictor steps kk-2, kk-3 (then kk)
        // the neighbour CTAs' end points of predictor step kk-2 (edge lines, two ticks old)
        if (A1) {
            const uint4* eb = cp.edge + (size_t)((kk - 2) & 3) * 2 * ncta;
            const bool nl = tid == 0, nr = tid == ntk - 1;
            const double v = r2w_wait(nl || nr, nl ? eb + 2 * kl + 1 : eb + 2 * kr, cp.tag0 + (unsigned)(kk - 2), cp, dead);
            if (nl) R(sn, K - 1, 0) = v;
            if (nr) R(sn, 0, ntk + 1) = v;
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
        // ---- the carries: the forward scans fed by the recurrences, the first x
        // published after the backward scans.  (Published before the
        // recurrences from dot products of the right-hand sides, as the warp
        // FEBE march does, they cost more FP64 issue than the hidden hop saves:
        // two CTAs per SM are issue bound, and one CTA per SM measured the same,
        // profiles/r2_res2w.json.)
        const bool pub = !dead;
        uint4* xl = left_local ? &s_line[par][warp][2] : box + 4 * chunk + 2;
        uint4* yl = right_local ? &s_line[par][warp][0] : box + 4 * chunk;
        // ---- the local forward recurrences (zero carry in) and their warp scans
        double y0 = 0.0, y1 = 0.0;
#pragma unroll
        for (int e = 0; e < K; ++e) {
            if (A0) { y0 = fma(lam, y0, u0[e]); u0[e] = y0; }
            if (A1) { y1 = fma(lam, y1, u1[e]); u1[e] = y1; }
        }
        double inc0 = y0, inc1 = y1;
        scan_fwd(inc0, inc1, A0, A1);
        double cf0 = __shfl_up_sync(FULL, inc0, 1), cf1 = __shfl_up_sync(FULL, inc1, 1);
        if (lane == 0) { cf0 = 0.0; cf1 = 0.0; }
        const double ye0 = __shfl_sync(FULL, inc0, 31), ye1 = __shfl_sync(FULL, inc1, 31);
        st_line_if(A0 && lane == 31 && pub, yl, ye0, tag);
        st_line_if(A1 && lane == 31 && pub, yl + 1, ye1, tag);
        // ---- the local backward recurrences (zero carry at the chunk end)
        double x0 = 0.0, x1 = 0.0;
#pragma unroll
        for (int e = K - 1; e >= 0; --e) {
            if (A0) { x0 = fma(lam, x0, u0[e]); u0[e] = x0; }
            if (A1) { x1 = fma(lam, x1, u1[e]); u1[e] = x1; }
        }
        // the neighbours' lines: lanes 0 / 1 the left chunk's y_end (level 0 / 1),
        // lanes 30 / 31 the right chunk's first x (level 0 / 1)
        const int lev = lane & 1;
        const bool need = (lane == 0 && A0) || (lane == 1 && A1) || (lane == 30 && A0) || (lane == 31 && A1);
        const uint4* src = lane < 2 ? (left_local ? &s_line[par][warp - 1][lev] : box + 4 * cl + lev)
                                    : (right_local ? &s_line[par][warp + 1][2 + lev] : box + 4 * cr + 2 + lev);
        double rinc0 = fma(cf0, cp.zf[0], x0), rinc1 = fma(cf1, cp.zf[0], x1);
        scan_bwd(rinc0, rinc1, A0, A1);
        double exr0 = __shfl_down_sync(FULL, rinc0, 1), exr1 = __shfl_down_sync(FULL, rinc1, 1);
        if (lane == 31) { exr0 = 0.0; exr1 = 0.0; }
        // lane 0: no forward carry inside the warp, only the backward one
        st_line_if(A0 && lane == 0 && pub, xl, fma(exr0, cp.pw[K - 1], u0[0]), tag);
        st_line_if(A1 && lane == 0 && pub, xl + 1, fma(exr1, cp.pw[K - 1], u1[0]), tag);
        uint4 lv = ld_line_if(need && !dead, src);
        bool ok = !need || dead || (lv.y == tag && lv.w == tag);
        if (!__all_sync(FULL, ok)) {
            const long long t0 = clock64();
            for (unsigned it = 1; !__all_sync(FULL, ok); ++it) {
                if (!ok) {
                    lv = ld_line_gen(src);
                    ok = lv.y == tag && lv.w == tag;
                    if (!ok && (it & 63u) == 0u && (clock64() - t0 > cp.spin_limit || *(volatile unsigned*)cp.abort)) {
                        atomicExch(cp.abort, 1u);
                        dead = true;
                        ok = true;
                    }
                }
            }
        }
        // acquire, then a warp barrier (memory ordering among the warp's lanes): the
        // lane that saw a neighbour's line need not be the lane that reads that
        // neighbour's ring cell at the next fold (start-up and trailing ticks
        // exchange one level's lines only), nor the lane whose ring store must
        // follow the neighbour's fold
        __threadfence_block();
        __syncwarp();
        const double lvv = need && !dead ? line_value(lv) : 0.0;
        // ---- every correction at once (ridc_febe_carry.cuh): one rank-2 update per level
        if (A0) {
            const double fw = cf0 * cp.inv1ml2;
            const double fc = fma(__shfl_sync(FULL, lvv, 0) * ml, cp.inv1ml2, fw);
            const double bc = fma(-fw, zk, exr0 + fma(ye0, zc, __shfl_sync(FULL, lvv, 30)) * mr);
#pragma unroll
            for (int e = 0; e < K; ++e) u0[e] = fma(bc, cp.pw[K - 1 - e], fma(fc, cp.pw[e], u0[e]));
        }
        if (A1) {
            const double fw = cf1 * cp.inv1ml2;
            const double fc = fma(__shfl_sync(FULL, lvv, 1) * ml, cp.inv1ml2, fw);
            const double bc = fma(-fw, zk, exr1 + fma(ye1, zc, __shfl_sync(FULL, lvv, 31)) * mr);
#pragma unroll
            for (int e = 0; e < K; ++e) u1[e] = fma(bc, cp.pw[K - 1 - e], fma(fc, cp.pw[e], u1[e]));
        }
        // ---- finite checks (engine.py:160-164), uniform test first
        {
            const bool bad0 = A0 && !chunk_finite(u0), bad1 = A1 && !chunk_finite(u1);
            if (__any_sync(FULL, bad0 || bad1)) {
                if (bad0) atomicMin(cp.err, err_code(kk, 0));
                if (bad1) atomicMin(cp.err, err_code(kk - 2, 1));
            }
        }
        if (A0) {
            // the predictor's new step into the ring (step kk over step kk-3), then
            // release it before the next tick's lines
            double* Pw = ring + so * K * NP + tid + 1;
#pragma unroll
            for (int e = 0; e < K; ++e) Pw[e * NP] = u0[e];
            __threadfence_block();
            // my CTA's end points of predictor step kk (the neighbour CTAs' stencils)
            uint4* eb = cp.edge + (size_t)(kk & 3) * 2 * ncta;
            st_line_if(tid == 0 && !dead, eb + 2 * k, u0[0], tag);
            st_line_if(tid == ntk - 1 && !dead, eb + 2 * k + 1, u0[K - 1], tag);
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
#pragma unroll
    for (int e = 0; e < K; e += 2) {
        *reinterpret_cast<double2*>(cp.fin0 + c0 + e) = make_double2(u0[e], u0[e + 1]);
        *reinterpret_cast<double2*>(cp.fin1 + c0 + e) = make_double2(u1[e], u1[e + 1]);
    }
}

}  // namespace ridc
