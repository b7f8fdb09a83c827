// ridc_febe_carry.cuh -- resident FEBE march with carry exchange (periodic
// reaction-diffusion lines, levels == 1).
//
// The predictor level (engine.py:167-175 _predict_core: rhs = eta + dt f^N(eta),
// then the shifted solve (I - dt L_S) x = rhs, problems.py:119-124) on a line
// split into one tile per SM.  Every tile solves its own points only; the
// neighbours enter through two numbers per step instead of a truncation halo:
//
//   (I - dt L_S) = (r/lam)(1 - lam E^-1)(1 - lam E)  (periodic; ridc_device.cuh)
//   forward   y_i = g rhs_i + lam y_{i-1}
//   backward  x_i = y_i + lam x_{i+1}
//
// A tile solves both recurrences with zero carries at its ends (the block scan
// of fast_solve, no halo).  The exact periodic solution differs from that
// local one only through
//   * the forward carry c = y at the left neighbour's last point:
//       x_i += c lam^(i+1) / (1 - lam^2)            (head: i < hc)
//   * the backward carry d = x at the right neighbour's first point:
//       x_i += d lam^(T-i)                          (tail: i >= T - hc)
// where hc is the truncation reach (lam^hc <= 2^-60, ridc_engine.cu halo_of)
// and every dropped term is below lam^T ~ 1e-290 (tiles are >= 2 hc long).
// c is the neighbour's LOCAL forward value (its own left carry contributes
// lam^T), and d is the right neighbour's local first x plus the head
// correction by MY OWN y_end -- which I can add myself.  So each step needs
// two messages per tile edge that depend on nothing but the sender's own
// step, both 16-byte tagged lines in the LL format of the halo mailbox
// (ridc_resident.cuh):
//   1. after the forward scan a tile publishes y_end (its last point's y);
//   2. after the backward scan it publishes its first point's local x.
// The head warp waits for the left neighbour's y_end, the tail warp for the
// right neighbour's local x (one L2 round trip each, in parallel); every
// other warp runs straight into the next step (their only coupling is the
// block scans' two barriers).
//
// Against the truncated-halo march this computes 12% fewer points at C2, moves
// 2 values per edge per step through L2 instead of ~440 tagged lines, and
// drops the redundant halo recurrences.  The states agree with the Thomas +
// Sherman-Morrison oracle to rounding (tests/test_gpu_resident.py); they are
// not bitwise those of the tick kernel (different association).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "ridc_device.cuh"
#include "ridc_resident.cuh"

namespace ridc {

constexpr int kCarryMaxNT = 512;   // 16 warps x 16 points: tiles up to 8192 points

struct CarryParams {
    DevProblem pb;
    double lam;                // decay factor of the shifted operator's factors
    double aa, bb;             // RD rhs with g folded in: g (u + dt rho u (1 - u)) = (aa + bb u) u
    double inv1ml2;            // 1 / (1 - lam^2)
    double pw[32];             // lam^(e+1) (16 entries; 32 for the 32-point-per-lane warp march)
    double zf[32];             // forward-carry response of a K-point backward pass (DevSolve::zf16 for K = 16)
    double mp[10];             // M^(2^i), M = lam^K (K = 16; 32 for the 32-point warp march)
    double* ring;              // level-0 ring, padded layout (data column c at GW + c)
    long long cap, Vs;
    int GW;
    int T;                     // tile points (multiple of 16); tile k = [k T, min(k T + T, nx))
    int nx, nseg;
    int hc;                    // carry reach (points) at either tile end
    uint4* mail;               // [2 parities][nseg][2] tagged lines: 0 = y_end, 1 = x_begin
    unsigned tag0;             // run epoch: step s is tagged tag0 + s
    long long steps, per;      // FEBE restarts are plain continuation; per: error-step numbering
    int full_every;            // 1: store every step (trajectory recording, cap = steps + 1)
    unsigned long long* err;
    unsigned* abort;
    long long spin_limit;
    int exp;                   // diagnostics (RIDC_WC_EXP, k_febe_wcarry): 1 = no exchange (WRONG states), 2 = late first x
};

__device__ __forceinline__ void csync_n(int n)
{
    asm volatile("bar.sync 1, %0;" ::"r"(n) : "memory");
}

// Poll a tagged line (one lane) until it carries `want`; the watchdog sets
// *abort and returns 0 (the CTA then drains without waiting again).
__device__ __forceinline__ double poll_line(const uint4* p, unsigned want, const CarryParams& cp, bool& dead)
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

template <int KIND>
__global__ void __launch_bounds__(kCarryMaxNT, 1) k_febe_carry(const __grid_constant__ CarryParams cp)
{
    static_assert(KIND == RD_1D, "carry-exchange FEBE: periodic reaction-diffusion lines");
    constexpr int K = 16;
    __shared__ double sx[2 * (kCarryMaxNT / 32)];
    __shared__ double s_yend;   // y at my tile's last point (this step), for the tail warps
    const unsigned FULL = 0xffffffffu;
    const int NT = blockDim.x, NW = NT >> 5;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int k = blockIdx.x, nseg = cp.nseg;
    const int c0 = k * cp.T;
    const int Tk = min(cp.T, cp.nx - c0);
    const int nch = Tk / K;                     // chunks of my tile
    const bool mine = tid < nch;
    const int i0 = tid * K;                     // my first tile point
    const bool head = mine && i0 < cp.hc;
    const bool tail = mine && i0 + K > Tk - cp.hc;
    const bool head_warp = warp * 32 * K < cp.hc;
    const bool tail_warp = (warp * 32 + 31) * K + K > Tk - cp.hc && warp * 32 < nch;
    const bool last = tid == nch - 1;           // owns the tile's last point: publishes y_end
    RIDC_CHECK(nch <= (int)blockDim.x && Tk % K == 0 && Tk >= 2 * cp.hc && c0 + Tk <= cp.nx);
    const int kl = k == 0 ? nseg - 1 : k - 1, kr = k == nseg - 1 ? 0 : k + 1;
    RIDC_CHECK(k < nseg && kl >= 0 && kl < nseg && kr >= 0 && kr < nseg);
    const double lam = cp.lam;

    // carry powers: M^t (head, with 1/(1 - lam^2)), M^(nch-1-t) (tail), M^lane, M^(31-lane)
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
    // lane-masked scan multipliers: a lane outside a shuffle step's reach gets 0,
    // so every scan step is one unpredicated FMA (no selects)
    double mf[5], mb[5];
#pragma unroll
    for (int i = 0; i < 5; ++i) {
        mf[i] = lane >= (1 << i) ? cp.mp[i] : 0.0;
        mb[i] = lane + (1 << i) < 32 ? cp.mp[i] : 0.0;
    }
    double* const fin = cp.ring + cp.GW + c0 + i0;   // + slot * Vs
    long long slot = 0;                              // ring slot of step s (s % cap, kept incrementally)

    double u[K];
    if (mine) {
        load_chunk_cg(cp.ring + cp.GW + c0 + i0, u);   // slot 0: the seeded initial state
    } else {
#pragma unroll
        for (int e = 0; e < K; ++e) u[e] = 0.0;
    }
    bool dead = false;

    for (long long s = 1; s <= cp.steps; ++s) {
        const unsigned tag = cp.tag0 + (unsigned)s;
        uint4* box = cp.mail + (size_t)(s & 1) * 2 * nseg;
        // ---- rhs (g folded in) and the local forward recurrence (zero carry in)
        double y = 0.0;
#pragma unroll
        for (int e = 0; e < K; ++e) {
            const double r = fma(cp.bb, u[e], cp.aa) * u[e];
            y = fma(lam, y, r);
            u[e] = y;
        }
        const double bf = mine ? y : 0.0;
        // ---- forward carries (chunk multiplier M = lam^16, as fast_solve)
        double inc = bf;
#pragma unroll
        for (int i = 0; i < 5; ++i) inc = fma(mf[i], __shfl_up_sync(FULL, inc, 1 << i), inc);
        if (lane == 31) sx[warp] = inc;
        double ex = __shfl_up_sync(FULL, inc, 1);
        if (lane == 0) ex = 0.0;
        csync_n(NT);
        double wi = lane < NW ? sx[lane] : 0.0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {   // lanes < NW: warp totals (lanes >= NW carry zeros or ignored sums)
            const double t = __shfl_up_sync(FULL, wi, 1 << i);
            if (lane >= (1 << i)) wi = fma(cp.mp[5 + i], t, wi);
        }
        double cw = __shfl_sync(FULL, wi, warp > 0 ? warp - 1 : 0);
        if (warp == 0) cw = 0.0;
        const double cf = fma(ml, cw, ex);
        // 1. publish y at my tile's last point (the right neighbour's forward carry)
        if (last) {
            const double yend = fma(cf, cp.pw[K - 1], bf);
            if (!dead) st_line(box + 2 * k, yend, tag);
            s_yend = yend;   // read by the tail warps after the backward scan's barrier
        }
        // ---- local backward recurrence (zero carry at the tile end)
        double x = 0.0;
#pragma unroll
        for (int e = K - 1; e >= 0; --e) {
            x = fma(lam, x, u[e]);
            u[e] = x;
        }
        double rinc = mine ? fma(cf, cp.zf[0], x) : 0.0;
#pragma unroll
        for (int i = 0; i < 5; ++i) rinc = fma(mb[i], __shfl_down_sync(FULL, rinc, 1 << i), rinc);
        if (lane == 0) sx[NW + warp] = rinc;
        double exr = __shfl_down_sync(FULL, rinc, 1);
        if (lane == 31) exr = 0.0;
        csync_n(NT);
        double wr = lane < NW ? sx[NW + (NW - 1 - lane)] : 0.0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const double t = __shfl_up_sync(FULL, wr, 1 << i);
            if (lane >= (1 << i)) wr = fma(cp.mp[5 + i], t, wr);
        }
        const int rl = NW - 1 - warp;
        double dw = __shfl_sync(FULL, wr, rl > 0 ? rl - 1 : 0);
        if (rl == 0) dw = 0.0;
        const double dc = fma(mr, dw, exr);
#pragma unroll
        for (int e = 0; e < K; ++e) u[e] = fma(dc, cp.pw[K - 1 - e], fma(cf, cp.zf[e], u[e]));
        // 2. publish my first point's LOCAL x (before my head correction): the left
        // neighbour completes it with its own y_end, so neither carry waits on the other
        if (tid == 0 && !dead) st_line(box + 2 * k + 1, u[0], tag);
        // ---- head: the left neighbour's forward carry
        if (head_warp) {
            double c = 0.0;
            if (lane == 0) c = poll_line(box + 2 * kl, tag, cp, dead);
            c = __shfl_sync(FULL, c, 0);
            if (head) {
                const double cm = c * Mh;
#pragma unroll
                for (int e = 0; e < K; ++e) u[e] = fma(cm, cp.pw[e], u[e]);
            }
        }
        // ---- tail: the right neighbour's backward carry d = x at its first point =
        // its local x there + its head correction by MY y_end (the very operations
        // the neighbour applies to its own first point: bitwise the same d)
        if (tail_warp) {
            double d = 0.0;
            if (lane == 0) {
                const double xl = poll_line(box + 2 * kr + 1, tag, cp, dead);
                d = fma(s_yend * cp.inv1ml2, cp.pw[0], xl);
            }
            d = __shfl_sync(FULL, d, 0);
            if (tail) {
                const double dm = d * Mt;
#pragma unroll
                for (int e = 0; e < K; ++e) u[e] = fma(dm, cp.pw[K - 1 - e], u[e]);
            }
        }
        // ---- finite check (engine.py:160-164); the tile to the ring at the end
        if (!mine) {   // threads past the tile feed zeros into the next step's scans
#pragma unroll
            for (int e = 0; e < K; ++e) u[e] = 0.0;
        } else {
            if (!chunk_finite(u)) atomicMin(cp.err, err_code((s - 1) % cp.per + 1, 0));
            if (cp.full_every) {   // trajectory: every step to its slot (cap = steps + 1)
                slot = slot + 1 == cp.cap ? 0 : slot + 1;
                double* out = fin + slot * cp.Vs;
#pragma unroll
                for (int e = 0; e < K; e += 2) *reinterpret_cast<double2*>(out + e) = make_double2(u[e], u[e + 1]);
            }
        }
    }
    if (mine && !cp.full_every) {   // the final state to ring slot steps % cap
        double* out = fin + (cp.steps % cp.cap) * cp.Vs;
#pragma unroll
        for (int e = 0; e < K; e += 2) *reinterpret_cast<double2*>(out + e) = make_double2(u[e], u[e + 1]);
    }
}

// ---------------------------------------------------------------------------
// Warp-chunk variant (k_febe_wcarry): the same march with every WARP owning a
// 512-point chunk (16 points per lane) and the chunks coupled exactly as the
// tiles above, by two carries per step -- but between the warps of a CTA the
// carries travel through shared memory (the same tagged 16-byte lines), so a
// step has no block barrier and no block scan: each warp's only waits are its
// two neighbours' lines of the same step, one hop each (L2 only where the
// neighbour sits in another CTA).  Lines of 512-point chunks (C2: 2048 chunks,
// 14 warps on each of 147 SMs; K = 16 points per lane) or 1024-point chunks
// (2^21: K = 32); dropped terms below lam^(32 K) <= 2^-60 (hc <= 32 K).
// Both outgoing carries are computed from the step's right-hand side (dot
// products with the pw tables) and published before the recurrences, so the
// L2 hop overlaps the solve; every one-lane store / load is predicated and the
// neighbour wait is a warp vote ("Early carries").

// Predicated forms (no branch around a one-lane store / load: the warp's basic
// block stays whole, so the scheduler interleaves the recurrences with the
// scans' shuffles and no convergence check precedes the next shuffle)
__device__ __forceinline__ void st_line_if(bool pred, uint4* p, double v, unsigned tag)
{
    const unsigned long long b = (unsigned long long)__double_as_longlong(v);
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %5, 0;\n\t@q st.volatile.v4.u32 [%0], {%1, %2, %3, %4};\n\t}"
                 ::"l"(p), "r"((unsigned)b), "r"(tag), "r"((unsigned)(b >> 32)), "r"(tag), "r"((int)pred)
                 : "memory");
}

__device__ __forceinline__ uint4 ld_line_if(bool pred, const uint4* p)
{
    uint4 v = make_uint4(0u, 0u, 0u, 0u);
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %5, 0;\n\t@q ld.volatile.v4.u32 {%0, %1, %2, %3}, [%4];\n\t}"
                 : "+r"(v.x), "+r"(v.y), "+r"(v.z), "+r"(v.w)
                 : "l"(p), "r"((int)pred)
                 : "memory");
    return v;
}

__device__ __forceinline__ uint4 ld_line_gen(const uint4* p)
{
    uint4 v;
    asm volatile("ld.volatile.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p) : "memory");
    return v;
}

constexpr int kWCarryMaxWarps = 14;   // 448 threads: C2's 2048 chunks on 147 SMs

// K points per lane: 16 (512-point chunks) or 32 (1024-point chunks: lines of
// up to 14 x 148 x 1024 points, carry reach <= 1024); cp.pw / zf / mp hold the
// K-point tables
template <int KIND, int K>
__global__ void __launch_bounds__(kWCarryMaxWarps * 32, 1) k_febe_wcarry(const __grid_constant__ CarryParams cp)
{
    static_assert(KIND == RD_1D, "carry-exchange FEBE: periodic reaction-diffusion lines");
    static_assert(K == 16 || K == 32, "16 or 32 points per lane");
    constexpr int CH = 32 * K;   // points per chunk
    __shared__ uint4 s_line[2][kWCarryMaxWarps][2];   // [parity][warp]: 0 = y_end, 1 = local first x
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wpc = cp.T;                                  // warps (chunks) per CTA
    const int nch = cp.nseg;                               // chunks of the line
    const int chunk = blockIdx.x * wpc + warp;
    if (threadIdx.x < 2 * kWCarryMaxWarps * 2)             // no stale tag from an earlier kernel's shared memory
        reinterpret_cast<uint4*>(s_line)[threadIdx.x] = make_uint4(0u, 0u, 0u, 0u);
    __syncthreads();
    if (warp >= wpc || chunk >= nch) return;               // no block barrier follows
    const int cl = chunk == 0 ? nch - 1 : chunk - 1, cr = chunk == nch - 1 ? 0 : chunk + 1;
    const bool left_local = warp > 0;                      // chunk - 1 is this CTA's previous warp
    const bool right_local = warp + 1 < wpc && chunk + 1 < nch;
    const int c0 = chunk * CH + lane * K;                  // data column of my first point
    RIDC_CHECK(c0 + K <= cp.nx && cp.hc <= CH && wpc <= kWCarryMaxWarps);
    const double lam = cp.lam;

    double ml = 1.0, mr = 1.0;
#pragma unroll
    for (int i = 0; i < 5; ++i) {
        if (lane & (1 << i)) ml *= cp.mp[i];
        if ((31 - lane) & (1 << i)) mr *= cp.mp[i];
    }
    const double zc = lam * cp.inv1ml2, zk = lam * cp.pw[K - 1];   // lam^(K+1)
    // diagnostics (RIDC_WC_EXP): 1 = no exchange (WRONG states), 2 = the first x
    // published after the backward scan, no early loads
    const bool late = cp.exp & 2;
    const double ilam = 1.0 / lam;
    const double xw = ml * cp.inv1ml2 * ilam;   // first-x weight of my points: M^lane lam^e / (1 - lam^2)
    double mf[5], mb[5];   // lane-masked scan multipliers (no selects in the scans)
#pragma unroll
    for (int i = 0; i < 5; ++i) {
        mf[i] = lane >= (1 << i) ? cp.mp[i] : 0.0;
        mb[i] = lane + (1 << i) < 32 ? cp.mp[i] : 0.0;
    }
    double* const fin = cp.ring + cp.GW + c0;   // + slot * Vs
    long long slot = 0;
    double u[K];
#pragma unroll
    for (int e = 0; e < K; e += 2) {   // slot 0: the seeded initial state
        const double2 v = __ldcg(reinterpret_cast<const double2*>(fin + e));
        u[e] = v.x;
        u[e + 1] = v.y;
    }
    bool dead = false;
    auto finite = [&]() {   // chunk_finite over K points
        double c0 = 0.0, c1 = 0.0, c2 = 0.0, c3 = 0.0;
#pragma unroll
        for (int e = 0; e < K; e += 4) {
            c0 = fma(u[e], 0.0, c0);
            c1 = fma(u[e + 1], 0.0, c1);
            c2 = fma(u[e + 2], 0.0, c2);
            c3 = fma(u[e + 3], 0.0, c3);
        }
        const double c = (c0 + c1) + (c2 + c3);
        return c == c;
    };

    for (long long s = 1; s <= cp.steps; ++s) {
        const unsigned tag = cp.tag0 + (unsigned)s;
        const int par = (int)(s & 1);
        uint4* box = cp.mail + (size_t)par * 2 * nch;
        const bool pub = !dead && !(cp.exp & 1);
        // ---- rhs (g folded in)
#pragma unroll
        for (int e = 0; e < K; ++e) u[e] = fma(cp.bb, u[e], cp.aa) * u[e];
        // Per lane, dot products of the rhs with pw[e] and pw[K-1-e]:
        //   sb = lam * (y at my last point, zero carry in): the forward scan's input,
        //        so the scan (and y_end) does not wait for the recurrence;
        //   sa gives my chunk's local first x for the left neighbour,
        //        x_0 = sum_j lam^j (1 - lam^(2 (CH - j))) / (1 - lam^2) r_j over the
        //        chunk's points j = K lane + e, the lam^(2 CH - j) part below
        //        lam^CH <= 2^-60 (the march's truncation) dropped: one butterfly.
        // Both carries leave before any recurrence: the L2 hop overlaps my two
        // recurrences and scans instead of following them
        // (profiles/r2_wcarry_early.json: also the A/Bs not kept -- the scan fed
        // by the recurrence, a third dot product for the backward scan, K = 32).
        double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
#pragma unroll
        for (int e = 0; e < K; e += 2) {
            a0 = fma(u[e], cp.pw[e], a0);
            a1 = fma(u[e + 1], cp.pw[e + 1], a1);
            b0 = fma(u[e], cp.pw[K - 1 - e], b0);
            b1 = fma(u[e + 1], cp.pw[K - 2 - e], b1);
        }
        if (!late) {
            double cx = (a0 + a1) * xw;
#pragma unroll
            for (int i = 16; i >= 1; i >>= 1) cx += __shfl_xor_sync(FULL, cx, i);
            st_line_if(lane == 0 && pub, left_local ? &s_line[par][warp][1] : box + 2 * chunk + 1, cx, tag);
        }
        // ---- forward carries: the warp scan of the lanes' last y
        double inc = (b0 + b1) * ilam;
#pragma unroll
        for (int i = 0; i < 5; ++i) inc = fma(mf[i], __shfl_up_sync(FULL, inc, 1 << i), inc);
        double cf = __shfl_up_sync(FULL, inc, 1);
        if (lane == 0) cf = 0.0;
        const double yend = __shfl_sync(FULL, inc, 31);   // y at my chunk's last point (zero carry in)
        // 1. publish y_end for the right neighbour
        st_line_if(lane == 31 && pub, right_local ? &s_line[par][warp][0] : box + 2 * chunk, yend, tag);
        // ---- the local forward and backward recurrences (zero carries)
        double y = 0.0;
#pragma unroll
        for (int e = 0; e < K; ++e) {
            y = fma(lam, y, u[e]);
            u[e] = y;
        }
        double x = 0.0;
#pragma unroll
        for (int e = K - 1; e >= 0; --e) {
            x = fma(lam, x, u[e]);
            u[e] = x;
        }
        // the neighbours' lines, loaded now and checked after the backward scan
        // (published early, they are usually there: the load's L2 round trip
        // overlaps the scan)
        // lane 0 reads the left neighbour's y_end, lane 31 the right one's first x
        const bool need = (lane == 0 || lane == 31) && !(cp.exp & 1);
        const uint4* src = lane == 0 ? (left_local ? &s_line[par][warp - 1][0] : box + 2 * cl)
                                     : (right_local ? &s_line[par][warp + 1][1] : box + 2 * cr + 1);
        uint4 lv = ld_line_if(need && !late, src);
        double rinc = fma(cf, cp.zf[0], x);
#pragma unroll
        for (int i = 0; i < 5; ++i) rinc = fma(mb[i], __shfl_down_sync(FULL, rinc, 1 << i), rinc);
        double exr = __shfl_down_sync(FULL, rinc, 1);
        if (lane == 31) exr = 0.0;
        // lane 0: no forward carry inside the warp, only the backward one
        st_line_if(late && lane == 0 && pub, left_local ? &s_line[par][warp][1] : box + 2 * chunk + 1,
                   fma(exr, cp.pw[K - 1], u[0]), tag);
        if (late) lv = ld_line_if(need, src);
        // ---- the neighbours' carries: one vote over lanes 0 and 31; the rare
        // re-poll is a warp-uniform loop (both lanes wait together, one L2 round
        // trip per round, the watchdog every 64 rounds)
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
        const double lvv = need && !dead ? line_value(lv) : 0.0;
        const double cv = lane == 0 ? lvv : 0.0, dv = lane == 31 ? lvv : 0.0;
        // ---- every correction at once.  The warp's own carries move x_e by
        // cf zf[e] + exr pw[K-1-e] with zf[e] = (pw[e] - lam^(K+1) pw[K-1-e]) /
        // (1 - lam^2); the left neighbour's y_end by cv M^lane pw[e] / (1 - lam^2)
        // (head), the right neighbour's first x (+ the head correction my y_end
        // causes there) by tm pw[K-1-e] (tail): one rank-2 update in the basis
        // pw[e], pw[K-1-e]
        const double fw = cf * cp.inv1ml2;
        const double fc = fma(__shfl_sync(FULL, cv, 0) * ml, cp.inv1ml2, fw);
        const double tm = fma(yend, zc, __shfl_sync(FULL, dv, 31)) * mr;
        const double bc = fma(-fw, zk, exr + tm);
#pragma unroll
        for (int e = 0; e < K; ++e) u[e] = fma(bc, cp.pw[K - 1 - e], fma(fc, cp.pw[e], u[e]));
        {
            const bool bad = !finite();
            if (__any_sync(FULL, bad) && bad) atomicMin(cp.err, err_code((s - 1) % cp.per + 1, 0));   // uniform test first
        }
        if (cp.full_every) {   // trajectory: every step to its slot (cap = steps + 1)
            slot = slot + 1 == cp.cap ? 0 : slot + 1;
            double* out = fin + slot * cp.Vs;
#pragma unroll
            for (int e = 0; e < K; e += 2) *reinterpret_cast<double2*>(out + e) = make_double2(u[e], u[e + 1]);
        }
    }
    if (!cp.full_every) {   // the final state to ring slot steps % cap
        double* out = fin + (cp.steps % cp.cap) * cp.Vs;
#pragma unroll
        for (int e = 0; e < K; e += 2) *reinterpret_cast<double2*>(out + e) = make_double2(u[e], u[e + 1]);
    }
}

}  // namespace ridc
