// ridc_sweep.cuh -- streaming FEBE step for long periodic lines (RIDC order 1,
// reaction-diffusion, lines too long to stay resident on the SMs).
//
// One launch per time step (engine.py:167-175 _predict_core over the whole
// line).  CTA c owns the contiguous range [R_c, R_{c+1}) of the line (~N/148
// points) and sweeps it in chunks of 8192 points, one TMA-staged chunk after
// the other, so every point is read once and written once (16 B/pt, the
// algorithmic minimum of SURVEY.md §8d): no truncation halos inside a range.
//
// The shifted solve (I - dt L_S) x = rhs factors into  y_i = g rhs_i + lam y_{i-1}
// (forward) and  x_i = y_i + lam x_{i+1}  (backward), ridc_device.cuh.  Along
// the sweep:
//   * the forward carry of chunk i is y at chunk i-1's last point: it enters
//     chunk i's block scan as its initial value (exact);
//   * chunk i's backward pass runs with a zero carry at its end; the true
//     carry, x at chunk i+1's first point, is known one iteration later (chunk
//     i+1's own block-local backward value there -- its carry from chunk i+2
//     arrives as lam^8192 ~ 1e-340) and corrects only chunk i's last hc points
//     (x_p += d lam^(L-p), hc = truncation reach, lam^hc <= 2^-60): the warps
//     holding them keep their chunk in registers one iteration longer, every
//     other warp stores at once;
//   * the range ends are closed by one warp each: the forward carry into R_c
//     from a truncated forward pass over the 512 points before it, the
//     backward carry at R_{c+1} from a truncated forward + backward pass over
//     the 512 points after it (hc <= 512 -- r <~ 140 -- else the tick kernel runs).
// Chunks stream through NSTAGE TMA stages released as soon as their values are
// in registers (two chunks of prefetch); results leave with 256-bit stores.
// The states agree with the tick kernel to rounding (different association),
// and with the oracle at <= 1e-10 (tests/test_gpu_fullsize.py C5 sizes).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "ridc_chunk.cuh"
#include "ridc_device.cuh"
#include "ridc_tma.cuh"

namespace ridc {

constexpr int kSweepStages = 3;
constexpr int kSweepPend = 34;   // tail threads of a chunk: hc / 16 + 1 <= 33 (hc <= 512)
// NT = 512: one CTA per SM, 8192-point chunks.  (A 256-thread variant with two
// CTAs per SM and 4096-point chunks measured the same speed and gave
// run-to-run differences at C5 2^23 that a one-CTA-per-SM launch of the same
// code did not: not used.)
template <int NT>
constexpr size_t sweep_smem() { return (size_t)kSweepStages * NT * 16 * sizeof(double) + 2 * kSweepStages * 8 + 1024; }

struct SweepParams {
    DevProblem pb;
    double lam;
    double aa, bb;             // RD rhs with g folded in: (aa + bb u) u
    double g;                  // the solve's scale (the level sweep folds it into every node)
    double pw[16];             // lam^(e+1)
    double zf[16];             // forward-carry response of a chunk's backward pass
    double mp[10];             // M^(2^i), M = lam^16
    double* ring;              // level-0 ring (padded layout: data column c at GW + c)
    long long cap, Vs;
    int GW, gpr, gdata;        // ChunkLayout (tensor-map group coordinates)
    int nx;
    int hc;                    // carry reach (<= 512)
    long long per;             // error-step numbering
    unsigned long long* err;
};

__device__ __forceinline__ void stg256(double* p, double a, double b, double c, double d)
{
    asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d) : "memory");
}

// RD rhs with g folded in, one point
__device__ __forceinline__ double sweep_rhs(const SweepParams& sp, double u) { return fma(sp.bb, u, sp.aa) * u; }

// Warp-level scans of the chunk carries (multiplier M = lam^16 per lane):
// inclusive forward (lane l accumulates lanes <= l) and backward (lanes >= l).
template <class PP>   // any parameter block with mp[i] = M^(2^i)
__device__ __forceinline__ double warp_fwd_incl(const PP& sp, double v, int lane)
{
#pragma unroll
    for (int i = 0; i < 5; ++i) {
        const double t = __shfl_up_sync(0xffffffffu, v, 1 << i);
        if (lane >= (1 << i)) v = fma(sp.mp[i], t, v);
    }
    return v;
}

template <class PP>
__device__ __forceinline__ double warp_bwd_incl(const PP& sp, double v, int lane)
{
#pragma unroll
    for (int i = 0; i < 5; ++i) {
        const double t = __shfl_down_sync(0xffffffffu, v, 1 << i);
        if (lane + (1 << i) < 32) v = fma(sp.mp[i], t, v);
    }
    return v;
}

// 16 points of column c0 + 16 lane .. (wrapped periodically), straight from global memory
__device__ __forceinline__ void load16_wrap(const double* row, int c0, int nx, double (&u)[16])
{
#pragma unroll
    for (int e = 0; e < 16; ++e) {
        int c = c0 + e;
        c = c < 0 ? c + nx : (c >= nx ? c - nx : c);
        u[e] = __ldcg(row + c);
    }
}

template <int KIND, int NT>
__global__ void __launch_bounds__(NT, 512 / NT)
    k_sweep_febe(const __grid_constant__ SweepParams sp, const __grid_constant__ TmapSet tm, long long off,
                 long long target)
{
    static_assert(KIND == RD_1D, "streaming FEBE sweep: periodic reaction-diffusion lines");
    constexpr int K = 16, C = NT * K, NW = NT / 32, NS = kSweepStages;
    using L = ChunkSmem<NT, 1, NS, 16>;
    extern __shared__ __align__(1024) char smraw[];
    char* stage = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(stage + (size_t)NS * L::STAGE);
    uint64_t* empty = full + NS;
    __shared__ double sx[2 * NW];
    __shared__ unsigned s_cnt[NS];   // warps done with each stage (refill when all are)
    __shared__ double s_bc[2];   // broadcasts: [0] forward carry into the next chunk, [1] x at its first point
    // tail threads park their chunk here one iteration (transposed: [e][slot], conflict-free)
    __shared__ double s_pend[16 * kSweepPend];
    // the 512 points after my range (the epilogue's truncated passes), prefetched by warp 0
    __shared__ double s_next[512];
    const unsigned FULL = 0xffffffffu;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int G = gridDim.x, cta = blockIdx.x;
    const int nx = sp.nx;
    const long long n16 = nx / 16;
    const int R0 = 16 * (int)((long long)cta * n16 / G), R1 = 16 * (int)((long long)(cta + 1) * n16 / G);
    const int Lr = R1 - R0;
    const int nch = (Lr + C - 1) / C;
    // nch nearly equal chunks (multiples of 16 points): none shorter than the carry reach
    const int Cr = 16 * ((Lr + 16 * nch - 1) / (16 * nch));
    const long long src = (off + target - 1) % sp.cap, dst = (off + target) % sp.cap;
    RIDC_CHECK(src != dst && Lr >= 1024 && Cr % 16 == 0 && Cr <= C && (nch - 1) * Cr < Lr && sp.hc <= 512);
    const double* usrc = sp.ring + src * sp.Vs + sp.GW;   // data column 0
    double* udst = sp.ring + dst * sp.Vs + sp.GW;
    const double lam = sp.lam;

    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (tid == 0) {
        for (int i = 0; i < NS; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], NW);
            s_cnt[i] = 0u;
        }
        mbar_fence_init();
    }
    // M^lane, M^(31-lane), M^tid (forward carry-in weight of my chunk)
    double ml = 1.0, mr = 1.0, mt = 1.0;
#pragma unroll
    for (int i = 0; i < 10; ++i) {
        if (i < 5 && (lane & (1 << i))) ml *= sp.mp[i];
        if (i < 5 && ((31 - lane) & (1 << i))) mr *= sp.mp[i];
        if (tid & (1 << i)) mt *= sp.mp[i];
    }
    __syncthreads();
    auto issue = [&](int i) {   // one lane: chunk i of my range into stage i % NS
        const int s = i % NS;
        constexpr int NBOX = NT / L::BR;
        mbar_arrive_expect_tx(&full[s], (uint32_t)(NBOX * L::BR * 128));
        const int g0 = sp.gdata + (R0 + i * Cr) / 16;
        for (int b = 0; b < NBOX; ++b)
            tma_load_3d(stage + (size_t)s * L::STAGE + b * L::BR * 128, &tm.map[0], 0, g0 + b * L::BR, (int)src,
                        &full[s]);
    };
    // every read of the previous step's state waits for the previous launch
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (tid == 0)
        for (int i = 0; i < NS && i < nch; ++i) issue(i);

    // ---- range start: forward carry into R0 (warp 0, truncated over the 512 points before it)
    if (warp == 0) {
        double u[K];
        load16_wrap(usrc, R0 - 512 + 16 * lane, nx, u);
        double y = 0.0;
#pragma unroll
        for (int e = 0; e < K; ++e) y = fma(lam, y, sweep_rhs(sp, u[e]));
        y = warp_fwd_incl(sp, y, lane);
        if (lane == 31) s_bc[0] = y;
        // and the 512 points after my range, for the range-end pass
        load16_wrap(usrc, R1 + 16 * lane, nx, u);
#pragma unroll
        for (int e = 0; e < K; ++e) s_next[16 * lane + e] = u[e];
    }
    __syncthreads();
    double cin = s_bc[0];   // forward carry into the current chunk (all threads)

    // tail threads (last hc points of a chunk) keep their chunk's block-local x one
    // iteration longer, until the next chunk's first x (the backward carry) is known
    bool bad = false;
    int pend_col = -1;      // data column of my parked chunk, -1: nothing pending
    int pend_slot = 0;      // its s_pend slot
    double pend_m = 0.0;    // M^q, q = chunks after mine in that chunk (times pw[15-e]: lam^(end - point))
    auto pend_flush = [&](double d) {   // apply the backward carry d, check, store
        const double dm = d * pend_m;
        double w[K];
#pragma unroll
        for (int e = 0; e < K; ++e) w[e] = fma(dm, sp.pw[K - 1 - e], s_pend[e * kSweepPend + pend_slot]);
        bad |= !chunk_finite(w);
#pragma unroll
        for (int e = 0; e < K; e += 4) stg256(udst + pend_col + e, w[e], w[e + 1], w[e + 2], w[e + 3]);
        pend_col = -1;
    };

    for (int i = 0; i < nch; ++i) {
        const int s = i % NS;
        const int cbase = R0 + i * Cr;                // data column of the chunk's first point
        const int len = min(Cr, R1 - cbase);          // points of this chunk (multiple of 16)
        const int nthr = len / K;
        const bool mine = tid < nthr;
        // ---- my 16 points from the stage (swizzled), then release the stage
        mbar_wait(&full[s], (uint32_t)((i / NS) & 1));
        const char* st = stage + (size_t)s * L::STAGE;
        double v[K];
#pragma unroll
        for (int q = 0; q < K / 2; ++q) {
            const double2 w = lds128(swz(st, tid, q));
            v[2 * q] = w.x;
            v[2 * q + 1] = w.y;
        }
        // ---- forward: rhs, local recurrence (this consumes every loaded value:
        // the stage is released only after the shared loads have returned --
        // mbarrier.arrive does not wait for a warp's outstanding LDS), then
        // the block scan with the chunk's carry-in
        double y = 0.0;
#pragma unroll
        for (int e = 0; e < K; ++e) {
            y = fma(lam, y, sweep_rhs(sp, v[e]));
            v[e] = y;
        }
        __syncwarp();
        if (lane == 0) {   // the last warp done with the stage refills it (no warp blocks on the slowest)
            __threadfence_block();
            if (atomicAdd(&s_cnt[s], 1u) == (unsigned)(NW - 1)) {
                s_cnt[s] = 0u;
                __threadfence_block();
                if (i + NS < nch) issue(i + NS);
            }
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
        const double cf = fma(mt, cin, fma(ml, cw, ex));   // carry into my chunk, range carry included
        const double yend = fma(cf, sp.pw[K - 1], bf);     // y at my last point
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
        if (tid == nthr - 1) s_bc[0] = yend;               // forward carry into the next chunk
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
        const double dprev = s_bc[1];
        if (pend_col >= 0) pend_flush(dprev);
        // ---- store my points, or keep them pending when the next carry reaches them
        if (mine) {
            const int col = cbase + tid * K;
            if (K * (tid + 1) > len - sp.hc) {
                pend_slot = tid - max(0, (len - sp.hc) / K);
                RIDC_CHECK(pend_slot >= 0 && pend_slot < kSweepPend && col >= R0 && col + K <= R1);
#pragma unroll
                for (int e = 0; e < K; ++e) s_pend[e * kSweepPend + pend_slot] = v[e];
                pend_col = col;
                pend_m = 1.0;   // M^(nthr - 1 - tid)
                const int q = nthr - 1 - tid;
#pragma unroll
                for (int b = 0; b < 10; ++b)
                    if (q & (1 << b)) pend_m *= sp.mp[b];
            } else {
                bad |= !chunk_finite(v);
#pragma unroll
                for (int e = 0; e < K; e += 4) stg256(udst + col + e, v[e], v[e + 1], v[e + 2], v[e + 3]);
            }
        }
    }
    __syncthreads();   // every warp has read the last iteration's broadcasts before s_bc is reused
    // ---- range end: the backward carry at R1 (warp 0: the 512 points after it,
    // forward from this range's last y, then backward from zero), for the
    // pending tail of the last chunk
    if (warp == 0) {
        double u[K];
#pragma unroll
        for (int e = 0; e < K; ++e) u[e] = s_next[16 * lane + e];
        double y = 0.0;
#pragma unroll
        for (int e = 0; e < K; ++e) {
            y = fma(lam, y, sweep_rhs(sp, u[e]));
            u[e] = y;
        }
        // carry into my 16 points: previous lanes' totals + the range's carry cin
        double inc = warp_fwd_incl(sp, y, lane);
        double ex = __shfl_up_sync(FULL, inc, 1);
        if (lane == 0) ex = 0.0;
        const double cf = fma(ml, cin, ex);   // M^lane cin + sum of the lower lanes
        double x = 0.0;
#pragma unroll
        for (int e = K - 1; e >= 0; --e) {
            x = fma(lam, x, fma(cf, sp.pw[e], u[e]));
        }
        // x at my first point; the lanes above me contribute lam^(16 (l' - l)) ...
        double xb = warp_bwd_incl(sp, x, lane);   // lane 0: x at R1 (truncated at 512 points)
        if (lane == 0) s_bc[1] = xb;
    }
    __syncthreads();
    if (pend_col >= 0) pend_flush(s_bc[1]);
    if (bad) atomicMin(sp.err, err_code((target - 1) % sp.per + 1, 0));
}

}  // namespace ridc
