// ridc_resident.cuh -- register-resident FEBE march (levels == 1, 1-D lines).
//
// The predictor level alone (RIDC order 1: forward/backward Euler IMEX,
// engine.py:167-175 _predict_core) needs, per step, only its own state.
// When the line's segments fit one CTA each on the GPU (N <= ~148 x 7000
// points: configs C1 and C2), a single cooperative launch marches every
// step with each thread's 16-point chunk kept in registers:
//
//   step s:  [halo threads reload their chunk from the ring slot of step s-1,
//             after the two neighbour segments published it]
//            accumulate -> x-stencils -> two recurrences (chunk_rhs_solve,
//            the very code of the tick kernel: bitwise the same states)
//            -> publish the columns a neighbour's halo can reach (+ periodic
//               ghosts) into ring slot s % cap, then a release flag.
//
// Only the truncation-halo edges (~2 x 470 of ~7100 columns) round-trip
// through L2 per step, instead of the whole state; the full tile is written
// once, after the last step (or every step when the trajectory is recorded).
// Neighbour skew is at most one step, so the two-slot ring is race-free:
// a segment writes slot s % 2 only after both neighbours finished step s-1,
// i.e. after they read slot (s-2) % 2 for the last time.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "ridc_chunk.cuh"
#include "ridc_device.cuh"

namespace ridc {

struct ResidentParams {
    DevProblem pb;
    DevSolve sv;
    ChunkLayout lay;
    const ChunkGeo* cgeo;
    double* ring;            // level-0 ring, cap slots of Vs doubles (padded layout)
    long long cap, Vs;
    double dt;
    long long steps;         // restarts * per (FEBE restarts are plain continuation)
    long long per;           // steps per restart interval (error-step numbering)
    int edge_w;              // columns within edge_w of a tile end are published every step
    int full_every;          // 1: publish whole tiles every step (trajectory recording)
    unsigned* flags;         // per segment: last published step (zeroed before the launch)
    unsigned long long* err; // earliest non-finite (step, level), atomicMin
    unsigned* abort;         // watchdog: set when a neighbour wait times out
    long long spin_limit;    // watchdog budget per wait (clock64 cycles)
    long long* dbg;          // optional phase trace (RIDC_PHASE_TIMING): CTA 0, thread 0, steps 1..8
};

// slots: steps 1..4 -> rows 0..3, steps S-3..S -> rows 4..7; col 6: globaltimer (ns) at row start
#define RIDC_RSTAMP(rp, s, idx)                                                              \
    do {                                                                                     \
        if ((rp).dbg && threadIdx.x == 0 && blockIdx.x == 0) {                               \
            const long long _r = (s) <= 4 ? (s) - 1 : ((s) > (rp).steps - 4 ? (s) - (rp).steps + 7 : -1); \
            if (_r >= 0) {                                                                   \
                (rp).dbg[_r * 16 + (idx)] = clock64();                                       \
                if ((idx) == 0) {                                                            \
                    unsigned long long _g;                                                   \
                    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_g));                  \
                    (rp).dbg[_r * 16 + 6] = (long long)_g;                                   \
                }                                                                            \
            }                                                                                \
        }                                                                                    \
    } while (0)

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p)
{
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v)
{
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// 16 consecutive doubles from L2 (bypassing L1: other SMs wrote them)
__device__ __forceinline__ void load_chunk_cg(const double* src, double (&u)[kChunk])
{
    const double2* s2 = reinterpret_cast<const double2*>(src);
#pragma unroll
    for (int i = 0; i < kChunk / 2; ++i) {
        const double2 v = __ldcg(s2 + i);
        u[2 * i] = v.x;
        u[2 * i + 1] = v.y;
    }
}

template <int KIND, int NT, int MODE>
__device__ __forceinline__ void resident_step(const ResidentParams& rp, const ChunkGeo& cg, bool mine,
                                              double (&u)[kChunk], double* edge, Aff* swarp, FastLane fl)
{
    constexpr int K = kChunk;
    constexpr bool has_wx = KIND == ADV_DIFF_1D || KIND == BURGERS_1D;
    double P[K], WS[K], WX[K];
#pragma unroll
    for (int e = 0; e < K; ++e) {
        P[e] = 0.0;
        WS[e] = 0.0;
        WX[e] = 0.0;
    }
    // the predictor's single node: ca = 1, cs = 0, cn = dt (build_item, level 0)
    if (mine) {
        const NodeCoef nc = node_coef<KIND>(rp.pb, 1.0, 0.0, rp.dt);
#pragma unroll
        for (int e = 0; e < K; ++e) accumulate_point<KIND>(nc, u[e], 0.0, 0.0, P[e], WS[e], WX[e]);
    }
    chunk_rhs_solve<KIND, NT, MODE>(rp.pb, rp.sv, cg, false, has_wx && rp.dt != 0.0, mine, P, WS, WX, u, edge,
                                    swarp, 99, fl);
}

// Finite check of 16 values: four independent FMA chains (x * 0 is NaN iff x is not finite).
__device__ __forceinline__ bool chunk_finite(const double (&u)[kChunk])
{
    double c0 = 0.0, c1 = 0.0, c2 = 0.0, c3 = 0.0;
#pragma unroll
    for (int e = 0; e < kChunk; e += 4) {
        c0 = fma(u[e], 0.0, c0);
        c1 = fma(u[e + 1], 0.0, c1);
        c2 = fma(u[e + 2], 0.0, c2);
        c3 = fma(u[e + 3], 0.0, c3);
    }
    const double c = (c0 + c1) + (c2 + c3);
    return c == c;
}

// MODE: the solve mode every segment shares (0 truncated, 1 cyclic whole
// line, 2 Dirichlet ends), or -1 to dispatch per segment.
template <int KIND, int NT, int MODE>
__global__ void __launch_bounds__(NT, 1) k_resident_febe(const __grid_constant__ ResidentParams rp)
{
    static_assert(KIND == ADV_DIFF_1D || KIND == BURGERS_1D || KIND == RD_1D, "1-D kinds only");
    constexpr int K = kChunk;
    constexpr bool periodic = KIND != BURGERS_1D;
    __shared__ double edge[4 * NT];
    __shared__ Aff swarp[2 * (NT / 32) + 1];
    __shared__ int s_stop;
    const int tid = threadIdx.x;
    const int seg = blockIdx.x, nseg = rp.sv.nseg;
    const ChunkGeo cg = rp.cgeo[seg];
    const bool mine = tid < cg.ng;
    const int col0 = (cg.g0 + tid) * K;   // data column of my first point
    const int lo = cg.c0, hi = cg.c0 + cg.tlen;
    const int nx = rp.pb.nx, GW = rp.lay.GW, W = rp.edge_w;
    // halo chunk: (partly) outside my tile -- reloaded every step from the
    // neighbour on that side (W < tile length: a halo reaches one neighbour)
    const bool halo = mine && nseg > 1 && (col0 < lo || col0 + K > hi);
    const int nb = !halo ? -1
                         : (col0 < lo ? (seg > 0 ? seg - 1 : (periodic ? nseg - 1 : -1))
                                      : (seg + 1 < nseg ? seg + 1 : (periodic ? 0 : -1)));
    // interior chunk: all 16 columns in my tile and >= W from both ends (no
    // neighbour reads them, no periodic ghost copies: W >= GW)
    const bool interior = mine && col0 - lo >= W && hi - (col0 + K) >= W;
    if (tid == 0) s_stop = 0;
    __syncthreads();

    double u[K];
#pragma unroll
    for (int e = 0; e < K; ++e) u[e] = 0.0;
    if (mine) load_chunk_cg(rp.ring + GW + col0, u);   // slot 0: the seeded initial state
    long long cur = 0;                                  // ring slot of step s-1
    const FastLane fl = fast_lane<K>(rp.sv);

    for (long long s = 1; s <= rp.steps; ++s) {
        const double* prev = rp.ring + cur * rp.Vs + GW;
        cur = cur + 1 == rp.cap ? 0 : cur + 1;
        double* out = rp.ring + cur * rp.Vs + GW;
        RIDC_RSTAMP(rp, s, 0);
        if (s > 1 && halo) {
            // acquire the neighbour's step s-1 publication, then reload my chunk
            if (nb >= 0) {
                const unsigned want = (unsigned)(s - 1);
                const long long t0 = clock64();
                while (ld_acquire_u32(rp.flags + nb) < want)
                    if (clock64() - t0 > rp.spin_limit || *(volatile unsigned*)rp.abort) {
                        atomicExch(rp.abort, 1u);
                        s_stop = 1;
                        break;
                    }
            }
            RIDC_RSTAMP(rp, s, 1);
            load_chunk_cg(prev + col0, u);
        }
        RIDC_RSTAMP(rp, s, 2);
        if (MODE >= 0) {
            resident_step<KIND, NT, (MODE >= 0 ? MODE : 0)>(rp, cg, mine, u, edge, swarp, fl);
        } else {
            switch (cg.mode) {
            case 0: resident_step<KIND, NT, 0>(rp, cg, mine, u, edge, swarp, fl); break;
            case 1: resident_step<KIND, NT, 1>(rp, cg, mine, u, edge, swarp, fl); break;
            default: resident_step<KIND, NT, 2>(rp, cg, mine, u, edge, swarp, fl);
            }
        }
        RIDC_RSTAMP(rp, s, 3);
        const bool full = s == rp.steps || rp.full_every;
        bool bad = false;
        if (interior) {
            bad = !chunk_finite(u);
            if (full) {
#pragma unroll
                for (int e = 0; e < K; e += 2)
                    *reinterpret_cast<double2*>(out + col0 + e) = make_double2(u[e], u[e + 1]);
            }
        } else if (mine) {
            // tile-edge chunk: per-column ownership, publication and periodic ghosts
            double chk = 0.0;
#pragma unroll
            for (int e = 0; e < K; ++e) {
                const int c = col0 + e;
                if (c >= lo && c < hi) {
                    chk = fma(u[e], 0.0, chk);
                    if (full || c - lo < W || hi - 1 - c < W) out[c] = u[e];
                    if (periodic && c < GW) out[c + nx] = u[e];
                    if (periodic && c >= nx - GW) out[c - nx] = u[e];
                }
            }
            bad = chk != chk;
        }
        if (bad) atomicMin(rp.err, err_code((s - 1) % rp.per + 1, 0));
        RIDC_RSTAMP(rp, s, 4);
        __syncthreads();   // publication complete (and shared scratch free for the next step)
        RIDC_RSTAMP(rp, s, 5);
        if (s_stop) return;
        if (nseg > 1 && tid == 0) st_release_u32(rp.flags + seg, (unsigned)s);
    }
}

}  // namespace ridc
