// ridc_tma.cuh -- TMA-bulk-copy pipelined level-step tick kernel (sm_100a).
//
// One persistent CTA per SM processes the work items of a tick (item = one
// level-step of one tile).  Warp NW (the producer) streams every node
// segment an item needs -- the level's own state and the (j+1) window
// states of level j-1, plus the rows above/below in 2-D -- from HBM/L2 into
// a ring of shared-memory stages with cp.async.bulk (the TMA engine),
// signalling per-stage mbarriers with the transaction byte count.  The NT
// consumer threads wait on a stage, fold it into their pointwise
// accumulators, release it, and after the last node apply the x-stencils,
// run the two first-order recurrences of the factored (I - dt L_S) with
// block-wide affine scans, and store the tile.  The producer runs ahead
// across nodes AND items, so load latency overlaps the previous item's
// scan; consumers never issue a global load on the fast path.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "ridc_device.cuh"

namespace ridc {

// ---------------------------------------------------------------- PTX helpers

__device__ __forceinline__ uint32_t smem_u32(const void* p)
{
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_fence_init()
{
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity)
{
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@P1 bra DONE_%=;\n\t"
        "bra WAIT_%=;\n"
        "DONE_%=:\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// As mbar_wait, but gives up when *abortp becomes non-zero (persistent kernel watchdog).
__device__ __forceinline__ void mbar_wait_or(uint64_t* bar, uint32_t parity, const volatile int* abortp)
{
    for (;;) {
        uint32_t ok;
        asm volatile(
            "{\n\t.reg .pred P1;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, P1;\n\t}"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
        if (ok || (abortp && *abortp)) return;
    }
}

// global -> shared bulk copy (UBLKCP), completion counted on `bar`
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

template <int N>
__device__ __forceinline__ void consumer_sync()
{
    asm volatile("bar.sync 1, %0;" ::"r"(N) : "memory");
}

// ---------------------------------------------------------------- staging plan

// Stage row layout: position q of the item's range [0, Q) lives at
// stage[kLead + sigma + q]; sigma in {0,1} aligns the largest contiguous
// source run to 16 bytes.  Aligned runs are copied by the TMA engine; the
// few positions it cannot cover (unaligned run ends, wrapped single columns,
// Dirichlet ghosts) are "fills" written by the consumers.  Plans depend only
// on (segment, parity of the row's element offset) and are precomputed on
// the host (build_plans in ridc_engine.cu) into a small device table.
constexpr int kLead = 2;
constexpr int kMaxBulk = 3;
constexpr int kMaxFill = 8;

struct PlanRow {
    int sigma;
    int nb;                      // bulk copies
    int bq0[kMaxBulk];           // first position
    int bcol[kMaxBulk];          // first source column (may be -1 / nx when widened)
    int bn[kMaxBulk];            // elements (even)
    int bytes;                   // total bulk bytes
    int nf;                      // fill ranges
    int fq0[kMaxFill], fn[kMaxFill];
};

// ---------------------------------------------------------------- the kernel

template <int NT, int KMAX, int ROWS, int NSTAGE>
struct TmaSmem {
    static constexpr int NW = NT / 32;
    static constexpr int CAP = NT * KMAX;
    static constexpr int SROW = CAP + 2 * kLead + 4;            // doubles per staged row
    static constexpr int STAGE = ROWS * SROW;
    static constexpr int SBUF = CAP + CAP / 16 + 1;
    static constexpr size_t OFF_SBUF = (size_t)NSTAGE * STAGE;  // in doubles
    static constexpr size_t OFF_BAR = OFF_SBUF + SBUF + 1;      // in doubles (8-byte slots)
    static constexpr size_t BYTES = (OFF_BAR + 2 * NSTAGE) * sizeof(double);
};

}  // namespace ridc

namespace ridc {

// Issue the bulk copies of one (item, node) segment into stage `st`.
template <int ROWS, int SROW>
__device__ __forceinline__ void issue_node(const DevProblem& pb, const DevSolve& sv, const double* vec,
                                           const Geo& geo, double* st, uint64_t* full)
{
    const int nx = pb.nx, ny = pb.ny;
    const int row = geo.row;
    const int rr[3] = {row, row == 0 ? ny - 1 : row - 1, row == ny - 1 ? 0 : row + 1};
    uint32_t bytes = 0;
    const PlanRow* plan[3];
#pragma unroll
    for (int r = 0; r < ROWS; ++r) {
        plan[r] = sv.plans + 2 * geo.seg + (int)(((long long)rr[r] * nx) & 1);
        bytes += (uint32_t)plan[r]->bytes;
    }
    mbar_arrive_expect_tx(full, bytes);
#pragma unroll
    for (int r = 0; r < ROWS; ++r) {
        const PlanRow* pl = plan[r];
        const double* rp = vec + (long long)rr[r] * nx;
        double* dst = st + r * SROW + kLead + pl->sigma;
        for (int b = 0; b < pl->nb; ++b)
            bulk_g2s(dst + pl->bq0[b], rp + pl->bcol[b], (uint32_t)pl->bn[b] * 8u, full);
    }
}

// Thread 0's cursor over this CTA's global load sequence: items
// i = blockIdx.x + m*gridDim.x, nodes 0..nnodes-1 each.  Load n lands in
// stage n % NSTAGE.
struct LoadCursor {
    int i, a;
    long long n;
};

// Consumer side of one TMA-staged item.  `n` counts this CTA's loads;
// thread 0 also refills each released stage with load n + NSTAGE.
template <int KIND, int NT, int KMAX, int ROWS, int NSTAGE, bool FAST, class Issue, class Ensure>
__device__ __forceinline__ void consume_item(const DevProblem& pb, const DevSolve& sv,
                                             const StepItem& it, const Geo& geo, double* stage,
                                             uint64_t* full, uint64_t* empty, long long& n,
                                             Issue&& refill, Ensure&& ensure, double* sbuf,
                                             Aff* swarp, unsigned long long* err,
                                             const volatile int* abortp = nullptr)
{
    using L = TmaSmem<NT, KMAX, ROWS, NSTAGE>;
    constexpr bool periodic = KIND != BURGERS_1D;
    constexpr bool two_d = ROWS == 3;
    const int nx = pb.nx, ny = pb.ny;
    const int tid = threadIdx.x, lane = tid & 31;
    const int cf = geo.s0 - 1;
    const int Q = geo.S + 2;
    const int row = geo.row;
    const int rown = row == 0 ? ny - 1 : row - 1, rows = row == ny - 1 ? 0 : row + 1;
    const long long roff[3] = {(long long)row * nx, (long long)rown * nx, (long long)rows * nx};
    const PlanRow* plan[3];
#pragma unroll
    for (int r = 0; r < ROWS; ++r) plan[r] = sv.plans + 2 * geo.seg + (int)(roff[r] & 1);

    double P[KMAX], WS[KMAX], WX[KMAX];
#pragma unroll
    for (int k = 0; k < KMAX; ++k) { P[k] = 0.0; WS[k] = 0.0; WX[k] = 0.0; }

    RIDC_STAMP(sv, geo.item_no, 0);
    for (int a = 0; a < it.nnodes; ++a, ++n) {
        const int s = (int)(n % NSTAGE);
        double* st = stage + (size_t)s * L::STAGE;
        if (tid == 0) ensure(n);   // persistent kernel: load n may still be unissued
        if (abortp) mbar_wait_or(&full[s], (uint32_t)((n / NSTAGE) & 1), abortp);
        else mbar_wait(&full[s], (uint32_t)((n / NSTAGE) & 1));
        if (a == 0) RIDC_STAMP(sv, geo.item_no, 1);
        if (!FAST) {
            bool filled = false;
#pragma unroll
            for (int r = 0; r < ROWS; ++r) {
                const PlanRow* pl = plan[r];
                const int nf = pl->nf;
                if (nf == 0) continue;
                filled = true;
                const double* rp = it.vec[a] + roff[r];
                double* dst = st + r * L::SROW + kLead + pl->sigma;
                for (int f = 0; f < nf; ++f) {
                    const int q0 = pl->fq0[f], cnt = pl->fn[f];
                    for (int q = q0 + tid; q < q0 + cnt; q += NT) dst[q] = at(rp, cf + q, nx, periodic);
                }
            }
            if (filled) csync<NT>();
        }
        const double ca = it.ca[a], cs = it.cs[a], cn = it.cn[a];
        const double* s0p = st + kLead + plan[0]->sigma;
        const double* s1p = two_d ? st + L::SROW + kLead + plan[ROWS > 1 ? 1 : 0]->sigma : s0p;
        const double* s2p = two_d ? st + 2 * L::SROW + kLead + plan[ROWS > 2 ? 2 : 0]->sigma : s0p;
#pragma unroll
        for (int k = 0; k < KMAX; ++k) {
            const int q = tid + k * NT;
            if (FAST || q < Q) {   // FAST: stale positions beyond Q are discarded later
                const double v = s0p[q];
                const double vn = two_d ? s1p[q] : 0.0;
                const double vs = two_d ? s2p[q] : 0.0;
                accumulate_point<KIND>(pb, ca, cs, cn, v, vn, vs, P[k], WS[k], WX[k]);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        if (tid == 0) refill(n, s);
    }
    finish_item<KIND, NT, KMAX, FAST>(pb, sv, it, geo, P, WS, WX, sbuf, swarp, err);
}

}  // namespace ridc
