// ridc_dispatch.cuh -- definitions of the per-kind launch entry points declared
// in ridc_kernels.cuh (template instantiation happens in ridc_inst.cu only).
#pragma once
#include "ridc_kernels.cuh"
#include "ridc_sweep_warp.cuh"

namespace ridc {

template <int KIND, int NT, int KMAX>
cudaError_t launch_item_t(int items, size_t smem, cudaStream_t st, const DevProblem& pb,
                          const DevSolve& sv, const StepItem& it, unsigned long long* err)
{
    static bool attr[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
    if (!attr[dev]) {
        cudaError_t e = cudaFuncSetAttribute(k_item<KIND, NT, KMAX>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        attr[dev] = true;
    }
    k_item<KIND, NT, KMAX><<<items, NT, smem, st>>>(pb, sv, it, err);
    return cudaGetLastError();
}

#define RIDC_DISPATCH_CFG(FN, KIND, CFG, ...)                          \
    ((CFG).id == 0 ? FN<KIND, 128, 8>(__VA_ARGS__)                     \
     : (CFG).id == 1 ? FN<KIND, 256, 8>(__VA_ARGS__)                   \
                     : FN<KIND, 512, 8>(__VA_ARGS__))

template <int KIND>
cudaError_t launch_item_k(const LaunchCfg& c, int items, cudaStream_t st, const DevProblem& pb,
                          const DevSolve& sv, const StepItem& it, unsigned long long* err)
{
    return RIDC_DISPATCH_CFG(launch_item_t, KIND, c, items, c.smem, st, pb, sv, it, err);
}

template <int KIND, int NT, int ROWS, int NSTAGE, int MODE, int KC>
cudaError_t launch_chunk_t(int grid, size_t smem, cudaStream_t st, const EngineParams& ep,
                           const TickParams& tp, int ipl, const TmapSet& tm)
{
    auto kfn = k_tick_chunk<KIND, NT, ROWS, NSTAGE, MODE, KC>;
    static bool attr[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
    if (!attr[dev]) {
        cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)(smem + kMaxLevels * sizeof(StepItem)));
        if (e != cudaSuccess) return e;
        attr[dev] = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = smem + (size_t)tp.nact * sizeof(StepItem);   // + the active levels' items
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kfn, ep, tp, ipl, tm);
}

template <int KIND>
cudaError_t launch_chunk_k(const ChunkCfg& c, int grid, cudaStream_t st, const EngineParams& ep,
                           const TickParams& tp, int ipl, const TmapSet& tm)
{
    constexpr bool two_d = KIND == ADV_DIFF_2D || KIND == RD_2D;
    // periodic kinds: truncated segments (0) or cyclic whole lines (1); Burgers:
    // Dirichlet whole lines (2) or Dirichlet ends + truncated middles (-1)
    constexpr bool periodic = KIND != BURGERS_1D;
    constexpr int MA = periodic ? 0 : 2, MB = periodic ? 1 : -1;
    if (periodic && c.mode != MA && c.mode != MB) return cudaErrorInvalidValue;
#define RIDC_CHUNK_CASE(ID, NT, ROWS, NSTAGE, KC)                                              \
    if (c.id == ID && two_d == (ROWS == 3)) {                                                  \
        if constexpr (two_d == (ROWS == 3))                                                    \
            return c.mode == MA ? launch_chunk_t<KIND, NT, ROWS, NSTAGE, MA, KC>(grid, c.smem, st, ep, tp, ipl, tm) \
                                : launch_chunk_t<KIND, NT, ROWS, NSTAGE, MB, KC>(grid, c.smem, st, ep, tp, ipl, tm); \
    }
    RIDC_CHUNK_CONFIGS(RIDC_CHUNK_CASE)
#undef RIDC_CHUNK_CASE
    return cudaErrorInvalidValue;
}

// ---- resident FEBE kernel (ridc_resident.cuh): same NT as the tick config
// (the block scans' association, hence the rounding, depends on NT)
template <int KIND, int NT, int MODE>
cudaError_t resident_t(bool launch, int grid, cudaStream_t st, const ResidentParams& rp, int* per_sm)
{
    auto kfn = k_resident_febe<KIND, NT, MODE>;
    if (!launch) return cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, kfn, NT, 0);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;   // all segments co-resident (neighbour waits)
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kfn, rp);
}

// mode: the common segment mode (0 truncated segments, 1 cyclic whole line,
// 2 Dirichlet whole line) or -1 (mixed: Dirichlet ends + truncated middle)
template <int KIND>
cudaError_t resident_k(int nt, int mode, bool launch, int grid, cudaStream_t st, const ResidentParams& rp,
                       int* per_sm)
{
    // periodic kinds have truncated (0) or cyclic (1) segments; Burgers has
    // Dirichlet whole lines (2) or Dirichlet ends around truncated middles (-1)
    constexpr bool periodic = KIND != BURGERS_1D;
    constexpr int MA = periodic ? 0 : 2, MB = periodic ? 1 : -1;
    if (mode != MA && mode != MB) {
        if (periodic) return cudaErrorInvalidValue;
        mode = MB;
    }
#define RIDC_RES_NT(NT)                                                                   \
    case NT:                                                                              \
        return mode == MA ? resident_t<KIND, NT, MA>(launch, grid, st, rp, per_sm)        \
                          : resident_t<KIND, NT, MB>(launch, grid, st, rp, per_sm);
    switch (nt) {
        RIDC_RES_NT(64)
        RIDC_RES_NT(128)
        RIDC_RES_NT(256)
        RIDC_RES_NT(512)
    default: return cudaErrorInvalidValue;
    }
#undef RIDC_RES_NT
}

template <int KIND, int NT, int MODE, bool SYS, int MINB>
cudaError_t levels_t(bool launch, int grid, cudaStream_t st, const LevelsParams& lp, const TmapSet& tm,
                     int* per_sm)
{
    auto kfn = k_resident_levels<KIND, NT, MODE, kResStages, SYS, MINB>;
    const size_t smem = LevSmem<NT, kResStages>::BYTES + 1024;
    static bool attr[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
    if (!attr[dev]) {
        cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        attr[dev] = true;
    }
    if (!launch) return cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, kfn, NT, smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;   // every level's segments co-resident (flag waits)
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kfn, lp, tm);
}

template <int KIND, bool SYS>
cudaError_t levels_k(int nt, int mode, bool launch, int grid, cudaStream_t st, const LevelsParams& lp,
                     const TmapSet& tm, int* per_sm, bool dense)
{
    constexpr bool periodic = KIND != BURGERS_1D;
    constexpr int MA = periodic ? 0 : 2, MB = periodic ? 1 : -1;
    if (mode != MA && mode != MB) {
        if (periodic) return cudaErrorInvalidValue;
        mode = MB;
    }
#define RIDC_LEV_NT(NT, MINB)                                                                    \
        return mode == MA ? levels_t<KIND, NT, MA, SYS, MINB>(launch, grid, st, lp, tm, per_sm)  \
                          : levels_t<KIND, NT, MB, SYS, MINB>(launch, grid, st, lp, tm, per_sm);
    switch (nt) {
    case 64: RIDC_LEV_NT(64, 1)
    case 128: RIDC_LEV_NT(128, 1)
    case 256:
        if (dense) { RIDC_LEV_NT(256, 2) }
        RIDC_LEV_NT(256, 1)
    case 512: RIDC_LEV_NT(512, 1)
    default: return cudaErrorInvalidValue;
    }
#undef RIDC_LEV_NT
}

// ---- carry-exchange FEBE march (ridc_febe_carry.cuh): nt threads (multiple of 32)
template <int KIND>
cudaError_t febe_carry_k(bool launch, int grid, int nt, cudaStream_t st, const CarryParams& cp, int* per_sm)
{
    auto kfn = k_febe_carry<KIND>;
    if (!launch) return cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, kfn, nt, 0);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(nt);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;   // all tiles co-resident (neighbour carry waits)
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kfn, cp);
}

// ---- warp-chunk carry FEBE march (ridc_febe_carry.cuh k_febe_wcarry): one
// cooperative launch, wpc warps (512-point chunks) per CTA
template <int KIND>
cudaError_t febe_wcarry_k(bool launch, int k, int grid, int nt, cudaStream_t st, const CarryParams& cp, int* per_sm)
{
    auto kfn = k == 32 ? k_febe_wcarry<KIND, 32> : k_febe_wcarry<KIND, 16>;
    if (!launch) return cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, kfn, nt, 0);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(nt);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;   // all chunks co-resident (neighbour carry waits)
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kfn, cp);
}

// ---- streaming FEBE sweep (ridc_sweep.cuh): one persistent CTA per SM, PDL
// between consecutive steps
template <int KIND, int NT>
cudaError_t sweep_t(int grid, cudaStream_t st, const SweepParams& sp, const TmapSet& tm, long long off,
                    long long target)
{
    auto kfn = k_sweep_febe<KIND, NT>;
    const size_t smem = sweep_smem<NT>();
    static bool attr[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
    if (!attr[dev]) {
        cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        attr[dev] = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kfn, sp, tm, off, target);
}

// ---- warp-sweep FEBE (ridc_sweep_warp.cuh): one 512-thread CTA per SM, every
// warp sweeps its own range; PDL between consecutive steps
template <int KIND>
cudaError_t sweep_warp_t(int grid, cudaStream_t st, const SweepParams& sp, const TmapSet& tm, long long off,
                         long long target)
{
    auto kfn = k_sweep_febe_warp<KIND>;
    const size_t smem = warp_sweep_smem();
    static bool attr[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
    if (!attr[dev]) {
        cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        attr[dev] = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kWarpSweepWarps * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kfn, sp, tm, off, target);
}

// ---- 2-D streaming FEBE sweep (ridc_sweep2d.cuh): nx = 16 NT, 512 / NT CTAs per SM
template <int KIND, int NT>
cudaError_t sweep2d_t(int grid, cudaStream_t st, const Sweep2DParams& sp, const TmapSet& tm, long long off,
                      long long target)
{
    auto kfn = k_sweep2d_febe<KIND, NT>;
    const size_t smem = sweep2d_smem<NT>();
    static bool attr[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
    if (!attr[dev]) {
        cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        attr[dev] = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kfn, sp, tm, off, target);
}

template <int KIND>
cudaError_t sweep2d_k(int nt, int grid, cudaStream_t st, const Sweep2DParams& sp, const TmapSet& tm, long long off,
                      long long target)
{
    switch (nt) {
    case 128: return sweep2d_t<KIND, 128>(grid, st, sp, tm, off, target);
    case 256: return sweep2d_t<KIND, 256>(grid, st, sp, tm, off, target);
    case 512: return sweep2d_t<KIND, 512>(grid, st, sp, tm, off, target);
    }
    return cudaErrorInvalidValue;
}

// ---- 1-D level sweep (ridc_sweep_levels.cuh): one 512-thread CTA per SM
template <int KIND>
cudaError_t sweep_levels_k(int grid, cudaStream_t st, const EngineParams& ep, const TickParams& tp,
                           const SweepParams& sp, const TmapSet& tm)
{
    auto kfn = k_sweep_levels<KIND>;
    static bool attr[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
    if (!attr[dev]) {
        cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)sweep_levels_smem(kMaxLevels));
        if (e != cudaSuccess) return e;
        attr[dev] = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(512);
    cfg.dynamicSmemBytes = sweep_levels_smem(tp.nact);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kfn, ep, tp, sp, tm);
}

// ---- resident RIDC-2 (ridc_carry_res2.cuh): one cooperative launch per interval
template <int KIND>
cudaError_t carry_res2_k(bool launch, int grid, int nt, cudaStream_t st, const CarryRes2Params& cp, int* per_sm)
{
    auto kfn = k_carry_res2<KIND>;
    const size_t smem = carry_res2_smem(nt);
    cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    if (!launch) return cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, kfn, nt, smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(nt);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;   // all tiles co-resident (neighbour carry waits)
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kfn, cp);
}

// ---- resident RIDC-2, one chunk per warp (ridc_carry_res2w.cuh): two CTAs per SM
template <int KIND>
cudaError_t carry_res2w_k(bool launch, int grid, cudaStream_t st, const CarryRes2Params& cp, int* per_sm)
{
    auto kfn = cp.T == 14 ? k_carry_res2w<KIND, 14> : k_carry_res2w<KIND, 7>;
    const int nt = 32 * cp.T;
    const size_t smem = carry_res2w_smem(cp.T);
    cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    if (!launch) return cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, kfn, nt, smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(nt);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;   // all chunks co-resident (neighbour carry waits)
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kfn, cp);
}

template <int KIND, int K>
cudaError_t carry_levels_t(int grid, int wpc, cudaStream_t st, const EngineParams& ep, const TickParams& tp,
                           const CarryLevParams& cp, const TmapSet& tm, unsigned tick)
{
    auto kfn = k_carry_levels<KIND, K>;
    static bool attr[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
    if (!attr[dev]) {
        cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)carry_levels_smem<K>());
        if (e != cudaSuccess) return e;
        attr[dev] = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(32 * wpc);
    cfg.dynamicSmemBytes = carry_levels_smem<K>();
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kfn, ep, tp, cp, tm, tick);
}

// ---- carry-exchange level tick (ridc_carry_levels.cuh): one chunk of 32 k
// points per warp (k = 16 or 32), wpc warps per CTA, PDL between ticks
template <int KIND>
cudaError_t carry_levels_k(int grid, int wpc, int k, cudaStream_t st, const EngineParams& ep, const TickParams& tp,
                           const CarryLevParams& cp, const TmapSet& tm, unsigned tick)
{
    return k == 32 ? carry_levels_t<KIND, 32>(grid, wpc, st, ep, tp, cp, tm, tick)
                   : carry_levels_t<KIND, 16>(grid, wpc, st, ep, tp, cp, tm, tick);
}

// ---- 2-D level sweep (ridc_sweep2d_levels.cuh): one CTA of nx / 16 threads per SM
template <int KIND, int NT>
cudaError_t sweep2d_levels_t(int grid, cudaStream_t st, const EngineParams& ep, const TickParams& tp,
                             const SweepLevParams& sp, const TmapSet& tm)
{
    auto kfn = k_sweep2d_levels<KIND, NT>;
    const size_t smem = SweepLevSmem<NT>::bytes(tp.nact);
    static bool attr[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
    if (!attr[dev]) {
        cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)SweepLevSmem<NT>::bytes(kMaxLevels));
        if (e != cudaSuccess) return e;
        attr[dev] = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kfn, ep, tp, sp, tm);
}

template <int KIND>
cudaError_t sweep2d_levels_k(int nt, int grid, cudaStream_t st, const EngineParams& ep, const TickParams& tp,
                             const SweepLevParams& sp, const TmapSet& tm)
{
    switch (nt) {
    case 256: return sweep2d_levels_t<KIND, 256>(grid, st, ep, tp, sp, tm);
    case 512: return sweep2d_levels_t<KIND, 512>(grid, st, ep, tp, sp, tm);
    }
    return cudaErrorInvalidValue;
}

// one 512-thread CTA per SM; grid = CTAs
template <int KIND>
cudaError_t sweep_k(int nt, int grid, cudaStream_t st, const SweepParams& sp, const TmapSet& tm, long long off,
                    long long target)
{
    return nt == 512 ? sweep_t<KIND, 512>(grid, st, sp, tm, off, target)
           : nt == 32 ? sweep_warp_t<KIND>(grid, st, sp, tm, off, target)
                      : cudaErrorInvalidValue;
}

}  // namespace ridc
