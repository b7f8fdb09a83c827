// ridc_inst.cu -- explicit instantiation of the launch entry points of ONE
// problem kind and ONE kernel family, selected at compile time:
//   RIDC_INST_KIND  1..5 (ridc::Kind)
//   RIDC_INST_PART  0: tick kernel + single-op item kernel
//                   1: resident FEBE march (1-D kinds; + the carry-exchange march, RD)
//                   2: resident level march, GPU-scope flags (1-D kinds)
//                   3: resident level march, system-scope flags (1-D kinds)
// __graft_entry__.build() compiles this file once per (kind, part) in
// parallel and links the objects with ridc_engine.cu into libridc_b200.so.
#include "ridc_dispatch.cuh"

#ifndef RIDC_INST_KIND
#error "RIDC_INST_KIND must be defined"
#endif
#ifndef RIDC_INST_PART
#error "RIDC_INST_PART must be defined"
#endif

namespace ridc {

#if RIDC_INST_PART == 0
#if RIDC_INST_KIND >= 4
template cudaError_t sweep2d_k<RIDC_INST_KIND>(int, int, cudaStream_t, const Sweep2DParams&, const TmapSet&,
                                               long long, long long);
template cudaError_t sweep2d_levels_k<RIDC_INST_KIND>(int, int, cudaStream_t, const EngineParams&,
                                                      const TickParams&, const SweepLevParams&, const TmapSet&);
#endif
template cudaError_t launch_chunk_k<RIDC_INST_KIND>(const ChunkCfg&, int, cudaStream_t, const EngineParams&,
                                                    const TickParams&, int, const TmapSet&);
template cudaError_t launch_item_k<RIDC_INST_KIND>(const LaunchCfg&, int, cudaStream_t, const DevProblem&,
                                                   const DevSolve&, const StepItem&, unsigned long long*);
#elif RIDC_INST_PART == 1
template cudaError_t resident_k<RIDC_INST_KIND>(int, int, bool, int, cudaStream_t, const ResidentParams&, int*);
#if RIDC_INST_KIND == 3
template cudaError_t febe_carry_k<RIDC_INST_KIND>(bool, int, int, cudaStream_t, const CarryParams&, int*);
template cudaError_t febe_wcarry_k<RIDC_INST_KIND>(bool, int, int, int, cudaStream_t, const CarryParams&, int*);
template cudaError_t sweep_k<RIDC_INST_KIND>(int, int, cudaStream_t, const SweepParams&, const TmapSet&, long long,
                                             long long);
template cudaError_t sweep_levels_k<RIDC_INST_KIND>(int, cudaStream_t, const EngineParams&, const TickParams&,
                                                    const SweepParams&, const TmapSet&);
template cudaError_t carry_res2_k<RIDC_INST_KIND>(bool, int, int, cudaStream_t, const CarryRes2Params&, int*);
template cudaError_t carry_res2w_k<RIDC_INST_KIND>(bool, int, cudaStream_t, const CarryRes2Params&, int*);
template cudaError_t carry_levels_k<RIDC_INST_KIND>(int, int, int, cudaStream_t, const EngineParams&,
                                                    const TickParams&, const CarryLevParams&, const TmapSet&, unsigned);
#endif
#elif RIDC_INST_PART == 2
template cudaError_t levels_k<RIDC_INST_KIND, false>(int, int, bool, int, cudaStream_t, const LevelsParams&,
                                                     const TmapSet&, int*, bool);
#elif RIDC_INST_PART == 3
template cudaError_t levels_k<RIDC_INST_KIND, true>(int, int, bool, int, cudaStream_t, const LevelsParams&,
                                                    const TmapSet&, int*, bool);
#else
#error "unknown RIDC_INST_PART"
#endif

}  // namespace ridc
