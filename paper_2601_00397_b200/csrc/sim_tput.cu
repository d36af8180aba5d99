// sim_tput.cu — the throughput variant of the event loop (k_sim<true>) in its own
// translation unit; see the note at sim_tput_prepare in sim.cu.
//
// Code placement differs from the latency variant: with 16 warps per SM at different
// points of the loop, instruction fetch bounds this variant, so the prediction-cache miss
// path and the audit dump live out of line (A/B on config 5, 65,536 configs: 289 ->
// 248 ms for the miss path, 289 -> 263 ms for the dump; profiles/README.md).
#define TWB_SIM_TPUT_TU 1
#ifndef TWB_TPUT_INLINE_PRED
#define TWB_SIM_OUTLINE_PRED 1
#endif
#ifndef TWB_TPUT_INLINE_COLD2
#define TWB_SIM_OUTLINE_COLD2 1
#endif
#ifdef TWB_TPUT_OUTLINE_IDLE
#define TWB_SIM_OUTLINE_IDLE 1
#endif
#ifdef TWB_TPUT_OUTLINE_WIDE
#define TWB_SIM_OUTLINE_WIDE 1
#endif
#include "sim.cu"
