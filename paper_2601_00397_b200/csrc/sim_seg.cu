// sim_seg.cu — the event loop's busy-period segments for the latency regime (at most 8
// configs per SM): k_seg_plan picks segment boundaries, k_sim_seg simulates every segment
// speculatively from an empty engine (mode 1 of run_config), k_sim_join chains the valid
// pieces, replays the Timekeeper log and writes each config's record.
// The throughput-variant geometry (blob read from global memory, <= 128 registers), in its
// own translation unit so the other variants' code is unchanged.
#define TWB_SIM_TPUT_TU 1
#define TWB_SIM_SEG_TU 1
#define TWB_TPUT_TK_FAST 1  // the join pass replays the Timekeeper: keep tk_run's entry closed forms
#ifndef TWB_TPUT_INLINE_PRED
#define TWB_SIM_OUTLINE_PRED 1
#endif
#ifndef TWB_TPUT_INLINE_COLD2
#define TWB_SIM_OUTLINE_COLD2 1
#endif
#include "sim.cu"
