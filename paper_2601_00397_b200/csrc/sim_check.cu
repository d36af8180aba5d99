// sim_check.cu — the event loop with on-device invariant counters (debug builds of the
// loop: tw_sim_set_checks). The throughput-variant geometry (blob read from global memory,
// slot state in shared memory), compiled in its own translation unit so the product
// variants' code is unchanged. Results are identical to the other variants'.
#define TWB_SIM_TPUT_TU 1
#define TWB_SIM_CHECK 1
#include "sim.cu"
