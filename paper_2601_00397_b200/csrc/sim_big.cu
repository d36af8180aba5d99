// sim_big.cu — the event loop for slot capacities above what shared memory holds
// (max_running > 4096): k_sim<true, true>, slot state in a global scratch slice per warp,
// the predictor blob read from global memory. Its own translation unit, like sim_tput.cu,
// so the shared-memory variants' code is unchanged.
#define TWB_SIM_TPUT_TU 1
#define TWB_SIM_BIG_TU 1
#include "sim.cu"
