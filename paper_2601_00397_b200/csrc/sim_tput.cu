// sim_tput.cu — the throughput variant of the event loop (k_sim<true>) in its own
// translation unit; see the note at sim_tput_prepare in sim.cu.
#define TWB_SIM_TPUT_TU 1
#include "sim.cu"
