// instrument.cu -- launch counter and optional per-phase CUDA-event instrumentation used
// by bench.py to time the dominant kernel live inside the timed region.
#include <cuda_runtime.h>

#include <atomic>

#include "../../include/squint.h"
#include "common.cuh"

namespace sq {

static std::atomic<long> g_launches{0};
static void** g_events = nullptr;  // cudaEvent_t[n_phases][reps][2]
static int g_phases = 0, g_reps = 0;

void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
long launch_count() { return g_launches.load(); }

PhaseScope::PhaseScope(int phase, int rep, cudaStream_t st) : idx(-1), s(st) {
  if (!g_events || phase >= g_phases || rep >= g_reps) return;
  idx = (phase * g_reps + rep) * 2;
  cudaEventRecord((cudaEvent_t)g_events[idx], s);
}
PhaseScope::~PhaseScope() {
  if (idx >= 0) cudaEventRecord((cudaEvent_t)g_events[idx + 1], s);
}

}  // namespace sq

extern "C" {

SQUINT_API long squint_launch_count(void) { return sq::launch_count(); }

SQUINT_API squint_status squint_set_phase_events(void** events, int n_phases, int reps) {
  sq::g_events = events;
  sq::g_phases = events ? n_phases : 0;
  sq::g_reps = events ? reps : 0;
  return SQUINT_OK;
}

SQUINT_API const char* squint_phase_name(int k) {
  static const char* names[] = {"insert",     "act_encode",   "act_mlp",     "enc_fwd",      "proj_fwd",
                                "actor_fwd",  "heads_fwd",    "target_ce",   "critic_bwd",   "critic_dw",
                                "enc_bwd",    "alpha_adam_c", "actor_loss",  "actor_bwd",    "actor_dw",
                                "adam_a_polyak"};
  return (k >= 0 && k < (int)(sizeof(names) / sizeof(names[0]))) ? names[k] : "";
}

}  // extern "C"
