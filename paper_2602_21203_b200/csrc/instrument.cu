// instrument.cu -- launch counter and optional per-phase CUDA-event instrumentation used
// by bench.py to time the dominant kernel live inside the timed region.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdio>

#include "../../include/squint.h"
#include "common.cuh"

namespace sq {
struct LaunchInfo;
static std::atomic<long> g_launches{0};
static void** g_events = nullptr;  // cudaEvent_t[n_phases][reps][2]
static int g_phases = 0, g_reps = 0;

// Optional launch timeline (squint_set_launch_events): an event recorded on the launch stream
// right before each launch, so event k..k+1 brackets launch k (kernel + any gap before k+1).
static void** g_lev = nullptr;
static int g_lev_n = 0, g_lev_used = 0;
struct LaunchInfo {
  const char* name;
  double flops, bytes;
};
static LaunchInfo g_info[8192];

void note_launch(cudaStream_t s, const char* name, double flops, double bytes) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (g_lev && g_lev_used < g_lev_n) {
    if (g_lev_used < 8192) g_info[g_lev_used] = LaunchInfo{name, flops, bytes};
    cudaError_t e = cudaEventRecordWithFlags((cudaEvent_t)g_lev[g_lev_used++], s, cudaEventRecordExternal);
    if (e != cudaSuccess) {
      fprintf(stderr, "[squint] launch event %d: %s\n", g_lev_used - 1, cudaGetErrorString(e));
      cudaGetLastError();
    }
  }
}
long launch_count() { return g_launches.load(); }
bool instrumentation_active() { return g_lev != nullptr || g_events != nullptr; }

PhaseScope::PhaseScope(int phase, int rep, cudaStream_t st) : idx(-1), s(st) {
  if (!g_events || phase >= g_phases || rep >= g_reps) return;
  idx = (phase * g_reps + rep) * 2;
  cudaEventRecordWithFlags((cudaEvent_t)g_events[idx], s, cudaEventRecordExternal);
}
PhaseScope::~PhaseScope() {
  if (idx >= 0) cudaEventRecordWithFlags((cudaEvent_t)g_events[idx + 1], s, cudaEventRecordExternal);
}

}  // namespace sq

extern "C" {

SQUINT_API long squint_launch_count(void) { return sq::launch_count(); }

// Closes the launch timeline: records the next event with no launch (end of the last kernel).
SQUINT_API squint_status squint_record_launch_event(squint_stream_t s) {
  if (sq::g_lev && sq::g_lev_used < sq::g_lev_n) {
    if (sq::g_lev_used < 8192) sq::g_info[sq::g_lev_used] = sq::LaunchInfo{"(end)", 0, 0};
    cudaEventRecordWithFlags((cudaEvent_t)sq::g_lev[sq::g_lev_used++], (cudaStream_t)s, cudaEventRecordExternal);
  }
  return SQUINT_OK;
}
// Name and algorithmic work of launch i of the current/last timeline.
SQUINT_API squint_status squint_launch_info(int i, const char** name, double* flops, double* bytes) {
  if (i < 0 || i >= 8192 || !name || !flops || !bytes) return SQUINT_EINVAL;
  *name = sq::g_info[i].name ? sq::g_info[i].name : "";
  *flops = sq::g_info[i].flops;
  *bytes = sq::g_info[i].bytes;
  return SQUINT_OK;
}

SQUINT_API int squint_set_launch_events(void** events, int n) {
  const int used = sq::g_lev_used;
  sq::g_lev = events;
  sq::g_lev_n = events ? n : 0;
  sq::g_lev_used = 0;
  return used;
}

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
