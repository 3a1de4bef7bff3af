// Engine-internal entry points shared between engine.cu and host_api.cu
// (not part of the C ABI in include/rs_abi.h).
#pragma once
#include <stdint.h>

#include "../../include/rs_abi.h"

// true when `cfg` runs on the lane-per-instance kernel (whole-prompt
// prefill, <= 64 instances), the only kernel that accepts streamed inputs
bool rs_internal_fast_path(const rs_batch_cfg* cfg);

// rs_replay_batch with optional streamed inputs: `resident` (device int,
// may be null) counts the requests of every replay already on the device;
// `inputs_done` (cudaEvent_t, may be null) is waited on before the
// percentile pass; `traj` (may be null) turns on record_trajectory.
// pass as `inputs_done` to skip the stats launch (the caller issues it
// later with rs_internal_stats)
#define kDeferStats (reinterpret_cast<void*>(static_cast<uintptr_t>(1)))

// Streamed outputs (lane-per-instance kernel, equal-length replays): the
// replays publish per-request results chunk by chunk as they become final.
// Chunk c covers request indices [bounds[c-1], bounds[c]) of every replay;
// marks[c] (device, zeroed by the caller) counts the replays whose requests
// below bounds[c] have all completed (their outputs final), and reaches
// num_replays when the chunk can be copied back.
struct rs_internal_stream_out {
  int* marks;
  int nbounds;
  int bounds[16];
  int used;  // out: 1 when the launched kernel publishes (the latency-regime
             // build has a streamed-output variant; other plans copy after)
};

rs_status rs_internal_replay_batch(const rs_batch_cfg* cfg, const rs_trace_soa* tr,
                                   rs_req_out* out, rs_replay_stats* stats, void* workspace,
                                   size_t workspace_bytes, void* stream, const int* resident,
                                   void* inputs_done, const rs_trajectory* traj,
                                   rs_internal_stream_out* sout = nullptr);

// The per-replay aggregates pass (stats_kernel) over a finished replay batch,
// after `wait_event` (may be null).
rs_status rs_internal_stats(const rs_trace_soa* tr, const rs_req_out* out, rs_replay_stats* stats,
                            void* stream, void* wait_event);

// Host Q-network parameters: every one finite.  The device forward skips
// exact-zero inputs (w * 0 = 0 for finite w, so the result is unchanged);
// an inf / NaN weight would turn the reference's w * 0 into NaN, which the
// skip does not reproduce, so such networks are rejected (RS_ERR_UNSUPPORTED).
rs_status rs_internal_check_weights(const double* params, size_t count);
