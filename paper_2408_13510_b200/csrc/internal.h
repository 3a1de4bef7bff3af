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

rs_status rs_internal_replay_batch(const rs_batch_cfg* cfg, const rs_trace_soa* tr,
                                   rs_req_out* out, rs_replay_stats* stats, void* workspace,
                                   size_t workspace_bytes, void* stream, const int* resident,
                                   void* inputs_done, const rs_trajectory* traj);

// The per-replay aggregates pass (stats_kernel) over a finished replay batch,
// after `wait_event` (may be null).
rs_status rs_internal_stats(const rs_trace_soa* tr, const rs_req_out* out, rs_replay_stats* stats,
                            void* stream, void* wait_event);
