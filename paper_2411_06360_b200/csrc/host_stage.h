// Host-side staging + classification of a session vector (host_stage.cpp, used by host.cu).
#pragma once

#include <stdint.h>

#include "../../include/rsr_b200.h"

namespace rsr {

enum StageKind { kStageI32 = 0, kStageWide = 1, kStageF32 = 2, kStageF64 = 3, kStageFixed = 4, kStageNonFinite = -1 };

struct StageInfo {
  int kind;          // StageKind
  uint64_t max_abs;  // max |v| for the integer classes (0 if unknown); max |v_q| for kStageFixed
  int exp2 = 0;      // kStageFixed: v_q = round(v * 2^exp2), staged as int64
};

// Copy v [n] of type t into dst (8 * n bytes of pinned staging) in the representation its class
// computes in: int32 for kStageI32, int64 for kStageWide, the input type for the float classes.
// force_i32 (int32 input only): stage as int32 whatever the sum (int32 arithmetic requested).
StageInfo stage_vector(const void* src, rsr_dtype t, int64_t n, void* dst, bool force_i32);

}  // namespace rsr
