// trace.h -- NVTX ranges around the library's entry points and phases
// (broadcast / GEMM / ewise ranges for nsys-style timelines).
// NVTX v3 is header-only: with no tool attached a push/pop is a few
// instructions and no library is loaded.
#pragma once

#include <nvtx3/nvToolsExt.h>

namespace mpmm {

struct TraceRange {
  explicit TraceRange(const char* name) { nvtxRangePushA(name); }
  ~TraceRange() { nvtxRangePop(); }
  TraceRange(const TraceRange&) = delete;
  TraceRange& operator=(const TraceRange&) = delete;
};

}  // namespace mpmm
