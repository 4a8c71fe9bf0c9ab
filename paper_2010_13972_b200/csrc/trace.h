// trace.h -- NVTX ranges around the C-ABI entry points (host preprocessing and
// kernel launches), so an nsys / ncu --nvtx timeline shows extract / pack /
// plan / write / shap / interactions by name.  NVTX v3 is header-only: with no
// tool attached each push/pop is a branch on a null function pointer.
#pragma once
#include <nvtx3/nvToolsExt.h>

namespace gts {
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
}  // namespace gts

#define GTS_NVTX(name) ::gts::NvtxRange gts_nvtx_range_(name)
