// Runtime-compiled tile-pass kernels (qsv_jit.cu; sources from qsv_tile_jit.cuh).
#pragma once

#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "qsv_internal.cuh"

namespace qsv {

struct JitKernel {
  cudaKernel_t kernel = nullptr;
  int regs = 0;
};

// Compile / fetch every source (nullptr or empty entries are skipped); out[i]
// stays null when source i failed (first_err receives the first message).
int jit_kernels(const std::vector<const std::string*>& srcs, std::vector<JitKernel>& out,
                std::string* first_err);
// the source's kernel is already loaded in this process
bool jit_cached(const std::string& src);
// raise the dynamic shared-memory limit of a kernel on the current device
int jit_set_smem(JitKernel k, size_t bytes);

// Host image of the kernel's __grid_constant__ parameter (layout shared with
// the generated `struct PassParams`): the fixed head, then `ndata` double2.
struct JitParamHead {
  double2* a;
  unsigned long long ntiles;
  unsigned long long* ctr;
  int nostagger;
  int stat;  // one tile per CTA (group 0 takes tile blockIdx.x), no work counter
  FixedBits tb;
};
static_assert(sizeof(JitParamHead) % 16 == 0, "payload must start 16-byte aligned");
constexpr size_t kJitMaxParamBytes = 32764;

}  // namespace qsv
