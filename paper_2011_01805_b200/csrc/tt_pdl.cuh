// tt_pdl.cuh -- programmatic dependent launch (PDL) for every kernel of the library.
//
// Consecutive operators on one stream form dependency chains (fold -> tree pass ->
// next product's fold ...).  Each kernel is launched with the programmatic
// stream-serialization attribute, so the next kernel's grid is dispatched while
// the current one still runs: its CTAs land on SMs as the current kernel's CTAs
// retire and sit in `griddepcontrol.wait` until the current grid has completed
// and its memory is visible.  What overlaps is the launch processing, CTA
// dispatch and the prologue -- not data work: every kernel waits before its
// first global memory access (read or write), so a kernel never sees an
// unfinished producer and never overwrites what an unfinished consumer reads.
// A kernel releases its own dependents only after its wait, so at most two
// grids of a stream are in flight.  TT_PDL=0 launches without the attribute
// (the kernels' wait / release are then no-ops).
#pragma once

#include <cuda_runtime.h>

#include <utility>

#include "tt_launch.hpp"

namespace ttb {

// First statement of every kernel: wait for the preceding grid, then allow the
// next one to be dispatched.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Wait only: the kernel releases its dependents when its CTAs exit (for
// shared-memory-heavy kernels whose successors should not land on SMs they
// still hold).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_enter(bool release_late) {
  if (release_late)
    pdl_wait();
  else
    pdl_enter();
}

int pdl_enabled();
// The stream's last launch releases its dependents only at exit: the next
// launch may take the attribute whatever its footprint.
void pdl_note_late_release(const LaunchCtx& c);
int pdl_oversub();
// Whether this launch may overlap its predecessor on the stream, and record
// its footprint for the next launch (see tt_kernels.cu).
bool pdl_allow(const LaunchCtx& c, const void* kernel, int threads, size_t dyn_smem, int64_t grid);
bool pdl_would_allow(const LaunchCtx& c, const void* kernel, int threads, size_t dyn_smem);

// kernel<<<grid, block, smem, c.stream>>>(args...) with the PDL attribute
template <typename... KArgs, typename... Args>
inline void launch_k(const LaunchCtx& c, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                     Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c.stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_allow(c, reinterpret_cast<const void*>(kernel),
                           static_cast<int>(block.x * block.y * block.z), smem,
                           static_cast<int64_t>(grid.x) * grid.y * grid.z) ? 1 : 0;
  // launch errors surface through cudaGetLastError() in post_launch()
  (void)cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

}  // namespace ttb
