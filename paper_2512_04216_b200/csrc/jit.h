// NVRTC specialisation of fused pass kernels (see jit.cu).
#pragma once
#include "program.h"

namespace svb {

// True when NVRTC and the driver entry points are usable in this process.
bool jit_available();

// Compile (cached) and launch every pass of `prog` as a specialised kernel.
// Returns false (nothing launched) when the JIT is unavailable or fails; the
// caller then runs the interpreter kernel.
template <typename R>
bool jit_launch_passes(cplx<R>* state, cplx<R>* out, const Program& prog, const PassDev* dpass, const uint8_t* dops,
                       cudaStream_t st, ProgramStats* stats, int nsm, bool zero_input);

// Asynchronous JIT for the calling thread: kernels not compiled yet are built
// by background threads and the program runs on the interpreter meanwhile.
void jit_set_async(bool on);

}  // namespace svb
