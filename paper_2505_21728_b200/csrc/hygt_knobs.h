// hygt_knobs.h -- development knobs of the kernel-family selection (test hook only).
//
// The library reads no environment variables (the reference contract). Plan
// creation takes its documented choices from hygt_plan_options (include/hygt_gpu.h); the
// remaining layout / variant switches the parity suite sweeps are set through the debug hook
// hygt_debug_set_knob(name, value) (not in the public header) and default to the measured best.
#pragma once

namespace hygt_gpu {
// The value set with hygt_debug_set_knob, or dflt.
int knob(const char* name, int dflt);
}  // namespace hygt_gpu
