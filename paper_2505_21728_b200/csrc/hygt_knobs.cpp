// hygt_knobs.cpp -- process-wide development knobs (see hygt_knobs.h).
#include "hygt_knobs.h"

#include <map>
#include <mutex>
#include <string>

namespace hygt_gpu {
std::mutex g_mu;
std::map<std::string, int>& table() {
  static std::map<std::string, int> t;
  return t;
}

int knob(const char* name, int dflt) {
  std::lock_guard<std::mutex> lk(g_mu);
  const auto it = table().find(name);
  return it == table().end() ? dflt : it->second;
}
}  // namespace hygt_gpu

// Debug hooks (not in the public header): set one knob, or clear them all.
extern "C" void hygt_debug_set_knob(const char* name, int value) {
  if (!name) return;
  std::lock_guard<std::mutex> lk(hygt_gpu::g_mu);
  hygt_gpu::table()[name] = value;
}
extern "C" void hygt_debug_clear_knobs() {
  std::lock_guard<std::mutex> lk(hygt_gpu::g_mu);
  hygt_gpu::table().clear();
}
