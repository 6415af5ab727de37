// Host wall-time breakdown of the solve setup (APC_SETUP_PROF=1).
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <utility>
#include <vector>

#include "apc_internal.hpp"

namespace apc {

// ---- setup profiler (APC_SETUP_PROF=1) ----
namespace {
std::vector<std::pair<const char*, double>> t_prof;  // single-solve diagnostics (not thread-safe)
double now_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
}  // namespace
bool SetupProf::on() {
  static const bool v = std::getenv("APC_SETUP_PROF") != nullptr;
  return v;
}
void SetupProf::add(const char* name, double ms) {
  if (!on()) return;
  for (auto& e : t_prof)
    if (std::strcmp(e.first, name) == 0) {
      e.second += ms;
      return;
    }
  t_prof.emplace_back(name, ms);
}
void SetupProf::dump_and_reset(const char* title) {
  if (!on()) return;
  std::fprintf(stderr, "%s:", title);
  for (auto& e : t_prof) std::fprintf(stderr, " %s %.1f", e.first, e.second);
  std::fprintf(stderr, " (ms)\n");
  t_prof.clear();
}
ProfScope::ProfScope(const char* n) : name(n), t0(SetupProf::on() ? now_ms() : 0.0) {}
ProfScope::~ProfScope() {
  if (SetupProf::on()) SetupProf::add(name, now_ms() - t0);
}

}  // namespace apc
