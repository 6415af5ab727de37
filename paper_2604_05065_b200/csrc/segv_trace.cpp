// Debug aid: APC_SEGV_TRACE=1 prints a native backtrace on SIGSEGV (frame
// addresses are resolved offline with addr2line against the same .so).
#include <execinfo.h>
#include <signal.h>
#include <unistd.h>

#include <cstdlib>

namespace {
void on_segv(int sig) {
  void* frames[64];
  const int n = backtrace(frames, 64);
  backtrace_symbols_fd(frames, n, 2);
  signal(sig, SIG_DFL);
  raise(sig);
}
struct Install {
  Install() {
    if (std::getenv("APC_SEGV_TRACE")) signal(SIGSEGV, on_segv);
  }
} install;
}  // namespace
