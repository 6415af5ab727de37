// A persistent host worker pool for host_parallel_for (host_rng.hpp): the
// exact-order host factorizations split per-column work into one task per
// reflection / pivot step, far too often for a thread start-up each time.
#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <exception>
#include <mutex>
#include <thread>
#include <vector>

#include "apc_internal.hpp"

namespace apc {
namespace {

thread_local bool t_in_pool = false;

class Pool {
 public:
  Pool() {
    unsigned hc = std::thread::hardware_concurrency();
    nworkers_ = static_cast<int>(std::max(1u, std::min(hc ? hc : 1u, 32u))) - 1;
    for (int w = 0; w < nworkers_; ++w) threads_.emplace_back([this, w] { loop(w); });
  }
  ~Pool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : threads_) t.join();
  }
  int workers() const { return nworkers_; }

  // chunks [0, nt) of [0, n); the caller runs chunk 0, workers the rest
  void run(i64 n, int nt, void (*fn)(void*, i64, i64), void* ctx) {
    std::unique_lock<std::mutex> job(run_mu_);  // one job at a time
    {
      std::lock_guard<std::mutex> lk(mu_);
      n_ = n;
      nt_ = nt;
      fn_ = fn;
      ctx_ = ctx;
      next_.store(1);
      done_ = 0;
      err_ = nullptr;
      ++gen_;
    }
    cv_.notify_all();
    work_chunks();
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [this] { return done_ == nt_ - 1; });
    if (err_) std::rethrow_exception(err_);
  }

 private:
  void chunk(int c) {
    const i64 per = (n_ + nt_ - 1) / nt_;
    const i64 b = c * per, e = std::min(n_, b + per);
    if (b < e) fn_(ctx_, b, e);
  }
  void work_chunks() {  // the caller's share: chunk 0, then any unclaimed
    try {
      chunk(0);
    } catch (...) {
      std::lock_guard<std::mutex> lk(mu_);
      if (!err_) err_ = std::current_exception();
    }
  }
  void loop(int) {
    t_in_pool = true;
    std::uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
      }
      for (;;) {
        const int c = next_.fetch_add(1);
        if (c >= nt_) break;
        try {
          chunk(c);
        } catch (...) {
          std::lock_guard<std::mutex> lk(mu_);
          if (!err_) err_ = std::current_exception();
        }
        std::lock_guard<std::mutex> lk(mu_);
        if (++done_ == nt_ - 1) done_cv_.notify_all();
      }
    }
  }

  int nworkers_ = 0;
  std::vector<std::thread> threads_;
  std::mutex mu_, run_mu_;
  std::condition_variable cv_, done_cv_;
  bool stop_ = false;
  std::uint64_t gen_ = 0;
  i64 n_ = 0;
  int nt_ = 1;
  void (*fn_)(void*, i64, i64) = nullptr;
  void* ctx_ = nullptr;
  std::atomic<int> next_{1};
  int done_ = 0;
  std::exception_ptr err_;
};

Pool& pool() {
  static Pool p;
  return p;
}

}  // namespace

int host_pool_workers() { return t_in_pool ? 0 : pool().workers(); }

void host_pool_run(i64 n, int nt, void (*fn)(void*, i64, i64), void* ctx) {
  if (t_in_pool || nt <= 1) {
    fn(ctx, 0, n);
    return;
  }
  pool().run(n, nt, fn, ctx);
}

}  // namespace apc
