// pool.hpp -- one persistent pool of host threads for the library's parallel
// loops (plan load, stage construction, lowering, front and back ends).
//
// Every parallel loop used to start and join its own std::threads; a
// verify_plan on a large plan runs dozens of such loops, and on a 16-core host
// the thread start/join alone was milliseconds per loop. The pool keeps its
// workers parked on a condition variable between jobs. One job runs at a time;
// a loop started while another job holds the pool (a nested loop, or a second
// host thread) gets `false` back and starts its own threads as before.
#pragma once

#include <unistd.h>

#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <cstdlib>
#include <exception>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace pqw {

class HostPool {
 public:
  // body(tid) for tid in [0, nt), tid 0 on the calling thread; false (nothing
  // run) when the pool is busy.
  bool run(unsigned nt, const std::function<void(unsigned)>& body) {
    std::unique_lock<std::mutex> job(job_mu_, std::try_to_lock);
    if (!job.owns_lock()) return false;
    {
      std::lock_guard<std::mutex> g(mu_);
      while (n_workers_ + 1 < nt) {
        const unsigned id = ++n_workers_;
        std::thread([this, id, g0 = gen_] { loop(id, g0); }).detach();
      }
      body_ = &body;
      want_ = nt;
      pending_ = nt - 1;
      ++gen_;
    }
    cv_.notify_all();
    std::exception_ptr err;
    try {
      body(0);
    } catch (...) {  // the workers still use the caller's frame: wait for them first
      err = std::current_exception();
    }
    {
      std::unique_lock<std::mutex> g(mu_);
      done_.wait(g, [&] { return pending_ == 0; });
      body_ = nullptr;
    }
    if (err) std::rethrow_exception(err);
    return true;
  }

 private:
  void loop(unsigned id, uint64_t seen) {
    for (;;) {
      const std::function<void(unsigned)>* b;
      {
        std::unique_lock<std::mutex> g(mu_);
        cv_.wait(g, [&] { return gen_ != seen; });
        seen = gen_;
        if (id >= want_) continue;  // not part of this job
        b = body_;
      }
      (*b)(id);
      std::lock_guard<std::mutex> g(mu_);
      if (--pending_ == 0) done_.notify_one();
    }
  }

  std::mutex job_mu_;  // held for the duration of one job
  std::mutex mu_;
  std::condition_variable cv_, done_;
  const std::function<void(unsigned)>* body_ = nullptr;
  unsigned n_workers_ = 0, want_ = 0, pending_ = 0;
  uint64_t gen_ = 0;
};

// The process-wide pool (never destroyed: its detached workers stay parked
// until the process exits). A forked child has none of the parent's workers
// (and may have inherited a held lock), so a process whose pid differs from
// the pool's creator gets a pool of its own.
inline HostPool& host_pool() {
  static std::atomic<HostPool*> pool{nullptr};
  static std::atomic<pid_t> owner{0};
  const pid_t me = getpid();
  HostPool* p = pool.load(std::memory_order_acquire);
  if (p == nullptr || owner.load(std::memory_order_acquire) != me) {
    p = new HostPool();  // a replaced pool is left alone (its users may still hold it)
    pool.store(p, std::memory_order_release);
    owner.store(me, std::memory_order_release);
  }
  return *p;
}

// body(tid) on nt threads: through the pool, or on fresh threads when it is busy.
inline void run_on_threads(unsigned nt, const std::function<void(unsigned)>& body) {
  if (nt <= 1) {
    body(0);
    return;
  }
  static const bool no_pool = std::getenv("PQW_NO_POOL") != nullptr;  // A/B switch
  if (!no_pool && host_pool().run(nt, body)) return;
  std::vector<std::thread> extra;
  for (unsigned t = 1; t < nt; ++t) extra.emplace_back(body, t);
  body(0);
  for (auto& t : extra) t.join();
}

}  // namespace pqw
