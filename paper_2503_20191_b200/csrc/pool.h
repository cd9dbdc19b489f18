// Persistent host worker pool for the engine's batch staging (generation,
// packing, arena copies).  Workers are created once and reused, so a call does
// not pay thread creation, and thread_local scratch (generator and packer
// buffers) keeps its capacity across batches.
#pragma once
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace maya {

class WorkerPool {
 public:
  // Pool 0 stages batches (generation + packing), pool 1 assembles arenas, so
  // a pipeline can assemble batch q while it generates batch q+1 (api.py
  // GenPipeline).  Each pool runs one parallel region at a time.
  static WorkerPool &get(int id = 0) {
    static WorkerPool p[2];
    return p[id & 1];
  }
  // Run `work` on nt threads (the caller is one of them) and wait for all.
  void run(int nt, const std::function<void()> &work) {
    if (nt <= 1) {
      work();
      return;
    }
    std::unique_lock<std::mutex> call(call_mu_);   // one parallel region at a time
    {
      std::unique_lock<std::mutex> lk(mu_);
      while ((int)threads_.size() < nt - 1) threads_.emplace_back([this] { loop(); });
      work_ = &work;
      want_ = nt - 1;
      taken_ = 0;
      done_ = 0;
      gen_++;
    }
    cv_.notify_all();
    work();
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [this] { return done_ == want_; });
    work_ = nullptr;
  }
  ~WorkerPool() {
    {
      std::unique_lock<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto &t : threads_) t.join();
  }

 private:
  void loop() {
    unsigned long seen = 0;
    for (;;) {
      const std::function<void()> *w;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || (gen_ != seen && taken_ < want_); });
        if (stop_) return;
        seen = gen_;
        taken_++;
        w = work_;
      }
      (*w)();
      {
        std::unique_lock<std::mutex> lk(mu_);
        done_++;
      }
      done_cv_.notify_one();
    }
  }
  std::mutex call_mu_, mu_;
  std::condition_variable cv_, done_cv_;
  std::vector<std::thread> threads_;
  const std::function<void()> *work_ = nullptr;
  int want_ = 0, taken_ = 0, done_ = 0;
  unsigned long gen_ = 0;
  bool stop_ = false;
};

}  // namespace maya
