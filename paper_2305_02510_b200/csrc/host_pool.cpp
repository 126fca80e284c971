// A process-wide pool of host worker threads for the raster expansion (the
// decode of a simulate call's spike words into (step, neuron) events runs per
// chunk while later chunks are on the GPU; spawning threads per chunk cost
// ~0.5 ms per call).  host_parallel(n, f) runs f(0..n-1) on the workers and
// the calling thread and returns when all are done.
#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace snb {

namespace {

class HostPool {
public:
    HostPool() {
        const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
        for (unsigned i = 1; i < hw; ++i) workers_.emplace_back([this] { loop(); });
    }
    ~HostPool() {
        {
            std::lock_guard<std::mutex> g(m_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : workers_) t.join();
    }
    int size() const { return static_cast<int>(workers_.size()) + 1; }
    void run(int n, const std::function<void(int)>& f) {
        std::unique_lock<std::mutex> call(call_m_);  // one job at a time
        {
            std::lock_guard<std::mutex> g(m_);
            job_ = &f;
            n_ = n;
            next_.store(0);
            pending_ = n;
            ++gen_;
        }
        cv_.notify_all();
        work();
        std::unique_lock<std::mutex> g(m_);
        done_cv_.wait(g, [this] { return pending_ == 0; });
        job_ = nullptr;
    }

private:
    void work() {
        for (;;) {
            const int i = next_.fetch_add(1);
            if (i >= n_) return;
            (*job_)(i);
            std::lock_guard<std::mutex> g(m_);
            if (--pending_ == 0) done_cv_.notify_all();
        }
    }
    void loop() {
        uint64_t seen = 0;
        for (;;) {
            {
                std::unique_lock<std::mutex> g(m_);
                cv_.wait(g, [&] { return stop_ || gen_ != seen; });
                if (stop_) return;
                seen = gen_;
            }
            work();
        }
    }
    std::vector<std::thread> workers_;
    std::mutex m_, call_m_;
    std::condition_variable cv_, done_cv_;
    const std::function<void(int)>* job_ = nullptr;
    std::atomic<int> next_{0};
    int n_ = 0, pending_ = 0;
    uint64_t gen_ = 0;
    bool stop_ = false;
};

HostPool& pool() {
    static HostPool p;
    return p;
}

}  // namespace

int host_threads() { return pool().size(); }

void host_parallel(int n, const std::function<void(int)>& f) {
    if (n <= 0) return;
    if (n == 1) {
        f(0);
        return;
    }
    pool().run(n, f);
}

}  // namespace snb
