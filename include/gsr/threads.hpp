// gsr/threads.hpp — the host worker pool of the public API.
//
// Keeps the interface of /root/reference/proj/include/gsr/threads.hpp:17-52
// (ThreadPool(threads), size(), parallel_for(n, fn(begin, end)) over contiguous
// chunks with the caller participating, and the free parallel_for(pool, ...)
// serial fallback for a null pool) so host code written against the reference
// compiles unchanged. The reference ships only the declaration; this is a
// header-only definition for the B200 build's host side (graph validation,
// metrics, file I/O around the C-ABI — the device path never runs on it).
//
// Determinism contract (threads.hpp:14-16): [0, n) is cut into size()
// contiguous chunks that depend only on n and size(); each index is handed to
// exactly one thread, so any row-partitioned loop with a fixed inner order
// gives bit-identical results for every worker count. Kernels must not throw
// (threads.hpp:28-29): an exception escaping fn calls std::terminate.
#pragma once

#include <condition_variable>
#include <cstdint>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "gsr/common.hpp"

namespace gsr {

class ThreadPool {
public:
    // threads ≤ 0 means one per hardware thread; the caller counts as one.
    explicit ThreadPool(int threads) {
        int t = threads > 0 ? threads : static_cast<int>(std::thread::hardware_concurrency());
        if (t < 1) t = 1;
        helpers_.reserve(static_cast<std::size_t>(t - 1));
        for (int id = 1; id < t; ++id) helpers_.emplace_back([this, id] { serve(id); });
    }
    ~ThreadPool() {
        {
            std::lock_guard<std::mutex> g(m_);
            quit_ = true;
        }
        wake_.notify_all();
        for (std::thread& h : helpers_) h.join();
    }
    ThreadPool(const ThreadPool&) = delete;
    ThreadPool& operator=(const ThreadPool&) = delete;

    int size() const { return static_cast<int>(helpers_.size()) + 1; }

    void parallel_for(index_t n, const std::function<void(index_t, index_t)>& fn) {
        if (n <= 0) return;
        const int parts = size();
        if (parts == 1 || n == 1) {
            fn(0, n);
            return;
        }
        {
            std::lock_guard<std::mutex> g(m_);
            job_ = &fn;
            n_ = n;
            outstanding_ = parts - 1;
            ++epoch_;
        }
        wake_.notify_all();
        run_part(0, fn, n);  // the caller takes part 0
        std::unique_lock<std::mutex> lk(m_);
        done_.wait(lk, [this] { return outstanding_ == 0; });
        job_ = nullptr;
    }

private:
    // part p of size() parts: [p·n/parts, (p+1)·n/parts)
    void run_part(int p, const std::function<void(index_t, index_t)>& fn, index_t n) const noexcept {
        const index_t parts = size();
        const index_t b = n * p / parts, e = n * (p + 1) / parts;
        if (b < e) fn(b, e);
    }
    void serve(int id) {
        std::uint64_t seen = 0;
        for (;;) {
            const std::function<void(index_t, index_t)>* fn;
            index_t n;
            {
                std::unique_lock<std::mutex> lk(m_);
                wake_.wait(lk, [&] { return quit_ || epoch_ != seen; });
                if (quit_) return;
                seen = epoch_;
                fn = job_;
                n = n_;
            }
            run_part(id, *fn, n);
            std::lock_guard<std::mutex> g(m_);
            if (--outstanding_ == 0) done_.notify_one();
        }
    }

    std::vector<std::thread> helpers_;
    std::mutex m_;
    std::condition_variable wake_, done_;
    const std::function<void(index_t, index_t)>* job_ = nullptr;
    index_t n_ = 0;
    int outstanding_ = 0;
    std::uint64_t epoch_ = 0;
    bool quit_ = false;
};

// Serial fallback wherever no pool is supplied (threads.hpp:51-52).
inline void parallel_for(ThreadPool* pool, index_t n, const std::function<void(index_t, index_t)>& fn) {
    if (pool) pool->parallel_for(n, fn);
    else if (n > 0) fn(0, n);
}

}  // namespace gsr
