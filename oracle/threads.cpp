// TEST INFRASTRUCTURE ONLY (CPU oracle). See threads.hpp.
#include "threads.hpp"

namespace gsro {

ThreadPool::ThreadPool(int threads) {
    if (threads < 1) threads = 1;
    tasks_.resize(static_cast<size_t>(threads));
    for (int i = 1; i < threads; ++i) workers_.emplace_back([this, i] { worker_loop(i); });
}

ThreadPool::~ThreadPool() {
    {
        std::lock_guard<std::mutex> lk(mu_);
        stop_ = true;
        ++generation_;
    }
    cv_work_.notify_all();
    for (auto& t : workers_) t.join();
}

void ThreadPool::worker_loop(int id) {
    std::uint64_t seen = 0;
    for (;;) {
        Task task;
        {
            std::unique_lock<std::mutex> lk(mu_);
            cv_work_.wait(lk, [&] { return generation_ != seen; });
            seen = generation_;
            if (stop_) return;
            task = tasks_[static_cast<size_t>(id)];
        }
        if (task.fn && task.begin < task.end) (*task.fn)(task.begin, task.end);
        {
            std::lock_guard<std::mutex> lk(mu_);
            if (--pending_ == 0) cv_done_.notify_one();
        }
    }
}

void ThreadPool::parallel_for(index_t n, const std::function<void(index_t, index_t)>& fn) {
    if (n <= 0) return;
    const int p = size();
    if (p == 1 || n < 2) {
        fn(0, n);
        return;
    }
    const index_t chunk = (n + p - 1) / p;
    {
        std::lock_guard<std::mutex> lk(mu_);
        for (int i = 0; i < p; ++i) {
            index_t b = chunk * i, e = b + chunk;
            if (b > n) b = n;
            if (e > n) e = n;
            tasks_[static_cast<size_t>(i)] = Task{&fn, b, e};
        }
        pending_ = p - 1;
        ++generation_;
    }
    cv_work_.notify_all();
    const Task mine = tasks_[0];
    if (mine.begin < mine.end) fn(mine.begin, mine.end);
    std::unique_lock<std::mutex> lk(mu_);
    cv_done_.wait(lk, [&] { return pending_ == 0; });
}

void parallel_for(ThreadPool* pool, index_t n, const std::function<void(index_t, index_t)>& fn) {
    if (pool) pool->parallel_for(n, fn);
    else if (n > 0) fn(0, n);
}

}  // namespace gsro
