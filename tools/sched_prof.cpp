// Host cost of IDAG generation per WaveSim step, without Python or CUDA: the
// scheduler alone (sched.cpp) with a counting sink, G devices, optionally the
// multi-process rank filter.  Build and run (CEL_SCHED_MEMO=0: no memo):
//   g++ -O2 -std=c++17 -Ipaper_2503_10516_b200/csrc tools/sched_prof.cpp paper_2503_10516_b200/csrc/sched.cpp
//       paper_2503_10516_b200/csrc/sched_memo.cpp -o /tmp/sched_prof && /tmp/sched_prof 8 [rank]
//   /tmp/sched_prof rsim 4 [rank] [T]      (RSim rows, W = 84,000)
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <deque>
#include <mutex>
#include <thread>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "sched.hpp"

using namespace cel;

struct Count : InstrSink {
    uint64_t n = 0;
    bool copy = getenv("CEL_PROF_COPY") != nullptr;
    void on_instr(const Instr& ins) override {
        ++n;
        if (copy) {
            Instr x = ins;                           // the hand-off's copy alone
            asm volatile("" ::"r"(&x) : "memory");
        }
    }
};

// the executor's hand-off without CUDA: copy into a mutex-guarded deque that
// a consumer thread drains (CEL_PROF_QUEUE=1)
struct QueueSink : InstrSink {
    std::mutex m;
    std::condition_variable cv;
    std::deque<Instr> q;
    std::vector<Instr> pool;                      // CEL_PROF_POOL=1: the executor's recycling
    bool pooled = getenv("CEL_PROF_POOL") != nullptr;
    bool stop = false, sleeping = false;
    bool batched = getenv("CEL_PROF_QUEUE")[0] == '2';
    std::atomic<size_t> size{0};
    uint64_t n = 0;
    std::thread th;
    QueueSink() {
        th = std::thread([this] {
            std::deque<Instr> batch;
            for (;;) {
                {
                    std::unique_lock<std::mutex> l(m);
                    if (q.empty()) {
                        l.unlock();
                        for (int i = 0; i < 20000 && size.load(std::memory_order_acquire) == 0 && !stop; ++i) {
                        }
                        l.lock();
                        while (q.empty() && !stop) {
                            sleeping = true;
                            cv.wait(l);
                            sleeping = false;
                        }
                        if (q.empty() && stop) return;
                    }
                    if (batched) {
                        batch.swap(q);
                    } else {
                        batch.push_back(std::move(q.front()));
                        q.pop_front();
                    }
                    size.store(q.size(), std::memory_order_release);
                }
                while (!batch.empty()) {
                    Instr x = std::move(batch.front());
                    batch.pop_front();
                    ++n;
                    if (pooled) {
                        std::lock_guard<std::mutex> g(m);
                        if (pool.size() < 4096) pool.push_back(std::move(x));
                    }
                }
            }
        });
    }
    ~QueueSink() {
        {
            std::lock_guard<std::mutex> g(m);
            stop = true;
        }
        cv.notify_one();
        th.join();
    }
    void on_instr(const Instr& ins) override {
        bool wake;
        Instr x;
        if (pooled) {
            std::lock_guard<std::mutex> g(m);
            if (!pool.empty()) {
                x = std::move(pool.back());
                pool.pop_back();
            }
        }
        x = ins;
        {
            std::lock_guard<std::mutex> g(m);
            q.push_back(std::move(x));
            size.store(q.size(), std::memory_order_release);
            wake = sleeping;
        }
        if (wake) cv.notify_one();
    }
};

static TaskDesc fill(int64_t n, uint32_t buf) {
    TaskDesc d;
    d.dims = 2;
    const int64_t lo[3] = {0, 0, 0}, hi[3] = {n, n, 1};
    d.range = Box::make(lo, hi);
    d.kernel = 0;
    Access a;
    a.buf = buf;
    a.mode = MODE_WRITE;
    d.acc.push_back(a);
    return d;
}

static TaskDesc wave(int64_t n, int k) {
    TaskDesc d;
    d.dims = 2;
    const int64_t lo[3] = {0, 0, 0}, hi[3] = {n, n, 1};
    d.range = Box::make(lo, hi);
    d.kernel = 3;
    const uint32_t u = k % 2 == 0 ? 0 : 1, up = 1 - u;
    Access r;
    r.buf = u;
    r.mode = MODE_READ;
    r.map.kind = MapKind::Neighborhood;
    r.map.border[0] = r.map.border[1] = 1;
    Access w;
    w.buf = up;
    w.mode = MODE_READ_WRITE;
    d.acc.push_back(r);
    d.acc.push_back(w);
    return d;
}

// the hand-off as a ring of reused slots (CEL_PROF_QUEUE=3): the producer
// copy-assigns into a free slot under the lock (vectors keep their capacity,
// nothing is allocated per instruction), the consumer reads its slot in place
struct RingSink : InstrSink {
    static constexpr size_t kCap = 16384;
    std::vector<Instr> ring = std::vector<Instr>(kCap);
    size_t head = 0, tail = 0;
    std::mutex m;
    std::condition_variable cv, full;
    bool stop = false, sleeping = false;
    std::atomic<size_t> size{0};
    uint64_t n = 0;
    std::thread th;
    RingSink() {
        th = std::thread([this] {
            for (;;) {
                size_t h;
                {
                    std::unique_lock<std::mutex> l(m);
                    if (head == tail) {
                        l.unlock();
                        for (int i = 0; i < 20000 && size.load(std::memory_order_acquire) == 0 && !stop; ++i) {
                        }
                        l.lock();
                        while (head == tail && !stop) {
                            sleeping = true;
                            cv.wait(l);
                            sleeping = false;
                        }
                        if (head == tail && stop) return;
                    }
                    h = head;
                }
                const Instr& x = ring[h];
                asm volatile("" ::"r"(&x), "r"(x.deps.size()) : "memory");
                ++n;
                {
                    std::lock_guard<std::mutex> g(m);
                    head = (h + 1) % kCap;
                    size.store((tail + kCap - head) % kCap, std::memory_order_release);
                }
                full.notify_one();
            }
        });
    }
    ~RingSink() {
        {
            std::lock_guard<std::mutex> g(m);
            stop = true;
        }
        cv.notify_one();
        th.join();
    }
    void on_instr(const Instr& ins) override {
        bool wake;
        {
            std::unique_lock<std::mutex> l(m);
            while ((tail + 1) % kCap == head) full.wait(l);
            ring[tail] = ins;
            tail = (tail + 1) % kCap;
            size.store((tail + kCap - head) % kCap, std::memory_order_release);
            wake = sleeping;
        }
        if (wake) cv.notify_one();
    }
};

// RSim row t (programs.rsim_row): read rows [0,t) (fixed), write row t (remap kernel dim 0 -> dim 1)
static TaskDesc rsim_row(int64_t W, int64_t t) {
    TaskDesc d;
    d.dims = 1;
    const int64_t lo[3] = {0, 0, 0}, hi[3] = {W, 1, 1};
    d.range = Box::make(lo, hi);
    d.kernel = 7;
    Access r;
    r.buf = 0;
    r.mode = MODE_READ;
    r.map.kind = MapKind::Fixed;
    const int64_t flo[3] = {0, 0, 0}, fhi[3] = {t, W, 1};
    r.map.fixed = Box::make(flo, fhi);
    Access w;
    w.buf = 0;
    w.mode = MODE_WRITE;
    w.map.kind = MapKind::Remap;
    w.map.fixed.lo[0] = t;
    w.map.fixed.hi[0] = t + 1;
    w.map.fixed.hi[2] = 1;
    w.map.from_kernel_dim[1] = 0;
    d.acc.push_back(r);
    d.acc.push_back(w);
    return d;
}

static int rsim_main(int G, int rank, int T) {
    const int64_t W = 84000;
    Count count;
    const char* qe = getenv("CEL_PROF_QUEUE");
    QueueSink* qs = qe && qe[0] != '3' ? new QueueSink : nullptr;
    RingSink* rs = qe && qe[0] == '3' ? new RingSink : nullptr;
    InstrSink* sk = qs ? static_cast<InstrSink*>(qs) : rs ? static_cast<InstrSink*>(rs) : static_cast<InstrSink*>(&count);
    struct { uint64_t n = 0; } sink;
    Scheduler s(G, 1, 4, true, sk, nullptr);
    if (rank >= 0) s.set_rank_filter(rank, G);
    const int64_t ext[3] = {T, W, 1};
    uint32_t b0;
    s.buffer_create(2, ext, 4, false, &b0);
    std::string err;
    uint64_t tid;
    TaskDesc f = rsim_row(W, 0);
    f.acc.erase(f.acc.begin());
    f.kernel = 0;
    s.task_submit(f, &tid, &err);
    const auto t0 = std::chrono::steady_clock::now();
    for (int t = 1; t < T; ++t) s.task_submit(rsim_row(W, t), &tid, &err);
    s.wait();
    const double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    sink.n = count.n;
    printf("rsim G=%d rank=%d T=%d%s: %.2f us/row, %.1f instructions/row\n", G, rank, T,
           qs ? " (queue sink)" : rs ? " (ring sink)" : "",
           dt / (T - 1) * 1e6, double(sink.n) / (T - 1));
    s.shutdown();
    delete qs;
    delete rs;
    return 0;
}

int main(int argc, char** argv) {
    if (argc > 1 && std::string(argv[1]) == "rsim")
        return rsim_main(argc > 2 ? atoi(argv[2]) : 4, argc > 3 ? atoi(argv[3]) : -1, argc > 4 ? atoi(argv[4]) : 1024);
    const int G = argc > 1 ? atoi(argv[1]) : 8;
    const int rank = argc > 2 ? atoi(argv[2]) : -1;
    const int K = argc > 3 ? atoi(argv[3]) : 20000;
    const int64_t n = 16384;
    Count sink;
    Scheduler s(G, 1, 4, true, &sink, nullptr);
    if (rank >= 0) s.set_rank_filter(rank, G);
    const int64_t ext[3] = {n, n, 1};
    uint32_t b0, b1;
    s.buffer_create(2, ext, 4, false, &b0);
    s.buffer_create(2, ext, 4, false, &b1);
    std::string err;
    uint64_t tid;
    s.task_submit(fill(n, 0), &tid, &err);
    s.task_submit(fill(n, 1), &tid, &err);
    const TaskDesc w[2] = {wave(n, 0), wave(n, 1)};
    for (int k = 0; k < 200; ++k) s.task_submit(w[k % 2], &tid, &err);
    s.wait();
    const uint64_t n0 = sink.n;
    const auto t0 = std::chrono::steady_clock::now();
    for (int k = 0; k < K; ++k) s.task_submit(w[k % 2], &tid, &err);
    s.wait();
    const double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    printf("G=%d rank=%d: %.2f us/step, %.1f instructions/step, memo %llu hits %llu misses\n", G, rank, dt / K * 1e6,
           double(sink.n - n0) / K, (unsigned long long)s.memo_hits(), (unsigned long long)s.memo_misses());
    s.shutdown();
    return 0;
}
