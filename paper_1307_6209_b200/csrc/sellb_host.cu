// sellb_host.cu -- host-side staging for the end-to-end path (sellb_spmv_host).
//
// A reference caller hands spmv_sell ordinary NumPy arrays
// (/root/reference/pkg/src/sellkit/spmv.py:105-122): pageable memory.  A DMA
// from pageable memory goes through the driver's own bounce buffer at
// 10-16 GB/s on the B200 boxes (tools/pcie_probe.py), a quarter of what the
// copy engines move from pinned memory (55 GB/s), while one host core copies
// only ~4 GB/s and all 16 together ~53 GB/s.  So the library stages pageable
// vectors itself: a pool of host threads copies each x piece into a pinned
// mirror while the previous piece is on the wire, and copies each finished
// row block of y out of a pinned (mapped) mirror the kernels store into
// while later blocks compute.  Pinned caller vectors need none of this.
#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "sellb_internal.cuh"

namespace sellb {
namespace {

// Fixed pool of worker threads; one parallel copy at a time (the caller
// thread takes part, so a copy uses n_workers + 1 threads).
class CopyPool {
  public:
    static CopyPool& get() {
        static CopyPool* pool = new CopyPool();   // never destroyed: no join at exit
        return *pool;
    }

    void copy(void* dst, const void* src, size_t n) {
        if (n < (size_t(1) << 20) || workers_.empty()) {
            std::memcpy(dst, src, n);
            return;
        }
        std::lock_guard<std::mutex> one(call_mu_);
        const size_t parts = workers_.size() + 1;
        // 4 KiB-aligned part boundaries
        const size_t step = ((n + parts - 1) / parts + 4095) & ~size_t(4095);
        {
            std::lock_guard<std::mutex> lk(mu_);
            dst_ = static_cast<char*>(dst);
            src_ = static_cast<const char*>(src);
            n_ = n;
            step_ = step;
            pending_ = workers_.size();
            ++gen_;
        }
        cv_.notify_all();
        run_part(0);
        std::unique_lock<std::mutex> lk(mu_);
        done_cv_.wait(lk, [&] { return pending_ == 0; });
    }

  private:
    CopyPool() {
        int n = (int)std::thread::hardware_concurrency();
        if (const char* e = getenv("SELLB_HOST_THREADS")) n = atoi(e);
        n = std::max(1, std::min(n, 64));
        for (int i = 1; i < n; ++i) workers_.emplace_back([this, i] { loop(i); });
        for (auto& t : workers_) t.detach();
    }

    void run_part(size_t i) {
        const size_t a = std::min(n_, i * step_), b = std::min(n_, (i + 1) * step_);
        if (b > a) std::memcpy(dst_ + a, src_ + a, b - a);
    }

    void loop(int i) {
        uint64_t seen = 0;
        while (true) {
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return gen_ != seen; });
                seen = gen_;
            }
            run_part((size_t)i);
            std::lock_guard<std::mutex> lk(mu_);
            if (--pending_ == 0) done_cv_.notify_one();
        }
    }

    std::vector<std::thread> workers_;
    std::mutex call_mu_, mu_;
    std::condition_variable cv_, done_cv_;
    char* dst_ = nullptr;
    const char* src_ = nullptr;
    size_t n_ = 0, step_ = 0, pending_ = 0;
    uint64_t gen_ = 0;
};

}  // namespace

void host_parallel_copy(void* dst, const void* src, size_t n) {
    if (n) CopyPool::get().copy(dst, src, n);
}

bool is_pinned(const void* p) {
    cudaPointerAttributes at{};
    const bool pinned = cudaPointerGetAttributes(&at, p) == cudaSuccess &&
                        at.type == cudaMemoryTypeHost;
    cudaGetLastError();   // clear a "not registered" status for pageable memory
    return pinned;
}

int ensure_host_mirror(void** slot, size_t bytes) {
    if (*slot) return 0;
    SELLB_CU(cudaHostAlloc(slot, std::max<size_t>(bytes, 16), cudaHostAllocMapped));
    return 0;
}

}  // namespace sellb
