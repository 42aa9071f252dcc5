// host_trig.cpp — see host_trig.h. Built by g++ with -ffp-contract=off.
#include "host_trig.h"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <condition_variable>
#include <cstdlib>
#include <mutex>
#include <thread>
#include <vector>

namespace sdfgi_host {
namespace {

constexpr double kPi = 3.14159265358979323846;  // vec.hpp:9

uint64_t hashU64(uint64_t x) {  // rng.hpp:10-15
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e9b5ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}
uint64_t hashCombine(uint64_t a, uint64_t b) {  // rng.hpp:17
    return hashU64(a ^ (b + 0x9e3779b97f4a7c15ull + (a << 6) + (a >> 2)));
}
struct Rng {  // rng.hpp:22-48
    uint64_t s;
    explicit Rng(uint64_t key) : s(hashU64(key)) {}
    uint64_t next() {
        s += 0x9e3779b97f4a7c15ull;
        uint64_t z = s;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e9b5ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        return z ^ (z >> 31);
    }
    double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
};

// A small persistent pool: per-pass work (one quaternion per probe, ~16k-500k
// probes) is too short to pay a thread spawn per call.
class Pool {
public:
    Pool() {
        unsigned hw = std::thread::hardware_concurrency();
        const char* env = std::getenv("SDFGI_HOST_THREADS");
        int n = env ? std::atoi(env) : static_cast<int>(std::min(hw ? hw : 1u, 16u));
        n = std::max(1, n);
        for (int i = 1; i < n; ++i) workers_.emplace_back([this] { loop(); });
        nThreads_ = n;
    }
    ~Pool() {
        {
            std::lock_guard<std::mutex> g(m_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : workers_) t.join();
    }
    int threads() const { return nThreads_; }
    void run(long long n, long long grain, const std::function<void(long long, long long)>& body) {
        if (n <= 0) return;
        grain = std::max(1LL, grain);
        if (nThreads_ == 1 || n <= grain) {
            body(0, n);
            return;
        }
        std::lock_guard<std::mutex> one(runM_);  // one job at a time
        {
            std::lock_guard<std::mutex> g(m_);
            body_ = &body;
            n_ = n;
            grain_ = grain;
            next_.store(0);
            pending_ = static_cast<int>(workers_.size());
            ++gen_;
        }
        cv_.notify_all();
        work();
        std::unique_lock<std::mutex> g(m_);
        done_.wait(g, [this] { return pending_ == 0; });
        body_ = nullptr;
    }

private:
    void work() {
        for (;;) {
            long long b = next_.fetch_add(grain_);
            if (b >= n_) break;
            (*body_)(b, std::min(n_, b + grain_));
        }
    }
    void loop() {
        unsigned long long seen = 0;
        for (;;) {
            {
                std::unique_lock<std::mutex> g(m_);
                cv_.wait(g, [&] { return stop_ || gen_ != seen; });
                if (stop_) return;
                seen = gen_;
            }
            work();
            {
                std::lock_guard<std::mutex> g(m_);
                if (--pending_ == 0) done_.notify_one();
            }
        }
    }
    std::vector<std::thread> workers_;
    int nThreads_ = 1;
    std::mutex m_, runM_;
    std::condition_variable cv_, done_;
    bool stop_ = false;
    unsigned long long gen_ = 0;
    const std::function<void(long long, long long)>* body_ = nullptr;
    long long n_ = 0, grain_ = 1;
    std::atomic<long long> next_{0};
    int pending_ = 0;
};

Pool& pool() {
    static Pool p;
    return p;
}

}  // namespace

void parallelFor(long long n, long long grain, const std::function<void(long long, long long)>& body) {
    pool().run(n, grain, body);
}

uint64_t probeKey(int cascadeLevel, int index) {
    return hashCombine(static_cast<uint64_t>(cascadeLevel) + 0x9e1du, static_cast<uint64_t>(index));
}

void fibTable(int n, double* out) {
    // sphericalFibonacci(i, n), sampling.hpp:11-17
    const double goldenAngle = kPi * (3.0 - std::sqrt(5.0));
    for (int i = 0; i < n; ++i) {
        double z = 1.0 - (2.0 * i + 1.0) / n;
        double r = std::sqrt(std::max(0.0, 1.0 - z * z));
        double phi = goldenAngle * i;
        out[3 * i] = r * std::cos(phi);
        out[3 * i + 1] = r * std::sin(phi);
        out[3 * i + 2] = z;
    }
}

void probeQuats(uint64_t seed, int frame, bool rotatePerFrame, const uint64_t* keys, int n, double* out) {
    // sampleDirections' stream, sampling.hpp:25-26: Rng(seed, frame | 0xf1b0, probeKey, 0x5df6d1)
    const uint64_t f = rotatePerFrame ? static_cast<uint64_t>(static_cast<int64_t>(frame)) : 0xf1b0ull;
    const uint64_t k0 = hashCombine(seed, f);
    // ~0.2 us per probe (four libm calls): 256-probe chunks spread a C2 pass
    // (16k probes) over every pool thread
    parallelFor(n, 256, [&](long long b, long long e) {
        for (long long i = b; i < e; ++i) {
            Rng rng(hashCombine(hashCombine(k0, keys[i]), 0x5df6d1ull));
            // randomRotation, rng.hpp:72-78
            double u1 = rng.uniform(), u2 = rng.uniform(), u3 = rng.uniform();
            double a = std::sqrt(1.0 - u1), bb = std::sqrt(u1);
            double* q = out + 4 * i;
            q[0] = a * std::sin(2 * kPi * u2);
            q[1] = a * std::cos(2 * kPi * u2);
            q[2] = bb * std::sin(2 * kPi * u3);
            q[3] = bb * std::cos(2 * kPi * u3);
        }
    });
}

void contactLocal(uint64_t seed, int w, int h, int samples, double* out) {
    const uint64_t k0 = hashCombine(seed, 0xc0417ffull);
    const long long np = static_cast<long long>(w) * h;
    parallelFor(np, 4096, [&](long long b, long long e) {
        for (long long pix = b; pix < e; ++pix) {
            // Rng(seed, 0xc0417ff, y * width + x), shading.hpp:451; pix = y * w + x
            Rng rng(hashCombine(k0, static_cast<uint64_t>(pix)));
            double* o = out + 2 * pix * samples;
            for (int s = 0; s < samples; ++s) {
                // cosineHemisphereDir, rng.hpp:58-63
                double u1 = rng.uniform();
                double u2 = rng.uniform();
                double r = std::sqrt(u1);
                double phi = 2.0 * kPi * u2;
                o[2 * s] = r * std::cos(phi);
                o[2 * s + 1] = r * std::sin(phi);
            }
        }
    });
}

double tanHalf(double fovYDeg) { return std::tan(fovYDeg * kPi / 360.0); }

}  // namespace sdfgi_host
