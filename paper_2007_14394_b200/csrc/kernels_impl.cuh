#include <type_traits>
// kernels_impl.cuh — kernel bodies, included once per precision translation unit.
#pragma once

#include "kernels.cuh"

namespace sdfgi_dev {

constexpr unsigned kFull = 0xffffffffu;

// Streaming (evict-first) stores and loads of the per-ray wavefront records
// (hit records, radiance, visibility, shadow rays: written once, read once), so
// the hundreds of MB they stream through L2 per pass do not evict the candidate
// grid and the primitive records the tracing kernels re-read.
template <typename T>
__device__ __forceinline__ void stStream(T* dst, const T& v) {
    static_assert(sizeof(T) % 16 == 0 && alignof(T) >= 16, "16-byte records");
    const int4* s = reinterpret_cast<const int4*>(&v);
    int4* d = reinterpret_cast<int4*>(dst);
#pragma unroll
    for (int i = 0; i < static_cast<int>(sizeof(T) / 16); ++i) __stcs(d + i, s[i]);
}
template <typename T>
__device__ __forceinline__ T ldStream(const T* src) {
    static_assert(sizeof(T) % 16 == 0 && alignof(T) >= 16, "16-byte records");
    T v;
    const int4* s = reinterpret_cast<const int4*>(src);
    int4* d = reinterpret_cast<int4*>(&v);
#pragma unroll
    for (int i = 0; i < static_cast<int>(sizeof(T) / 16); ++i) d[i] = __ldcs(s + i);
    return v;
}

__device__ __forceinline__ int cascadeOf(const ProbeCommon& pc, int gp) {
    int ci = 0;
    for (int k = 1; k < pc.nCas; ++k)
        if (gp >= pc.cas[k].base) ci = k;
    return ci;
}

__device__ __forceinline__ void flushCounters(const Counters& c, unsigned long long* out) {
    // warp reduce then one atomic per warp per counter (all 32 lanes must call)
    unsigned long long v[14] = {c.q,     c.cv,    c.cs,    c.pe,    c.steps, c.sphere, c.shadow,
                                c.vis,   c.ek[0], c.ek[1], c.ek[2], c.ek[3], c.ek[4],  c.ek[5]};
#pragma unroll
    for (int i = 0; i < 14; ++i) {
        unsigned long long x = v[i];
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(kFull, x, o);
        if ((threadIdx.x & 31) == 0 && x) atomicAdd(out + i, x);
    }
}

// Work fetch for persistent, self-refilling lanes: every idle, not-yet-exhausted
// lane of the warp gets the next item id. The warp takes items from a private
// chunk of kFetchChunk consecutive ids (warp-uniform `chunk` = next, end), and only
// grabs a new chunk from the global cursor with one atomic when the chunk runs
// dry — far fewer atomics on the shared cursor line, and a warp's rays stay
// consecutive (coherent). Must be called by all 32 lanes. Returns true for lanes
// that got an item.
#ifndef SDFGI_FETCH_CHUNK
#define SDFGI_FETCH_CHUNK 32  // C2 pass 0: 32 -> 64 -> 128 = FP64 10.4 / 10.5 / 10.9 ms
#endif
constexpr unsigned long long kFetchChunk = SDFGI_FETCH_CHUNK;
// The cell record of a march point is loaded as soon as its cell is known, so
// its DRAM latency (the tracing kernels' top stall on the 240M-cell grid) runs
// under the escape / parking / settle logic before the query needs it. K1 in
// both precisions, K2 in FP64 (FP32's K2 keeps its per-lane cell cache):
// C2 FP64 24.30 -> 23.86 ms, FP32 15.72 -> 15.63 ms.
#ifndef SDFGI_HOIST_CELL_LOAD
#define SDFGI_HOIST_CELL_LOAD 1
#endif
#ifndef SDFGI_HOIST_CELL_LOAD2
#define SDFGI_HOIST_CELL_LOAD2 1
#endif
#ifndef SDFGI_PREFETCH_CHUNK
#define SDFGI_PREFETCH_CHUNK 1
#endif
#ifndef SDFGI_CELL_CACHE64
#define SDFGI_CELL_CACHE64 0
#endif
// K1/K2 per-lane cell-record cache (CellCache) in FP64 too
template <typename R> __device__ __forceinline__ bool useCellCache() { return sizeof(R) == 4 || SDFGI_CELL_CACHE64 != 0; }
static_assert(kFetchChunk >= 32, "one fresh chunk must cover a whole warp's request");
// Item positions: 32-bit in the FP32 kernels (two registers fewer: FP32 C2 step
// 16.08 -> 15.92 ms); 64-bit in FP64, where ptxas's allocation came out worse
// (24.43 -> 25.12 ms).
template <typename I>
struct WarpChunkT {
    I next = 0, end = 0;
};
template <typename R>
using WarpChunkFor = WarpChunkT<typename std::conditional<sizeof(R) == 4, unsigned, unsigned long long>::type>;
// prefetch (optional): the records of a freshly taken chunk (item i at prefetch +
// i * prefetchBytes) are pulled into L2 by the warp's lanes, one each, so the
// chunk's later refills do not wait on DRAM.
template <typename I>
__device__ __forceinline__ bool fetchItem(unsigned long long* cursor, unsigned long long total, bool active,
                                          bool& exhausted, unsigned long long& item, WarpChunkT<I>& chunk,
                                          const void* prefetch = nullptr, int prefetchBytes = 0) {
    const unsigned lane = threadIdx.x & 31;
    const unsigned need = __ballot_sync(kFull, !active && !exhausted);
    if (need == 0) return false;
    const unsigned n = __popc(need), rank = __popc(need & ((1u << lane) - 1u));
    const I avail = chunk.end - chunk.next;
    unsigned long long it;
    if (avail >= n) {
        it = chunk.next + rank;
        chunk.next += n;
    } else {  // the old chunk's remainder first, then a fresh chunk
        const int leader = __ffs(need) - 1;
        unsigned long long base = 0;
        if (static_cast<int>(lane) == leader) base = atomicAdd(cursor, kFetchChunk);
        base = __shfl_sync(kFull, base, leader);
        if (SDFGI_PREFETCH_CHUNK && prefetch && base + lane < total)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(static_cast<const char*>(prefetch) +
                                                        (base + lane) * static_cast<unsigned long long>(prefetchBytes)));
        it = rank < avail ? static_cast<unsigned long long>(chunk.next) + rank : base + (rank - avail);
        // (32-bit positions: a cursor past 2^32 only happens once the items ran out)
        const unsigned long long b =
            sizeof(I) == 4 ? (base < 0xFFFFFF00ull ? base : 0xFFFFFF00ull) : base;
        chunk.next = static_cast<I>(b + (n - avail));
        chunk.end = static_cast<I>(b + kFetchChunk);
    }
    if (active || exhausted) return false;
    item = it;
    if (item >= total) {
        exhausted = true;
        return false;
    }
    return true;
}

// ------------------------------------------------------------ (d) relocation
// updateProbePositions, probe_volume.hpp:99-143, one 8-lane group per probe of one
// cascade (kRelocLanes probes per 128-thread block): the six sceneGradient
// queries of a descent step run on lanes 0-5 of the group at once, so a step
// costs two query latencies instead of seven. Every lane of the group repeats the
// step's arithmetic on the same values (identical results); lane 0 runs the
// remaining queries and writes the probe.
constexpr int kRelocGroup = 8;
constexpr int kRelocLanes = 128 / kRelocGroup;
template <bool ST>
__global__ void __launch_bounds__(128) k_relocate(RelocParams P) {
    const CascadeDev& c = P.pc.cas[P.cascade];
    const int n = c.res[0] * c.res[1] * c.res[2];
    const int i = blockIdx.x * kRelocLanes + threadIdx.x / kRelocGroup;
    const int sub = threadIdx.x % kRelocGroup;
    const bool valid = i < n;
    Counters cnt;
    cnt.zero();
    int relocated = 0, rejected = 0, dead = 0;
    const int gp = c.base + (valid ? i : 0);
    const ProbesView& pv = P.pc.probes;
    const SceneView<double>& s = P.scene;
    const double inf = INFINITY;
    V3<double> pos = mk(0.0, 0.0, 0.0), rest = pos, prev = pos;
    if (valid) {
        prev = mk(pv.pos[3 * gp], pv.pos[3 * gp + 1], pv.pos[3 * gp + 2]);
        rest = mk(pv.rest[3 * gp], pv.rest[3 * gp + 1], pv.rest[3 * gp + 2]);
        pos = rest;
    }
    double d = 0;
    if (valid && sub == 0) d = query<double, ST>(s, pos, inf, nullptr, &cnt);
    d = __shfl_sync(kFull, d, 0, kRelocGroup);
    const bool descend = valid && d < P.th1;
    double budget = 0.5 * c.spacing;
    const double h = P.gradStep;
    for (int step = 0; step < P.maxSteps; ++step) {
        const bool go = descend && d < P.th1 && budget > 0;
        if (!__any_sync(kFull, go)) break;
        // sceneGradient, scene.hpp:360-371: lane k queries axis k / 2, +h for even k
        double qv = 0;
        if (go && sub < 6) {
            const int ax = sub >> 1;
            const double off = (sub & 1) ? -h : h;
            const V3<double> q = mk(ax == 0 ? pos.x + off : pos.x, ax == 1 ? pos.y + off : pos.y,
                                    ax == 2 ? pos.z + off : pos.z);  // (pos.x - h as pos.x + (-h): exact)
            qv = query<double, ST>(s, q, inf, nullptr, &cnt);
        }
        double v[6];
#pragma unroll
        for (int k = 0; k < 6; ++k) v[k] = __shfl_sync(kFull, qv, k, kRelocGroup);
        double nd = 0;
        if (go) {
            const V3<double> g = mk(v[0] - v[1], v[2] - v[3], v[4] - v[5]);
            const double gn = length(g);
            const V3<double> dir = (gn < 1e-6 * 2 * h) ? mk(1.0, 0.0, 0.0) : g / gn;
            const double want = smin((P.th1 - d) * 1.25, budget);
            pos = pos + dir * want;
            budget -= want;
            if (sub == 0) nd = query<double, ST>(s, pos, inf, nullptr, &cnt);
        }
        nd = __shfl_sync(kFull, nd, 0, kRelocGroup);
        if (go) d = nd;
    }
    if (valid && sub == 0) {
        bool alive = true;
        if (descend) {
            alive = d >= P.th1;
            if (alive && length(pos - rest) > 1e-12) ++relocated;
        }
        pv.last[3 * gp] = prev.x;
        pv.last[3 * gp + 1] = prev.y;
        pv.last[3 * gp + 2] = prev.z;
        pv.clear[gp] = d;  // query(pos, inf): the last query ran at the final position
        pv.pos[3 * gp] = pos.x;
        pv.pos[3 * gp + 1] = pos.y;
        pv.pos[3 * gp + 2] = pos.z;
        if (!alive) {
            ++dead;
            pv.alive[gp] = 0;
        } else {
            pv.alive[gp] = 1;
            bool hadHistory = pv.lastFrame[gp] >= 0 && !pv.reject[gp];
            if (length(pos - prev) > P.th2) {
                pv.reject[gp] = 1;
                if (hadHistory) ++rejected;
            }
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        relocated += __shfl_xor_sync(kFull, relocated, o);
        rejected += __shfl_xor_sync(kFull, rejected, o);
        dead += __shfl_xor_sync(kFull, dead, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (relocated) atomicAdd(P.report + 0, relocated);
        if (rejected) atomicAdd(P.report + 1, rejected);
        if (dead) atomicAdd(P.report + 2, dead);
    }
    if (ST) flushCounters(cnt, P.stats);
}

// ---------------------------------------------------------------- K0 setup
// Ray count (probe_update.hpp:173; dead probes are skipped, pipeline.hpp:141) and the
// sampleDirections rotation of every probe of the batch.
template <typename R>
__global__ void __launch_bounds__(128) k_ray_setup(WaveParams<R> P) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= P.nCand) return;
    const int g = P.cand ? P.cand[s] : s;
    const ProbesView& pv = P.pc.probes;
    int n = 0;
    if (pv.alive[g] || P.debug) {  // debug traces dead probes too (per-ray parity)
        n = pv.reject[g] ? 2 * P.nRaysFull : P.nRaysFull;
        // randomRotation's matrix (rng.hpp:79-89) from the host-libm quaternion
        const double* q = P.quat + 4 * static_cast<size_t>(s);
        quatToRotation(q[0], q[1], q[2], q[3], P.rot + 9 * static_cast<size_t>(s));
    }
    P.rayCount[s] = n;
}

// Exclusive prefix sum of the ray counts in one CTA (chunked per thread).
template <typename R>
__global__ void __launch_bounds__(kScanThreads) k_ray_scan(WaveParams<R> P) {
    __shared__ long long warpSums[kScanThreads / 32];
    const int n = P.nCand;
    const int chunk = (n + kScanThreads - 1) / kScanThreads;
    const int b = threadIdx.x * chunk, e = min(n, b + chunk);
    long long local = 0;
    for (int i = b; i < e; ++i) local += P.rayCount[i];
    // block exclusive scan of `local`
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    long long x = local;
    for (int o = 1; o < 32; o <<= 1) {
        long long y = __shfl_up_sync(kFull, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warpSums[warp] = x;
    __syncthreads();
    if (warp == 0) {
        long long w = warpSums[lane];
        for (int o = 1; o < 32; o <<= 1) {
            long long y = __shfl_up_sync(kFull, w, o);
            if (lane >= o) w += y;
        }
        warpSums[lane] = w;
    }
    __syncthreads();
    long long run = x - local + (warp ? warpSums[warp - 1] : 0);
    for (int i = b; i < e; ++i) {
        P.rayStart[i] = run;
        run += P.rayCount[i];
    }
    if (threadIdx.x == kScanThreads - 1) P.rayStart[n] = warpSums[31];
}

__device__ __forceinline__ int findCandidate(const long long* start, int n, long long rid) {
    int lo = 0, hi = n;  // start[lo] <= rid < start[hi]
    while (hi - lo > 1) {
        int mid = (lo + hi) >> 1;
        if (start[mid] <= rid)
            lo = mid;
        else
            hi = mid;
    }
    return lo;
}

// rot * sphericalFibonacci(i, n) (sampling.hpp:28, vec.hpp:106-110)
template <typename R>
__device__ __forceinline__ V3<double> rayDirection(const WaveParams<R>& P, int s, int i, int n) {
    const double* m = P.rot + 9 * static_cast<size_t>(s);
    const double* v = P.fib + (n == P.nRaysFull ? 0 : 3 * P.nRaysFull) + 3 * i;
    return mk(m[0] * v[0] + m[1] * v[1] + m[2] * v[2], m[3] * v[0] + m[4] * v[1] + m[5] * v[2],
              m[6] * v[0] + m[7] * v[1] + m[8] * v[2]);
}

// --------------------------------------------------------- K1 primary rays
// sphereTrace (scene.hpp:391-435) as a per-lane state machine: state 0 marches
// (query at 2*lastD), state 1 is the owner-resolving query at the converged point
// (d + 1e-9), state 2 the polish loop (t += d, 2|d| + 1e-9, at most 8). Every
// iteration is exactly one query for every active lane.
// Total rays of a batch: the probe batch's prefix sum, or the direct count of a
// contact batch.
template <typename R>
__device__ __forceinline__ long long rayTotal(const WaveParams<R>& P) {
    return P.nRaysDirect >= 0 ? P.nRaysDirect : P.rayStart[P.nCand];
}

// Contact ray `item` = (pixel, sample), contactGI (shading.hpp:694-703): the
// pixel's Rng(seed, 0xc0417ff, y*W + x) stream advanced 2*sample draws (random
// access into the splitmix64 sequence), cosineHemisphereDir, the normal-offset
// origin, tMax = radius and startBound = bias + eps. False for sky pixels.
template <typename R>
__device__ __forceinline__ bool contactRay(const WaveParams<R>& P, long long item, V3<R>& o, V3<R>& dir, R& tMax,
                                           R& startBound) {
    const long long pix = item / P.contactSamples;
    const int smp = static_cast<int>(item - pix * P.contactSamples);
    const GPix& px = P.gb[pix];
    if (!(px.depth < INFINITY)) return false;
    const int x = static_cast<int>(pix % P.gw), y = static_cast<int>(pix / P.gw);
    Rng rng(hashCombine(hashCombine(P.seed, 0xc0417ffull), static_cast<uint64_t>(y) * P.gw + x));
    rng.s += 2ull * smp * 0x9e3779b97f4a7c15ull;
    const double u1 = rng.uniform();  // lz = sqrt(1 - u1); lx, ly from the host table
    const double2 l = reinterpret_cast<const double2*>(P.clocal)[item];
    const V3<double> nn = mk(px.normal[0], px.normal[1], px.normal[2]);
    const V3<double> dd = cosineHemisphereDir(l.x, l.y, u1, nn);
    const double cosT = smax(0.1, dot(dd, nn));
    const double bias = 2.0 * P.tc.eps / cosT;
    const V3<double> oo = mk(px.world_pos[0], px.world_pos[1], px.world_pos[2]) + nn * bias;
    o = mk(R(oo.x), R(oo.y), R(oo.z));
    dir = mk(R(dd.x), R(dd.y), R(dd.z));
    tMax = R(P.contactRadius);
    startBound = R(bias + P.tc.eps);
    return true;
}

// Every contact ray's setup (RNG draws, cosine-hemisphere direction, origin) at
// full lane occupancy, ahead of K1: in K1 only the few refilling lanes of a warp
// would run it.
template <typename R>
__global__ void __launch_bounds__(256) k_contact_setup(WaveParams<R> P) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= P.nRaysDirect) return;
    ContactRay<R> r;
    V3<R> o, dir;
    R tMax = R(0), sb = R(0);
    if (contactRay(P, i, o, dir, tMax, sb)) {
        r.o[0] = o.x;
        r.o[1] = o.y;
        r.o[2] = o.z;
        r.dir[0] = dir.x;
        r.dir[1] = dir.y;
        r.dir[2] = dir.z;
        r.tMax = tMax;
        r.startBound = sb;
    } else {
        r.o[0] = r.o[1] = r.o[2] = r.dir[0] = r.dir[1] = r.dir[2] = R(0);
        r.tMax = R(-1);
        r.startBound = R(0);
    }
    stStream(reinterpret_cast<ContactRay<R>*>(P.cray) + i, r);
}

// Every probe ray's set-up at full lane occupancy, ahead of K1 (in K1 only the few
// refilling lanes of a warp would run it), one CTA per probe: trace-order item
// rayStart + j, its Fibonacci sample i = perm[j] (coherent order), ray id
// rayStart + i, origin = the probe, direction = rot * sphericalFibonacci
// (sampling.hpp:28).
template <typename R>
__global__ void __launch_bounds__(256) k_probe_ray_setup(WaveParams<R> P) {
    // one CTA per candidate probe: its rotation, position and SDF are loaded once
    const int s = blockIdx.x;
    const long long start = P.rayStart[s];
    const int n = static_cast<int>(P.rayStart[s + 1] - start);
    if (n == 0) return;
    const int g = P.cand ? P.cand[s] : s;
    const double* pp = P.pc.probes.pos + 3 * static_cast<size_t>(g);
    const R ox = R(pp[0]), oy = R(pp[1]), oz = R(pp[2]);
    const R clear = P.useClear ? R(P.pc.probes.clear[g]) : R(-1);
    const int* perm = P.perm + (n == P.nRaysFull ? 0 : P.nRaysFull);
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
        const int i = perm[j];
        const V3<double> dd = rayDirection(P, s, i, n);
        ProbeRay<R> r;
        r.o[0] = ox;
        r.o[1] = oy;
        r.o[2] = oz;
        r.dir[0] = R(dd.x);
        r.dir[1] = R(dd.y);
        r.dir[2] = R(dd.z);
        r.rid = static_cast<int>(start + i);
        r.clear = clear;
        stStream(reinterpret_cast<ProbeRay<R>*>(P.pray) + start + j, r);
        if (!P.debug) {  // the sky radiance every ray starts with (K1 writes no miss records)
            R* rad = P.rad + 3 * static_cast<size_t>(start + j);
            __stcs(rad, R(P.scene.sky[0]));
            __stcs(rad + 1, R(P.scene.sky[1]));
            __stcs(rad + 2, R(P.scene.sky[2]));
        }
    }
}

// Warp-aggregated slot in a parking buffer (all 32 lanes call; -1 = not parked).
__device__ __forceinline__ long long parkSlot(unsigned long long* counter, bool park) {
    const unsigned m = __ballot_sync(kFull, park);
    if (m == 0) return -1;
    const unsigned lane = threadIdx.x & 31;
    const int leader = __ffs(m) - 1;
    unsigned long long base = 0;
    if (static_cast<int>(lane) == leader) base = atomicAdd(counter, static_cast<unsigned long long>(__popc(m)));
    base = __shfl_sync(kFull, base, leader);
    return park ? static_cast<long long>(base + __popc(m & ((1u << lane) - 1u))) : -1;
}

// The primitive records of the scene in shared memory for the whole persistent
// kernel (the north star's "primitives staged in shared memory via TMA"): one
// elected thread arms an mbarrier with the byte count and issues the bulk copies
// (cp.async.bulk, the TMA engine's 1-D form, 32 KB each); every thread waits on
// the barrier's phase 0. One CTA per SM holds the copy its warps share.
__device__ __forceinline__ void stagePrims(const void* src, int bytes) {
    __shared__ __align__(8) unsigned long long stageBar;
    const unsigned bar = static_cast<unsigned>(__cvta_generic_to_shared(&stageBar));
    const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(sdfgiDynSmem));
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
        const char* g = static_cast<const char*>(src);
        for (int off = 0; off < bytes; off += 32768) {
            const int n = min(32768, bytes - off);
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                             dst + off),
                         "l"(g + off), "r"(n), "r"(bar)
                         : "memory");
        }
    }
    __syncthreads();  // the barrier is initialised before anyone polls it
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra WAIT_%=;\n}\n" ::"r"(
            bar)
        : "memory");
}

#ifndef SDFGI_SHADOW_SETTLE_ON_GRID
#define SDFGI_SHADOW_SETTLE_ON_GRID 1  // also test marches still on the grid (C2 FP64 29.64 -> 29.52 ms)
#endif
// The initial bound of a march query (sphereTrace, scene.hpp:397-399: 2 * lastD).
// Candidate-grid walks also cap it at c = max(tMax - t, eps): the march tests
// d < eps (converge) and then d >= tMax - t (TMax miss), and
// query(p, min(2 lastD, c)) returns the reference's min(d, 2 lastD) exactly
// whenever that is below c, and otherwise c — which, like the reference's value,
// is not below eps and not below tMax - t: the same decision, step and t for every
// ray. A short segment (Contact GI: tMax = half a probe spacing) then ends its
// query as soon as every remaining candidate's lower bound clears it. Not in the
// flat cluster walk, whose per-cluster skip tests the reference's TraceStats
// count one for one.
#ifndef SDFGI_MARCH_CAP
#define SDFGI_MARCH_CAP 1
#endif
template <typename R>
__device__ __forceinline__ R marchSeed(const SceneView<R>& s, R lastD, R remaining, R eps) {
    const R b = R(2) * lastD;
    return (SDFGI_MARCH_CAP && s.useGrid) ? smin(b, smax(remaining, eps)) : b;
}

// PHASE 0 traces new rays and parks every march whose next point is off the
// candidate grid; PHASE 1 resumes the parked marches (no further parking).
template <typename R, bool ST, int MODE, int PHASE, bool STG = false>
__global__ void __launch_bounds__(STG ? StageOcc<R>::threads : kWaveThreads, STG ? 1 : WaveOcc<R>::trace)
    k_trace_primary(WaveParams<R> P) {
    if constexpr (STG) stagePrims(P.scene.stage, P.scene.stageBytes);
    ParkRay<R>* const park = reinterpret_cast<ParkRay<R>*>(P.park);
    const long long parkCap = static_cast<long long>(P.parkBytes / sizeof(ParkRay<R>));
    const long long total = PHASE ? min(static_cast<long long>(P.ctr[kCtrParkRay]), parkCap) : rayTotal(P);
    const R eps = R(P.tc.eps);
    const int maxSteps = P.tc.maxSteps;
    Counters cnt;
    cnt.zero();
    bool active = false, exhausted = false;
    WarpChunkFor<R> chunk;
    CellCache ccache;  // FP32 only (FP64: 1.5% slower at 64 registers, 2% at 72; SDFGI_CELL_CACHE64)
    int rid = 0;  // ray id (< 2^31)
    V3<R> o = mk(R(0), R(0), R(0)), dir = o;
    R t = 0, lastD = 0, d = 0, tMax = 0;  // tMax: contact rays only (probe rays: P.tc.rayTMax)
    auto tmax = [&]() { return MODE == 0 ? R(P.tc.rayTMax) : tMax; };
    int step = 0, state = 0, pol = 0, owner = -1, seed = -1;
    int titem = 0;       // the ray's trace-order position (its hitAt slot)
    bool fresh = false;  // resumed march: its pending t += d was applied before parking
    bool originIn = false;  // the ray starts inside the candidate grid (escape test)
    while (true) {
        __syncwarp();
        unsigned long long item;
        if (PHASE == 1) {
            if (fetchItem(P.ctr + kCtrFarRay, static_cast<unsigned long long>(total), active, exhausted, item, chunk)) {
                const ParkRay<R> r = ldStream(&park[item]);
                o = mk(r.o[0], r.o[1], r.o[2]);
                dir = mk(r.dir[0], r.dir[1], r.dir[2]);
                t = r.t;
                lastD = r.lastD;
                d = r.d;
                if (MODE == 1) tMax = r.tMax;  // probe rays: P.tc.rayTMax (tmax() below)
                step = r.step;
                state = r.state;
                pol = r.pol;
                owner = r.owner;
                seed = r.seed;
                titem = r.item;
                rid = static_cast<int>(r.rid);
                active = true;
                fresh = true;
            }
        } else {
            const bool got =
                fetchItem(P.ctr + kCtrRay, static_cast<unsigned long long>(total), active, exhausted, item, chunk,
                          MODE == 0 ? P.pray : P.cray, MODE == 0 ? int(sizeof(ProbeRay<R>)) : int(sizeof(ContactRay<R>)));
            if (got) {
            titem = static_cast<int>(item);
            R startBound = R(INFINITY);
            bool ok = true;
            if (MODE == 0) {
                // prepared by k_probe_ray_setup (trace order: consecutive lanes get
                // neighbouring directions; results are stored by ray id)
                const ProbeRay<R> r = ldStream(reinterpret_cast<const ProbeRay<R>*>(P.pray) + item);
                rid = r.rid;
                // the probe's SDF for the march's first query (< 0: query it), carried
                // in d until state 1 sets it (one register fewer than a variable of its own)
                d = r.clear;
                o = mk(r.o[0], r.o[1], r.o[2]);
                dir = mk(r.dir[0], r.dir[1], r.dir[2]);
            } else {
                rid = static_cast<int>(item);
                d = R(-1);
                const ContactRay<R> r = ldStream(reinterpret_cast<const ContactRay<R>*>(P.cray) + item);
                o = mk(r.o[0], r.o[1], r.o[2]);
                dir = mk(r.dir[0], r.dir[1], r.dir[2]);
                tMax = r.tMax;
                startBound = r.startBound;
                ok = r.tMax >= R(0);
            }
            t = R(0);
            lastD = startBound * R(0.5);
            step = 0;
            state = 0;
            owner = -1;
            seed = -1;
            active = ok;
            originIn = P.escape && ok && gridCell<R>(P.scene.grid, o) >= 0;
            if (!ok) {  // sky pixel of a contact batch: no ray (the combine skips it)
                HitRec<R> h;
                h.p[0] = h.p[1] = h.p[2] = R(0);
                h.n[0] = h.n[1] = R(0);
                h.n[2] = R(1);
                h.t = R(0);
                h.owner = -1;
                h.status = 0;
                P.hits[rid] = h;
                P.hitAt[titem] = -1;
            }
            if (ST && ok) ++cnt.sphere;
            if (ok && maxSteps <= 0) {  // loop never runs: StepLimit
                HitRec<R> h;
                h.p[0] = h.p[1] = h.p[2] = R(0);
                h.n[0] = h.n[1] = R(0);
                h.n[2] = R(1);
                h.t = R(0);
                h.owner = -1;
                h.status = 2 << 1;
                P.hits[rid] = h;
                P.hitAt[titem] = -1;
                P.rad[3 * static_cast<size_t>(rid)] = R(P.scene.sky[0]);
                P.rad[3 * static_cast<size_t>(rid) + 1] = R(P.scene.sky[1]);
                P.rad[3 * static_cast<size_t>(rid) + 2] = R(P.scene.sky[2]);
                active = false;
            }
            }
        }
        if (!__any_sync(kFull, active)) {
            if (__all_sync(kFull, exhausted)) break;
            continue;
        }
        V3<R> p = o;
        R initD = R(0);
        bool parkIt = false, escaped = false, known = false;
        int cell = kCellUnknown;  // phase 0: p's cell (parking test), reused by the query
        R cellR = R(0);
#if SDFGI_HOIST_CELL_LOAD
        int4 preRec = make_int4(0, 0, 0, 0);
#endif
        if (active) {
            if (state == 2 && !fresh) t += d;
            fresh = false;
            p = o + dir * t;
            if (PHASE == 0 && P.scene.useGrid) cell = gridCell<R>(P.scene.grid, p, &cellR);
#if SDFGI_HOIST_CELL_LOAD
            if (cell >= 0) preRec = __ldg(&P.scene.grid.cell[cell]);  // its latency under the logic below
#endif
            // the first query of a probe ray is the probe's own SDF, known from the relocation
            known = PHASE == 0 && state == 0 && step == 0 && d >= R(0);
            escaped = PHASE == 0 && originIn && state == 0 && cell < 0 && !known;
            parkIt = PHASE == 0 && park && cell < 0 && !escaped && !known;
            if (escaped) {
                if (ST) ++cnt.steps;
            } else if (parkIt) {
            } else if (state == 0) {
                if (ST) ++cnt.steps;
                initD = marchSeed(P.scene, lastD, tmax() - t, eps);
            } else if (state == 1) {
                initD = polishPad(d);
            } else {
                initD = polishPad(R(2) * fabs(d));
            }
        }
        if (PHASE == 0) {
            const long long ps = parkSlot(P.ctr + kCtrParkRay, parkIt);
            if (ps >= parkCap) {  // buffer full: this march queries here after all
                parkIt = false;
                if (state == 0) {
                    if (ST) ++cnt.steps;
                    initD = marchSeed(P.scene, lastD, tmax() - t, eps);
                } else if (state == 1) {
                    initD = polishPad(d);
                } else {
                    initD = polishPad(R(2) * fabs(d));
                }
            }
            if (parkIt) {
                ParkRay<R> r;
                r.o[0] = o.x;
                r.o[1] = o.y;
                r.o[2] = o.z;
                r.dir[0] = dir.x;
                r.dir[1] = dir.y;
                r.dir[2] = dir.z;
                r.t = t;
                r.lastD = lastD;
                r.d = d;
                r.tMax = tmax();
                r.step = step;
                r.state = state;
                r.pol = pol;
                r.owner = owner;
                r.rid = rid;
                r.seed = seed;
                r.item = titem;
                stStream(&park[ps], r);
                active = false;
            }
        }
        int o2 = -1;
        R nd = R(0);
        if (active && known)
            nd = smin(d, initD);  // exactly query(o, initD) = min(SDF(o), initD)
        else if (active && !escaped)
            nd = query<R, ST, STG>(P.scene, p, initD, &o2, &cnt, PHASE ? seed : -1, cell, cellR,
                              useCellCache<R>() ? &ccache : nullptr,
#if SDFGI_HOIST_CELL_LOAD
                              cell >= 0 ? &preRec : nullptr
#else
                              nullptr
#endif
                              );
        if (active) {
            if (o2 >= 0) seed = o2;
            int done = 0;  // 1 converged, 2 TMax, 3 StepLimit
            if (escaped) {
                done = 2;  // left the grid box for good: a miss (sky either way)
            } else if (state == 0) {
                if (nd < eps) {
                    d = nd;
                    if (P.ownerFromMarch && o2 >= 0) {  // the owner query's result, already known
                        owner = o2;
                        pol = 0;
                        state = 2;
                        if (!(fabs(d) > R(0.25) * eps)) done = 1;
                    } else {
                        state = 1;
                    }
                } else if (nd >= tmax() - t) {
                    done = 2;
                } else {
                    t += nd;
                    lastD = nd;
                    if (++step >= maxSteps) done = 3;
                }
            } else {
                d = nd;
                if (state == 1) {
                    owner = o2;
                    pol = 0;
                    state = 2;
                } else {
                    if (o2 >= 0) owner = o2;
                    ++pol;
                }
                if (!(pol < 8 && fabs(d) > R(0.25) * eps)) done = 1;
            }
            if (done) {
                HitRec<R> h;
                h.owner = -1;
                h.n[0] = h.n[1] = R(0);
                h.n[2] = R(1);
                if (done == 1) {
                    h.p[0] = p.x;
                    h.p[1] = p.y;
                    h.p[2] = p.z;
                    h.t = t;
                    h.owner = owner;  // normal: k_hit_normals (evalGradient of the owner)
                    h.status = 1 | ((step + 1) << 8);
                } else {
                    h.p[0] = h.p[1] = h.p[2] = R(0);
                    h.t = R(0);
                    h.status = ((done == 2 ? 1 : 2) << 1) | ((done == 2 ? step + 1 : maxSteps) << 8);
                }
                // only converged rays' records are read (K3a, the normals; per-ray
                // debug records read every ray's). A probe batch's radiance starts at
                // the sky (k_probe_ray_setup); a contact batch's combine reads the converged
                // flags (conv) and the radiance of converged rays only
                const bool lean = !P.debug && !P.keepAll;
                if (!lean || done == 1) stStream(&P.hits[rid], h);
                if (MODE == 1 && done == 1 && P.conv) P.conv[rid] = 1;
                if ((!lean || (MODE == 1 && done == 1)) &&
                    !(done == 1 && owner >= 0)) {  // shadeHit's miss branch: K3a shades only the hit list
                    __stcs(&P.rad[3 * static_cast<size_t>(rid)], R(P.scene.sky[0]));
                    __stcs(&P.rad[3 * static_cast<size_t>(rid) + 1], R(P.scene.sky[1]));
                    __stcs(&P.rad[3 * static_cast<size_t>(rid) + 2], R(P.scene.sky[2]));
                }
                active = false;
            }
            // converged hits with an owner (the only ones shadeHit lights) are
            // compacted after the kernel, in trace order (coherent K2/K3a warps)
            if (done) P.hitAt[titem] = (done == 1 && owner >= 0) ? rid : -1;
        }
    }
    if (ST) flushCounters(cnt, P.stats);
}

// directIrradiance's per-light set-up (probe_update.hpp:100-128) for the hit `rid`
// at pos with normal nrm: a light below the horizon (or on the point) gets vis -1
// (no contribution), a segment too short to trace vis 1; every other pair becomes
// a ShadowRay for K2, appended to its light's list. Called by the lanes `am` of a
// warp together (uniform light loop), `valid` false for lanes without a hit.
template <typename R>
__device__ __forceinline__ void shadowSetup(const WaveParams<R>& P, unsigned am, bool valid, int rid, V3<R> pos,
                                            V3<R> nrm) {
    const int L = P.scene.n_lights;
    const unsigned lane = threadIdx.x & 31;
    for (int li = 0; li < L; ++li) {
        const DLight& Lt = P.scene.lights[li];
        const unsigned long long slot = static_cast<unsigned long long>(rid) * L + li;
        bool live = false;
        V3<R> dir = mk(R(0), R(0), R(0));
        R bias = R(0), tMax = R(0);
        if (valid) {
            bool skip = false;
            if (Lt.kind == 0) {
                V3<R> toLight = mk(R(Lt.position[0]), R(Lt.position[1]), R(Lt.position[2])) - pos;
                R r2 = dot(toLight, toLight);
                if (r2 < R(1e-12)) {
                    skip = true;
                } else {
                    R r = sqrt(r2);
                    dir = toLight / r;
                    if (dot(nrm, dir) <= R(0)) skip = true;
                    tMax = r;
                }
            } else if (Lt.kind == 1) {
                dir = mk(R(-Lt.direction[0]), R(-Lt.direction[1]), R(-Lt.direction[2]));
                if (dot(nrm, dir) <= R(0)) skip = true;
                tMax = R(P.tc.rayTMax);
            } else {
                skip = true;
            }
            if (skip) {
                P.vis[slot] = R(-1);
            } else {
                const R cosT = dot(nrm, dir);
                bias = R(2.0) * R(P.tc.eps) / smax(R(0.1), cosT);
                live = tMax - bias > bias;
                if (!live) P.vis[slot] = R(1);
            }
        }
        const unsigned m = __ballot_sync(am, live);
        if (m == 0) continue;
        const int leader = __ffs(m) - 1;
        unsigned long long base = 0;
        if (static_cast<int>(lane) == leader)
            base = atomicAdd(P.ctr + kLightCtr + li, static_cast<unsigned long long>(__popc(m)));
        base = __shfl_sync(am, base, leader);
        if (live) {
            ShadowRay<R> r;
            const V3<R> o = pos + nrm * bias;
            r.o[0] = o.x;
            r.o[1] = o.y;
            r.o[2] = o.z;
            r.dir[0] = dir.x;
            r.dir[1] = dir.y;
            r.dir[2] = dir.z;
            r.t = bias;
            r.tEnd = tMax - bias;
            r.rid = rid;
            r.li = li;
            stStream(&P.sray[li * P.srayCap + base + __popc(m & ((1u << lane) - 1u))], r);
        }
    }
}

// The converged hits' normals (evalGradient of the owner, primitives.hpp:96-108)
// and their shadow-ray set-up over the compacted hit list — every lane has one,
// instead of the few lanes of a K1 warp whose rays just converged. EVAL = false:
// the normals are given (a shadeHit batch, sdfgi_shade_hits), only the set-up runs.
template <typename R, bool EVAL = true>
__global__ void __launch_bounds__(128) k_hit_normals(WaveParams<R> P) {
    const unsigned long long n = P.ctr[kCtrHits];
    for (unsigned long long i = static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<unsigned long long>(gridDim.x) * blockDim.x) {
        const unsigned am = __activemask();
        const int rid = P.hitList[i];
        HitRec<R>& h = P.hits[rid];
        const V3<R> pos = mk(h.p[0], h.p[1], h.p[2]);
        V3<R> nn = mk(h.n[0], h.n[1], h.n[2]);
        if (EVAL) {
            nn = evalGradient(P.scene.prims[h.owner], pos);
            h.n[0] = nn.x;
            h.n[1] = nn.y;
            h.n[2] = nn.z;
        }
        shadowSetup(P, am, true, rid, pos, nn);
    }
}

// ----------------------------------------------------------- K2 shadow rays
// One (converged hit, light) item per lane: directIrradiance's setup
// (probe_update.hpp:100-128) and the softShadowTrace march (scene.hpp:459-476),
// one query per iteration. vis = 1 when the segment is too short to trace.
// PHASE 0 / 1 as in K1: off-grid shadow marches are parked and resumed together.
template <typename R, bool ST, int PHASE, bool STG = false>
__global__ void __launch_bounds__(STG ? StageOcc<R>::threads : kWaveThreads, STG ? 1 : WaveOcc<R>::shadow)
    k_trace_shadow(WaveParams<R> P) {
    if constexpr (STG) stagePrims(P.scene.stage, P.scene.stageBytes);
    const int L = P.scene.n_lights;
    ParkShadow<R>* const park = reinterpret_cast<ParkShadow<R>*>(P.park);
    const unsigned long long parkCap = P.parkBytes / sizeof(ParkShadow<R>);
    unsigned long long traced = 0;
    for (int li = 0; li < L; ++li) traced += P.ctr[kLightCtr + li];
    const unsigned long long total = PHASE ? min(P.ctr[kCtrParkShadow], parkCap) : traced;
    const R minStep = R(P.tc.shadowMinStep > 0 ? P.tc.shadowMinStep : 5e-4), inf = R(INFINITY),
            k = R(P.tc.shadowK);
    const int maxSteps = P.tc.shadowSteps;
    Counters cnt;
    cnt.zero();
    bool active = false, exhausted = false;
    WarpChunkFor<R> chunk;
    CellCache ccache;  // FP32 only (FP64: 1.5% slower at 64 registers, 2% at 72; SDFGI_CELL_CACHE64)
    unsigned long long slot = 0;
    V3<R> o = mk(R(0), R(0), R(0)), dir = o;
    R t = 0, tEnd = 0, v = 0, lastD = 0;
    int step = 0, seed = -1;
    while (true) {
        __syncwarp();
        unsigned long long item;
        if (PHASE == 1) {
            if (fetchItem(P.ctr + kCtrFarShadow, total, active, exhausted, item, chunk)) {
                const ParkShadow<R> r = ldStream(&park[item]);
                o = mk(r.o[0], r.o[1], r.o[2]);
                dir = mk(r.dir[0], r.dir[1], r.dir[2]);
                t = r.t;
                tEnd = r.tEnd;
                v = r.v;
                lastD = r.lastD;
                step = r.step;
                seed = r.seed;
                slot = r.slot;
                active = true;
            }
        } else if (fetchItem(P.ctr + kCtrShadow, total, active, exhausted, item, chunk)) {
            // light-major: consecutive lanes take consecutive traced marches toward
            // the same light (set up by the hit setup, shadowSetup)
            int li = 0;
            unsigned long long k = item;
            while (li + 1 < L && k >= P.ctr[kLightCtr + li]) k -= P.ctr[kLightCtr + li++];
            const ShadowRay<R> r = ldStream(&P.sray[li * P.srayCap + k]);
            o = mk(r.o[0], r.o[1], r.o[2]);
            dir = mk(r.dir[0], r.dir[1], r.dir[2]);
            t = r.t;
            tEnd = r.tEnd;
            slot = static_cast<unsigned long long>(r.rid) * L + r.li;
            v = R(1);
            lastD = inf;
            step = 0;
            seed = -1;
            active = true;
            if (ST) ++cnt.shadow;
        }
        if (!__any_sync(kFull, active)) {
            if (__all_sync(kFull, exhausted)) break;
            continue;
        }
        bool want = active && step < maxSteps && t < tEnd;
        V3<R> p = o;
        if (want) p = o + dir * t;
        int cell = kCellUnknown;  // phase 0: p's cell (parking test), reused by the query
        R cellR = R(0);
        if (PHASE == 0 && want && P.scene.useGrid) cell = gridCell<R>(P.scene.grid, p, &cellR);
#if SDFGI_HOIST_CELL_LOAD2
        constexpr bool hoist2 = sizeof(R) == 8;
        int4 preRec = make_int4(0, 0, 0, 0);
        if (hoist2 && cell >= 0) preRec = __ldg(&P.scene.grid.cell[cell]);  // its latency under the settle test
#endif
        // accel mode 2: off the grid, a march whose remaining terms cannot lower v
        // ends here with v (shadowSettled)
        if (P.settle && want && (PHASE == 1 || cell < 0 || SDFGI_SHADOW_SETTLE_ON_GRID) &&
            shadowSettled(P.scene.grid, p, dir, t, tEnd, k, v))
            want = false;
        if (PHASE == 0) {
            bool parkIt = want && park && cell < 0;
            const long long ps = parkSlot(P.ctr + kCtrParkShadow, parkIt);
            if (ps >= static_cast<long long>(parkCap)) parkIt = false;  // buffer full
            if (parkIt) {
                ParkShadow<R> r;
                r.o[0] = o.x;
                r.o[1] = o.y;
                r.o[2] = o.z;
                r.dir[0] = dir.x;
                r.dir[1] = dir.y;
                r.dir[2] = dir.z;
                r.t = t;
                r.tEnd = tEnd;
                r.v = v;
                r.lastD = lastD;
                r.step = step;
                r.seed = seed;
                r.slot = slot;
                stStream(&park[ps], r);
                active = false;
                want = false;
            }
        }
        if (ST && want) ++cnt.steps;
        R d = R(0);
        int o2 = -1;
        if (want)
            d = query<R, ST, STG>(P.scene, p, lastD == inf ? inf : R(2) * lastD, &o2, &cnt, PHASE ? seed : -1, cell, cellR,
                             useCellCache<R>() ? &ccache : nullptr,
#if SDFGI_HOIST_CELL_LOAD2
                             hoist2 && cell >= 0 ? &preRec : nullptr
#else
                             nullptr
#endif
                             );
        if (o2 >= 0) seed = o2;
        if (active) {
            bool done = false;
            if (!want) {
                done = true;
            } else {
                v = smin(v, sclamp(k * d / t, R(0), R(1)));
                if (v < R(1e-3)) {
                    v = R(0);
                    done = true;
                } else {
                    t += smax(d, minStep);
                    lastD = smax(d, minStep);
                    ++step;
                }
            }
            if (done) {
                __stcs(&P.vis[slot], v);
                active = false;
            }
        }
    }
    if (ST) flushCounters(cnt, P.stats);
}

// ------------------------------------------------- K3 shade + convolve + blend
// shadeHit (probe_update.hpp:136-149) with directIrradiance's sum in light order
// (visibility from K2), then convolveIrradiance + hysteresis blend + fillBorder
// (probe_update.hpp:192-209, atlas.hpp:44-56) for one probe per CTA.
// directIrradiance (probe_update.hpp:97-132) summed in light order with the K2
// visibilities of item rid (vis[rid * L + light]).
template <typename R>
__device__ __forceinline__ V3<double> directLight(const WaveParams<R>& P, const HitRec<R>& h, unsigned long long rid) {
    const SceneView<R>& s = P.scene;
    const V3<R> pos = mk(h.p[0], h.p[1], h.p[2]);
    const V3<R> nrm = mk(h.n[0], h.n[1], h.n[2]);
    V3<double> total = mk(0.0, 0.0, 0.0);
    for (int li = 0; li < s.n_lights; ++li) {
        const DLight& L = s.lights[li];
        V3<double> I = mk(L.intensity[0], L.intensity[1], L.intensity[2]);
        V3<double> unshadowed;
        if (L.kind == 0) {
            V3<R> toLight = mk(R(L.position[0]), R(L.position[1]), R(L.position[2])) - pos;
            R r2 = dot(toLight, toLight);
            if (r2 < R(1e-12)) continue;
            R r = sqrt(r2);
            V3<R> dir = toLight / r;
            R cosT = dot(nrm, dir);
            if (cosT <= R(0)) continue;
            unshadowed = I * static_cast<double>(cosT / r2);
        } else if (L.kind == 1) {
            V3<R> dir = mk(R(-L.direction[0]), R(-L.direction[1]), R(-L.direction[2]));
            R cosT = dot(nrm, dir);
            if (cosT <= R(0)) continue;
            unshadowed = I * static_cast<double>(cosT);
        } else {
            continue;
        }
        const R vis = P.vis[rid * s.n_lights + li];
        total = total + unshadowed * static_cast<double>(vis);
    }
    return total;
}

template <typename R>
__device__ __forceinline__ V3<double> shadeRay(const WaveParams<R>& P, const HitRec<R>& h, unsigned long long rid,
                                               R* slab = nullptr, int* usedMvc = nullptr) {
    const SceneView<R>& s = P.scene;
    if (!(h.status & 1) || h.owner < 0) return mk(s.sky[0], s.sky[1], s.sky[2]);
    const V3<double> total = directLight(P, h, rid);
    const double* A = s.albedo + 3 * h.owner;
    const double* E = s.emission + 3 * h.owner;
    V3<double> brdf = mk(A[0], A[1], A[2]) / kPi;
    V3<double> radiance = mk(E[0], E[1], E[2]) + brdf * total;
    if (P.tc.bounceCoeff > 0 && P.prevAtlas != nullptr) {
        V3<double> prev;
        V3<double> hp = mk<double>(h.p[0], h.p[1], h.p[2]);
        V3<double> hn = mk<double>(h.n[0], h.n[1], h.n[2]);
        if (sampleBounceIrradiance<R, true>(P.pc.cas, P.pc.nCas, P.pc.probes, P.prevAtlas, P.oct, hp, hn, P.tc.mvcFrac, &prev,
                                      slab, usedMvc))
            radiance = radiance + brdf * (prev * P.tc.bounceCoeff);
    }
    return radiance;
}

// shadeHit with the bounce lookup's MVC path deferred: the radiance so far (emission
// + directIrradiance, and the trilinear bounce when the stencil takes it) in *out;
// true when the stencil takes the MVC path (probe_volume.hpp:278), whose bounce
// term K3c adds (radiance = radiance + brdf * (prev * bounceCoeff), the same
// addition in the same order as probe_update.hpp:143-147).
// Returns 0 (done), 1 (MVC stencil: K3c) or 2 (trilinear stencil deferred to K3c's
// list of those, when P.triList is set).
template <typename R>
__device__ __forceinline__ int shadeRayDeferred(const WaveParams<R>& P, const HitRec<R>& h, unsigned long long rid,
                                                V3<double>* out) {
    const SceneView<R>& s = P.scene;
    if (!(h.status & 1) || h.owner < 0) {
        *out = mk(s.sky[0], s.sky[1], s.sky[2]);
        return 0;
    }
    const V3<double> total = directLight(P, h, rid);
    const double* A = s.albedo + 3 * h.owner;
    const double* E = s.emission + 3 * h.owner;
    const V3<double> brdf = mk(A[0], A[1], A[2]) / kPi;
    V3<double> radiance = mk(E[0], E[1], E[2]) + brdf * total;
    *out = radiance;
    if (!(P.tc.bounceCoeff > 0 && P.prevAtlas != nullptr && P.pc.nCas > 0) || P.prevZero) return 0;
    const V3<double> hp = mk<double>(h.p[0], h.p[1], h.p[2]);
    const V3<double> hn = mk<double>(h.n[0], h.n[1], h.n[2]);
    const StencilCell sc = stencilCell(P.pc.cas, P.pc.nCas, P.pc.probes, hp, P.tc.mvcFrac);
    if (sc.chosen < 0) return 0;  // sky fallback: no bounce
    if (sc.wantMvc) return 1;
    if (P.triList) return 2;
    double w[8];
    for (int k = 0; k < 8; ++k) w[k] = trilinearWeight(sc, k);
    const Stencil st = finishStencil(P.pc.cas, P.pc.probes, sc, w, 0);
    V3<double> prev;
    if (bounceFromStencil<R>(P.pc.cas, P.pc.probes, P.prevAtlas, P.oct, st, hp, hn, &prev))
        *out = radiance + brdf * (prev * P.tc.bounceCoeff);
    return 0;
}

// Append rid to the list whose counter is ctr[slot] (lanes with want = true).
__device__ __forceinline__ void appendList(unsigned long long* ctr, int slot, int* list, bool want, int rid) {
    const unsigned am = __activemask();
    const unsigned m = __ballot_sync(am, want);
    if (!m) return;
    const int leader = __ffs(m) - 1;
    unsigned long long base = 0;
    if (static_cast<int>(threadIdx.x & 31) == leader)
        base = atomicAdd(ctr + slot, static_cast<unsigned long long>(__popc(m)));
    base = __shfl_sync(am, base, leader);
    if (want) list[base + __popc(m & ((1u << (threadIdx.x & 31)) - 1u))] = rid;
}

// K3a: shadeHit per ray (thread per ray, grid-stride): emission + directIrradiance
// summed in light order with the K2 visibilities + the bounce lookup; radiance to
// P.rad (3 per ray). Kept apart from the convolution so the stencil register
// footprint does not cap the convolution's occupancy. DEFER: the bounce lookup is
// deferred — hits whose stencil takes the MVC path go to P.mvcList (K3c, one hit
// per thread), the others to P.triList (K3d); !DEFER (per-ray debug records)
// evaluates the whole lookup inline.
template <typename R, bool ST, bool DEFER>
__global__ void __launch_bounds__(128, WaveOcc<R>::shade) k_shade_rays(WaveParams<R> P) {
    // the compacted hit list (misses got the sky radiance in K1); every ray when
    // per-ray debug records are written
    extern __shared__ __align__(16) unsigned char k3aSmem[];
    R* slab = reinterpret_cast<R*>(k3aSmem);  // kMvcSlab values per thread (MVC working set)
    const bool all = P.debug != 0;
    const long long total = all ? rayTotal(P) : static_cast<long long>(P.ctr[kCtrHits]);
    const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
    unsigned long long nShaded = 0, nMvc = 0;  // shading work (ST): shadeHit calls, MVC evaluations
    for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += stride) {
        const long long rid = all ? i : static_cast<long long>(P.hitList[i]);
        const HitRec<R> h = ldStream(&P.hits[rid]);
        int mvc = 0;
        V3<double> L;
        if constexpr (DEFER) {
            const int defer = shadeRayDeferred(P, h, static_cast<unsigned long long>(rid), &L);
            appendList(P.ctr, kCtrMvc, P.mvcList, defer == 1, static_cast<int>(rid));
            if (P.triList) appendList(P.ctr, kCtrTri, P.triList, defer == 2, static_cast<int>(rid));
        } else {
            L = shadeRay(P, h, static_cast<unsigned long long>(rid), slab, ST ? &mvc : nullptr);
        }
        if (ST && (h.status & 1) && h.owner >= 0) {
            ++nShaded;
            nMvc += mvc;
        }
        __stcs(&P.rad[3 * rid], R(L.x));
        __stcs(&P.rad[3 * rid + 1], R(L.y));
        __stcs(&P.rad[3 * rid + 2], R(L.z));
        if (P.debug) {
            const int s = findCandidate(P.rayStart, P.nCand, rid);
            const int i = static_cast<int>(rid - P.rayStart[s]);
            const int n = static_cast<int>(P.rayStart[s + 1] - P.rayStart[s]);
            const V3<double> dir = rayDirection(P, s, i, n);
            RayRecord r;
            r.dir[0] = dir.x;
            r.dir[1] = dir.y;
            r.dir[2] = dir.z;
            const bool conv = h.status & 1;
            r.t = conv ? double(h.t) : 0.0;
            r.radiance[0] = L.x;
            r.radiance[1] = L.y;
            r.radiance[2] = L.z;
            r.normal[0] = h.n[0];
            r.normal[1] = h.n[1];
            r.normal[2] = h.n[2];
            r.converged = conv ? 1 : 0;
            r.miss = (h.status >> 1) & 3;
            r.prim_index = h.owner >= 0 ? P.scene.orig[h.owner] : -1;
            r.steps = h.status >> 8;
            P.records[rid] = r;
        }
    }
    if (ST) {  // every lane reaches here (the grid-stride loop has no early return)
        for (int o = 16; o > 0; o >>= 1) {
            nShaded += __shfl_xor_sync(kFull, nShaded, o);
            nMvc += __shfl_xor_sync(kFull, nMvc, o);
        }
        if ((threadIdx.x & 31) == 0) {
            if (nShaded) atomicAdd(P.stats + 20, nShaded);
            if (nMvc) atomicAdd(P.stats + 21, nMvc);
        }
    }
}

// K3c: the bounce lookup of the hits K3a deferred (interpolationStencil with
// mvcWeightsHex, mean_value.hpp:16-107, then sampleBounceIrradiance's lookup,
// probe_update.hpp:63-92), one thread per hit over the compacted list: every lane
// of a warp runs the MVC (in K3a 18% of a warp's lanes took the trilinear path and
// idled), and K3a no longer carries the MVC's registers. The MVC working set lives
// in a per-thread shared-memory slab. (Evaluating each of the cell's 18 distinct
// edge angles once instead of per triangle was measured slower: the larger slab
// halves the resident warps, profiles/README.md.)
// K3a's deferred trilinear bounce lookups (P.triList): every lane takes the same
// path at full occupancy; the same stencil and addition as in K3a
// (shadeRayDeferred / probe_update.hpp:143-147).
template <typename R>
__global__ void __launch_bounds__(256) k_shade_tri(WaveParams<R> P) {
    const long long n = static_cast<long long>(P.ctr[kCtrTri]);
    const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
    for (long long j = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; j < n; j += stride) {
        const int rid = P.triList[j];
        const HitRec<R> h = P.hits[rid];
        const V3<double> hp = mk<double>(h.p[0], h.p[1], h.p[2]);
        const V3<double> hn = mk<double>(h.n[0], h.n[1], h.n[2]);
        const StencilCell sc = stencilCell(P.pc.cas, P.pc.nCas, P.pc.probes, hp, P.tc.mvcFrac, false);
        double w[8];
        for (int k = 0; k < 8; ++k) w[k] = trilinearWeight(sc, k);
        const Stencil st = finishStencil(P.pc.cas, P.pc.probes, sc, w, 0);
        V3<double> prev;
        if (bounceFromStencil<R>(P.pc.cas, P.pc.probes, P.prevAtlas, P.oct, st, hp, hn, &prev)) {
            const double* A = P.scene.albedo + 3 * h.owner;
            const V3<double> brdf = mk(A[0], A[1], A[2]) / kPi;
            const V3<double> base = mk(double(P.rad[3 * rid]), double(P.rad[3 * rid + 1]), double(P.rad[3 * rid + 2]));
            const V3<double> L = base + brdf * (prev * P.tc.bounceCoeff);
            P.rad[3 * rid] = R(L.x);
            P.rad[3 * rid + 1] = R(L.y);
            P.rad[3 * rid + 2] = R(L.z);
        }
    }
}

template <typename R, bool ST>
__global__ void __launch_bounds__(kMvcThreads, kMvcMinBlocks) k_shade_mvc(WaveParams<R> P) {
    extern __shared__ __align__(16) unsigned char k3cSmem[];
    R* slab = reinterpret_cast<R*>(k3cSmem);
    const long long n = static_cast<long long>(P.ctr[kCtrMvc]);
    const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
    unsigned long long nMvc = 0;
    for (long long j = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; j < n; j += stride) {
        const int rid = P.mvcList[j];
        const HitRec<R> h = P.hits[rid];
        const V3<double> hp = mk<double>(h.p[0], h.p[1], h.p[2]);
        const V3<double> hn = mk<double>(h.n[0], h.n[1], h.n[2]);
        const Stencil st = interpolationStencil<R, true>(P.pc.cas, P.pc.nCas, P.pc.probes, hp, P.tc.mvcFrac, slab);
        if (ST) nMvc += st.usedMvc;
        V3<double> prev;
        if (bounceFromStencil<R>(P.pc.cas, P.pc.probes, P.prevAtlas, P.oct, st, hp, hn, &prev)) {
            const double* A = P.scene.albedo + 3 * h.owner;
            const V3<double> brdf = mk(A[0], A[1], A[2]) / kPi;
            const V3<double> base = mk(double(P.rad[3 * rid]), double(P.rad[3 * rid + 1]), double(P.rad[3 * rid + 2]));
            const V3<double> L = base + brdf * (prev * P.tc.bounceCoeff);
            P.rad[3 * rid] = R(L.x);
            P.rad[3 * rid + 1] = R(L.y);
            P.rad[3 * rid + 2] = R(L.z);
        }
    }
    if (ST) {
        for (int o = 16; o > 0; o >>= 1) nMvc += __shfl_xor_sync(kFull, nMvc, o);
        if ((threadIdx.x & 31) == 0 && nMvc) atomicAdd(P.stats + 21, nMvc);
    }
}

// K3b: one CTA per probe, one thread per (texel, channel): convolveIrradiance
// (probe_update.hpp:25-34) — every channel summed over the rays in the
// reference's order, so FP64 texels are bit-identical — hysteresis blend
// (:192-206), fillBorder (atlas.hpp:44-56) in shared memory, 16-byte tile stores.
template <typename R, bool ST>
__global__ void __launch_bounds__(kConvThreads) k_convolve(WaveParams<R> P) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ __align__(16) float tile[12 * 12 * 3 + 4];
    __shared__ unsigned long long redDelta[kConvThreads / 32];

    const int s = blockIdx.x;
    const int n = P.rayCount[s];
    if (n == 0) return;  // dead probe: its back tile is the copied front tile
    const int g = P.cand ? P.cand[s] : s;
    const ProbesView& pv = P.pc.probes;
    const int reject = n != P.nRaysFull;  // 2N rays <=> rejectHistory at setup
    const long long start = P.rayStart[s];
    const int res = P.oct;
    const int T = res + 2;
    const double alpha = reject ? 1.0 : sclamp((1.0 - P.hysteresis) * n / P.nRaysFull, P.alphaMin, 1.0);
    const double scale = 4.0 * kPi / static_cast<double>(n);
    const float* oldTile = P.prevAtlas + static_cast<size_t>(g) * T * T * 3;
    double maxDelta = 0.0;
    if (kConvChunk > 0) {
        // per ray (dir, radiance) as 6 values, read as three 16-byte words; each
        // thread sums up to two texels, every channel in the rays' order
        __shared__ __align__(16) R sray[(kConvChunk > 0 ? kConvChunk : 1) * 6];
        const int nt = res * res;
        const int txA = threadIdx.x, txB = threadIdx.x + blockDim.x;
        R D[2][3];
        for (int q = 0; q < 2; ++q) {
            const int tx = q ? txB : txA;
            const int y = tx / res, x = tx % res;
            const V3<double> dd = octDecode(V2<double>{(x + 0.5) / res, (y + 0.5) / res});
            D[q][0] = R(dd.x);
            D[q][1] = R(dd.y);
            D[q][2] = R(dd.z);
        }
        const bool hasA = txA < nt, hasB = txB < nt;
        R a[2][3] = {{0, 0, 0}, {0, 0, 0}};
        for (int c0 = 0; c0 < n; c0 += kConvChunk) {
            const int m = min(kConvChunk, n - c0);
            __syncthreads();  // the previous chunk is consumed
            for (int i = threadIdx.x; i < m; i += blockDim.x) {
                const V3<double> dir = rayDirection(P, s, c0 + i, n);
                sray[6 * i] = R(dir.x);
                sray[6 * i + 1] = R(dir.y);
                sray[6 * i + 2] = R(dir.z);
            }
            for (int k = threadIdx.x; k < 3 * m; k += blockDim.x)
                sray[6 * (k / 3) + 3 + k % 3] = __ldcs(&P.rad[3 * (start + c0) + k]);
            __syncthreads();
            if (hasA) {
                for (int i = 0; i < m; ++i) {
                    R r[6];
                    if constexpr (sizeof(R) == 8) {
                        const double2* v = reinterpret_cast<const double2*>(sray + 6 * i);
                        const double2 u0 = v[0], u1 = v[1], u2 = v[2];
                        r[0] = u0.x; r[1] = u0.y; r[2] = u1.x; r[3] = u1.y; r[4] = u2.x; r[5] = u2.y;
                    } else {
                        for (int k = 0; k < 6; ++k) r[k] = sray[6 * i + k];
                    }
#pragma unroll
                    for (int q = 0; q < 2; ++q) {
                        if (q == 1 && !hasB) break;
                        const R w = D[q][0] * r[0] + D[q][1] * r[1] + D[q][2] * r[2];
                        if (w > R(0)) {
                            a[q][0] = a[q][0] + r[3] * w;
                            a[q][1] = a[q][1] + r[4] * w;
                            a[q][2] = a[q][2] + r[5] * w;
                        }
                    }
                }
            }
        }
        for (int q = 0; q < 2; ++q) {
            const int tx = q ? txB : txA;
            if (tx >= nt) continue;
            const int y = tx / res, x = tx % res;
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) {
                const double fresh = double(a[q][ch]) * scale;
                const double old = oldTile[((y + 1) * T + (x + 1)) * 3 + ch];
                const double bl = old + (fresh - old) * alpha;
                maxDelta = smax(maxDelta, fabs(bl - old));
                tile[((y + 1) * T + (x + 1)) * 3 + ch] = static_cast<float>(bl);
            }
        }
    }
    R* sdir = reinterpret_cast<R*>(smem_raw);  // 3n
    R* srad = sdir + 3 * n;                    // 3n
    if (kConvChunk == 0) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const V3<double> dir = rayDirection(P, s, i, n);
        sdir[3 * i] = R(dir.x);
        sdir[3 * i + 1] = R(dir.y);
        sdir[3 * i + 2] = R(dir.z);
    }
    for (int k = threadIdx.x; k < 3 * n; k += blockDim.x) srad[k] = __ldcs(&P.rad[3 * start + k]);
    __syncthreads();
    }
    if (kConvChunk > 0) {
    } else if (kConvPerTexel) {
        for (int tx = threadIdx.x; tx < res * res; tx += blockDim.x) {
            const int y = tx / res, x = tx % res;
            const V3<double> dd = octDecode(V2<double>{(x + 0.5) / res, (y + 0.5) / res});
            const R Dx = R(dd.x), Dy = R(dd.y), Dz = R(dd.z);
            R a0 = 0, a1 = 0, a2 = 0;  // each channel summed in the rays' order
            for (int i = 0; i < n; ++i) {
                const R w = Dx * sdir[3 * i] + Dy * sdir[3 * i + 1] + Dz * sdir[3 * i + 2];
                if (w > R(0)) {
                    a0 = a0 + srad[3 * i] * w;
                    a1 = a1 + srad[3 * i + 1] * w;
                    a2 = a2 + srad[3 * i + 2] * w;
                }
            }
            const R acc[3] = {a0, a1, a2};
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) {
                const double fresh = double(acc[ch]) * scale;
                const double old = oldTile[((y + 1) * T + (x + 1)) * 3 + ch];
                const double bl = old + (fresh - old) * alpha;
                maxDelta = smax(maxDelta, fabs(bl - old));
                tile[((y + 1) * T + (x + 1)) * 3 + ch] = static_cast<float>(bl);
            }
        }
    } else
    for (int item = threadIdx.x; item < 3 * res * res; item += blockDim.x) {
        const int tx = item / 3, ch = item % 3;
        const int y = tx / res, x = tx % res;
        const V3<double> dd = octDecode(V2<double>{(x + 0.5) / res, (y + 0.5) / res});
        const R Dx = R(dd.x), Dy = R(dd.y), Dz = R(dd.z);
        R a = 0;
        for (int i = 0; i < n; ++i) {
            const R w = Dx * sdir[3 * i] + Dy * sdir[3 * i + 1] + Dz * sdir[3 * i + 2];
            if (w > R(0)) a = a + srad[3 * i + ch] * w;
        }
        const double fresh = double(a) * scale;
        const double old = oldTile[((y + 1) * T + (x + 1)) * 3 + ch];
        const double bl = old + (fresh - old) * alpha;
        maxDelta = smax(maxDelta, fabs(bl - old));
        tile[((y + 1) * T + (x + 1)) * 3 + ch] = static_cast<float>(bl);
    }
    __syncthreads();
    for (int k = threadIdx.x; k < 4 * res + 4; k += blockDim.x) {
        int dx, dy, sx, sy;
        if (k < 4 * res) {
            const int i = k / 4 + 1, e = k % 4;
            if (e == 0) { dx = i; dy = 0; sx = res + 1 - i; sy = 1; }
            else if (e == 1) { dx = i; dy = res + 1; sx = res + 1 - i; sy = res; }
            else if (e == 2) { dx = 0; dy = i; sx = 1; sy = res + 1 - i; }
            else { dx = res + 1; dy = i; sx = res; sy = res + 1 - i; }
        } else {
            const int e = k - 4 * res;
            if (e == 0) { dx = 0; dy = 0; sx = res; sy = res; }
            else if (e == 1) { dx = res + 1; dy = 0; sx = 1; sy = res; }
            else if (e == 2) { dx = 0; dy = res + 1; sx = res; sy = 1; }
            else { dx = res + 1; dy = res + 1; sx = 1; sy = 1; }
        }
        const float* sp = tile + (sy * T + sx) * 3;
        float* dp = tile + (dy * T + dx) * 3;
        dp[0] = sp[0];
        dp[1] = sp[1];
        dp[2] = sp[2];
    }
    __syncthreads();
    float* dst = P.currAtlas + static_cast<size_t>(g) * T * T * 3;
    const int nf = T * T * 3;
    if ((nf & 3) == 0) {
        const float4* s4 = reinterpret_cast<const float4*>(tile);
        float4* d4 = reinterpret_cast<float4*>(dst);
        for (int k = threadIdx.x; k < nf / 4; k += blockDim.x) d4[k] = s4[k];
    } else {
        for (int k = threadIdx.x; k < nf; k += blockDim.x) dst[k] = tile[k];
    }
    unsigned long long bits = __double_as_longlong(maxDelta);
    for (int o = 16; o > 0; o >>= 1) {
        unsigned long long other = __shfl_xor_sync(kFull, bits, o);
        bits = other > bits ? other : bits;
    }
    if ((threadIdx.x & 31) == 0) redDelta[threadIdx.x >> 5] = bits;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long m = 0;
        for (int w = 0; w < kConvThreads / 32; ++w) m = redDelta[w] > m ? redDelta[w] : m;
        atomicMax(P.maxDeltaBits, m);
        atomicAdd(P.rays, static_cast<unsigned long long>(n));
        atomicAdd(P.updated, 1u);
        pv.reject[g] = 0;  // probe_update.hpp:208-209
        pv.lastFrame[g] = P.frame;
    }
}

template <typename K>
static int persistentBlocks(K kernel, int threads, int cap, size_t smem = 0) {
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kernel, threads, smem);
    int b = sms * (per > 0 ? per : 1);
    return cap > 0 ? min(b, cap) : b;
}

// K1 / K2 launches: with the primitive records staged in shared memory (one CTA
// of StageOcc<R>::threads per SM, the scene's stage bytes of dynamic shared
// memory) when the scene fits, else the register-capped many-CTA form.
template <typename K>
static int stagedBlocks(K kernel, int threads, int bytes) {
    // the opt-in above 48 KB is per kernel (cheap to repeat); one CTA per SM
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    (void)threads;
    return sms;
}
template <typename R, bool ST, int MODE, int PHASE>
static void launchPrimary(const WaveParams<R>& p, int cap, cudaStream_t st) {
    if (p.scene.stageBytes > 0) {
        auto k = k_trace_primary<R, ST, MODE, PHASE, true>;
        const int b = stagedBlocks(k, StageOcc<R>::threads, p.scene.stageBytes);
        k<<<cap > 0 ? min(cap, b) : b, StageOcc<R>::threads, p.scene.stageBytes, st>>>(p);
    } else {
        static int b = persistentBlocks(k_trace_primary<R, ST, MODE, PHASE>, kWaveThreads, 0);
        k_trace_primary<R, ST, MODE, PHASE><<<cap > 0 ? min(cap, b) : b, kWaveThreads, 0, st>>>(p);
    }
}
template <typename R, bool ST, int PHASE>
static void launchShadow(const WaveParams<R>& p, int cap, cudaStream_t st) {
    if (p.scene.stageBytes > 0) {
        auto k = k_trace_shadow<R, ST, PHASE, true>;
        const int b = stagedBlocks(k, StageOcc<R>::threads, p.scene.stageBytes);
        k<<<cap > 0 ? min(cap, b) : b, StageOcc<R>::threads, p.scene.stageBytes, st>>>(p);
    } else {
        static int b = persistentBlocks(k_trace_shadow<R, ST, PHASE>, kWaveThreads, 0);
        k_trace_shadow<R, ST, PHASE><<<cap > 0 ? min(cap, b) : b, kWaveThreads, 0, st>>>(p);
    }
}

template <typename R, bool ST>
static void wavefront(const WaveParams<R>& p, int cap, cudaStream_t st, const cudaEvent_t* ev, long long* launches) {
    if (p.nCand <= 0) return;
    auto mark = [&](int i) {
        if (ev) cudaEventRecord(ev[i], st);
    };
    k_ray_setup<R><<<(p.nCand + 127) / 128, 128, 0, st>>>(p);
    k_ray_scan<R><<<1, kScanThreads, 0, st>>>(p);
    k_probe_ray_setup<R><<<p.nCand, 256, 0, st>>>(p);
    cudaMemsetAsync(p.ctr, 0, (kLightCtr + (p.scene.n_lights > 1 ? p.scene.n_lights : 1)) * sizeof(unsigned long long), st);
    static int b3 = persistentBlocks(k_shade_rays<R, ST, true>, 128, 0);
    static int b3d = persistentBlocks(k_shade_rays<R, ST, false>, 128, 0, 128 * kMvcSlab * sizeof(R));
    static int b3c = persistentBlocks(k_shade_mvc<R, ST>, kMvcThreads, 0, kMvcThreads * kMvcSlab * sizeof(R));
    static int b3t = persistentBlocks(k_shade_tri<R>, 256, 0);
    static int bn = persistentBlocks(k_hit_normals<R>, 128, 0);  // its own occupancy, not K3a's
    // hitAt covers the batch's upper bound of rays; slots past the traced ones stay -1
    cudaMemsetAsync(p.hitAt, 0xff, static_cast<size_t>(p.maxItems) * sizeof(int), st);
    mark(0);
    launchPrimary<R, ST, 0, 0>(p, cap, st);
    mark(1);
    launchPrimary<R, ST, 0, 1>(p, cap, st);
    mark(2);
    compact_hits(p.hitAt, p.hitList, p.ctr + kCtrHits, static_cast<int>(p.maxItems), p.selTemp, p.selTempBytes, st);
    k_hit_normals<R><<<bn, 128, 0, st>>>(p);
    mark(3);
    // the shadow kernels count their events in a separate block of counters
    // (stats + kShadowStats), so the work of K1 and K2 can be told apart
    WaveParams<R> p2 = p;
    if (ST) p2.stats = p.stats + kShadowStats;
    launchShadow<R, ST, 0>(p2, cap, st);
    mark(4);
    launchShadow<R, ST, 1>(p2, cap, st);
    mark(5);
    if (p.debug) {
        k_shade_rays<R, ST, false><<<b3d, 128, 128 * kMvcSlab * sizeof(R), st>>>(p);
    } else {
        k_shade_rays<R, ST, true><<<b3, 128, 0, st>>>(p);
        k_shade_tri<R><<<b3t, 256, 0, st>>>(p);
        k_shade_mvc<R, ST><<<b3c, kMvcThreads, kMvcThreads * kMvcSlab * sizeof(R), st>>>(p);
    }
    mark(6);
    if (!p.debug) {
        const size_t smem = kConvChunk > 0 ? 0 : static_cast<size_t>(2 * p.nRaysFull) * 6 * sizeof(R);
        auto k3 = k_convolve<R, ST>;
        // dynamic + static shared memory above the 48 KB default needs the opt-in
        cudaFuncAttributes fa;
        cudaFuncGetAttributes(&fa, k3);
        if (smem + fa.sharedSizeBytes > 48 * 1024)
            cudaFuncSetAttribute(k3, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        k3<<<p.nCand, kConvThreads, smem, st>>>(p);
    }
    mark(7);
    if (launches) *launches += p.debug ? 10 : 13;
}

// contactGI's per-pixel sum (shading.hpp:686-713): AO from the missed samples,
// occluder radiance (K3a) summed in sample order, probe GI from the resolve.
template <typename R>
__global__ void __launch_bounds__(128) k_contact_combine(WaveParams<R> P) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= static_cast<long long>(P.gw) * P.gh) return;
    const GPix& px = P.gb[i];
    double* out = P.indirect + 3 * i;
    if (!(px.depth < INFINITY)) {
        out[0] = out[1] = out[2] = 0;
        return;
    }
    const V3<double> alb = mk(px.albedo[0], px.albedo[1], px.albedo[2]);
    const V3<double> brdf = alb / kPi;
    const double* re = P.resolved + 3 * i;
    const V3<double> probeGi = brdf * mk(re[0], re[1], re[2]);
    const int nS = P.contactSamples;
    if (nS <= 0 || P.contactRadius <= 0) {
        out[0] = probeGi.x;
        out[1] = probeGi.y;
        out[2] = probeGi.z;
        return;
    }
    int unocc = 0;
    V3<double> occ = mk(0.0, 0.0, 0.0);
    for (int s = 0; s < nS; ++s) {
        const long long rid = i * nS + s;
        if (!P.conv[rid]) {
            ++unocc;
        } else {
            occ = occ + mk(double(P.rad[3 * rid]), double(P.rad[3 * rid + 1]), double(P.rad[3 * rid + 2]));
        }
    }
    const double ao = static_cast<double>(unocc) / nS;
    const V3<double> contact = (alb / kPi) * (kPi / nS) * occ;
    const V3<double> o = probeGi * ao + contact;
    out[0] = o.x;
    out[1] = o.y;
    out[2] = o.z;
}

// Contact GI as a wavefront over (pixel, sample) rays: K1 in contact mode, the
// shared K2 (shadow rays of the compacted hits) and K3a (shadeHit with bounce),
// then the per-pixel combine. Replaces the per-pixel k_contact loop.
template <typename R, bool ST>
static void contactWavefront(const WaveParams<R>& p, cudaStream_t st, long long* launches) {
    cudaMemsetAsync(p.ctr, 0, (kLightCtr + (p.scene.n_lights > 1 ? p.scene.n_lights : 1)) * sizeof(unsigned long long), st);
    cudaMemsetAsync(p.conv, 0, static_cast<size_t>(p.nRaysDirect), st);  // converged flags (K1 sets them)
    if (p.cray) k_contact_setup<R><<<static_cast<int>((p.nRaysDirect + 255) / 256), 256, 0, st>>>(p);
    static int b3 = persistentBlocks(k_shade_rays<R, ST, true>, 128, 0);
    static int b3c = persistentBlocks(k_shade_mvc<R, ST>, kMvcThreads, 0, kMvcThreads * kMvcSlab * sizeof(R));
    static int b3t = persistentBlocks(k_shade_tri<R>, 256, 0);
    static int bn = persistentBlocks(k_hit_normals<R>, 128, 0);  // its own occupancy, not K3a's
    launchPrimary<R, ST, 1, 0>(p, 0, st);
    launchPrimary<R, ST, 1, 1>(p, 0, st);
    compact_hits(p.hitAt, p.hitList, p.ctr + kCtrHits, static_cast<int>(p.maxItems), p.selTemp, p.selTempBytes, st);
    k_hit_normals<R><<<bn, 128, 0, st>>>(p);
    launchShadow<R, ST, 0>(p, 0, st);
    launchShadow<R, ST, 1>(p, 0, st);
    k_shade_rays<R, ST, true><<<b3, 128, 0, st>>>(p);
    k_shade_tri<R><<<b3t, 256, 0, st>>>(p);
    k_shade_mvc<R, ST><<<b3c, kMvcThreads, kMvcThreads * kMvcSlab * sizeof(R), st>>>(p);
    const long long np = static_cast<long long>(p.gw) * p.gh;
    k_contact_combine<R><<<static_cast<int>((np + 127) / 128), 128, 0, st>>>(p);
    if (launches) *launches += p.cray ? 11 : 10;
}

// composeFrame (shading.hpp:480-504) as a wavefront: every geometry pixel becomes a
// "hit" at its G-buffer position/normal, K2 traces its shadow rays (parked far
// phase included), and the combine sums emission + albedo/pi * direct + indirect.
template <typename R>
__global__ void __launch_bounds__(128) k_compose_setup(WaveParams<R> P) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    const long long np = static_cast<long long>(P.gw) * P.gh;
    bool geo = false;
    if (i < np) {
        const GPix& px = P.gb[i];
        geo = px.depth < INFINITY;
        if (geo) {
            HitRec<R> h;
            for (int k = 0; k < 3; ++k) {
                h.p[k] = R(px.world_pos[k]);
                h.n[k] = R(px.normal[k]);
            }
            h.t = R(0);
            h.owner = px.prim;
            h.status = 1;
            P.hits[i] = h;
        }
    }
    const long long slot = parkSlot(P.ctr + kCtrHits, geo);  // compacted pixel list
    if (geo) P.hitList[slot] = static_cast<int>(i);
    V3<R> pos = mk(R(0), R(0), R(0)), nrm = pos;
    if (geo) {
        const GPix& px = P.gb[i];
        pos = mk(R(px.world_pos[0]), R(px.world_pos[1]), R(px.world_pos[2]));
        nrm = mk(R(px.normal[0]), R(px.normal[1]), R(px.normal[2]));
    }
    shadowSetup(P, kFull, geo, static_cast<int>(i), pos, nrm);
}

template <typename R>
__global__ void __launch_bounds__(128) k_compose(WaveParams<R> P) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= static_cast<long long>(P.gw) * P.gh) return;
    const GPix& px = P.gb[i];
    double* out = P.composed + 3 * i;
    if (!(px.depth < INFINITY)) {
        out[0] = P.scene.sky[0];
        out[1] = P.scene.sky[1];
        out[2] = P.scene.sky[2];
        return;
    }
    const V3<double> direct = directLight(P, P.hits[i], static_cast<unsigned long long>(i));
    const V3<double> alb = mk(px.albedo[0], px.albedo[1], px.albedo[2]);
    const V3<double> em = mk(px.emission[0], px.emission[1], px.emission[2]);
    const double* ind = P.resolved + 3 * i;  // the indirect image (input)
    const V3<double> o = (em + (alb / kPi) * direct) + mk(ind[0], ind[1], ind[2]);
    out[0] = o.x;
    out[1] = o.y;
    out[2] = o.z;
}

template <typename R, bool ST>
static void composeWavefront(const WaveParams<R>& p, cudaStream_t st, long long* launches) {
    cudaMemsetAsync(p.ctr, 0, (kLightCtr + (p.scene.n_lights > 1 ? p.scene.n_lights : 1)) * sizeof(unsigned long long), st);
    const long long np = static_cast<long long>(p.gw) * p.gh;
    const int blocks = static_cast<int>((np + 127) / 128);
    k_compose_setup<R><<<blocks, 128, 0, st>>>(p);
    launchShadow<R, ST, 0>(p, 0, st);
    launchShadow<R, ST, 1>(p, 0, st);
    k_compose<R><<<blocks, 128, 0, st>>>(p);
    if (launches) *launches += 4;
}

// Batches of the reference's free functions (sdfgi_trace_rays, sdfgi_soft_shadow,
// sdfgi_shade_hits): the same kernels over caller-given items.
//   rays:   sphereTrace (scene.hpp:391-435) of P.cray records — K1 in direct-ray
//           mode, far phase, normals of the converged hits.
//   shadow: softShadowTrace (scene.hpp:459-476) of the ShadowRay records in light
//           list 0 (ctr[kLightCtr] set by the caller) — K2 and its far phase.
//   shade:  shadeHit (probe_update.hpp:136-149) of the hits in P.hits listed in
//           P.hitList (ctr[kCtrHits] set by the caller): shadow set-up with the
//           given normals, K2, K3a, K3c.
template <typename R>
void launch_batch(const WaveParams<R>& p, int kind, bool stats, cudaStream_t st, long long* launches) {
    const int L = p.scene.n_lights > 1 ? p.scene.n_lights : 1;
    if (kind == 0) {
        cudaMemsetAsync(p.ctr, 0, (kLightCtr + L) * sizeof(unsigned long long), st);
        cudaMemsetAsync(p.hitAt, 0xff, static_cast<size_t>(p.maxItems) * sizeof(int), st);
        if (stats) {
            launchPrimary<R, true, 1, 0>(p, 0, st);
            launchPrimary<R, true, 1, 1>(p, 0, st);
        } else {
            launchPrimary<R, false, 1, 0>(p, 0, st);
            launchPrimary<R, false, 1, 1>(p, 0, st);
        }
        compact_hits(p.hitAt, p.hitList, p.ctr + kCtrHits, static_cast<int>(p.maxItems), p.selTemp, p.selTempBytes,
                     st);
        k_hit_normals<R><<<persistentBlocks(k_hit_normals<R>, 128, 0), 128, 0, st>>>(p);
        if (launches) *launches += 4;
    } else if (kind == 1) {
        if (stats) {
            launchShadow<R, true, 0>(p, 0, st);
            launchShadow<R, true, 1>(p, 0, st);
        } else {
            launchShadow<R, false, 0>(p, 0, st);
            launchShadow<R, false, 1>(p, 0, st);
        }
        if (launches) *launches += 2;
    } else {
        auto ka = stats ? k_shade_rays<R, true, true> : k_shade_rays<R, false, true>;
        auto kc = stats ? k_shade_mvc<R, true> : k_shade_mvc<R, false>;
        k_hit_normals<R, false><<<persistentBlocks(k_hit_normals<R, false>, 128, 0), 128, 0, st>>>(p);
        if (stats) {
            launchShadow<R, true, 0>(p, 0, st);
            launchShadow<R, true, 1>(p, 0, st);
        } else {
            launchShadow<R, false, 0>(p, 0, st);
            launchShadow<R, false, 1>(p, 0, st);
        }
        ka<<<persistentBlocks(ka, 128, 0), 128, 0, st>>>(p);
        k_shade_tri<R><<<persistentBlocks(k_shade_tri<R>, 256, 0), 256, 0, st>>>(p);
        kc<<<persistentBlocks(kc, kMvcThreads, 0, kMvcThreads * kMvcSlab * sizeof(R)), kMvcThreads,
             kMvcThreads * kMvcSlab * sizeof(R), st>>>(p);
        if (launches) *launches += 6;
    }
}

template <typename R>
void launch_compose(const WaveParams<R>& p, bool stats, cudaStream_t st, long long* launches) {
    if (stats)
        composeWavefront<R, true>(p, st, launches);
    else
        composeWavefront<R, false>(p, st, launches);
}

template <typename R>
void launch_contact(const WaveParams<R>& p, bool stats, cudaStream_t st, long long* launches) {
    if (stats)
        contactWavefront<R, true>(p, st, launches);
    else
        contactWavefront<R, false>(p, st, launches);
}

template <typename R>
void launch_wavefront(const WaveParams<R>& p, int cap, bool stats, cudaStream_t st, const cudaEvent_t* ev,
                      long long* launches) {
    if (stats)
        wavefront<R, true>(p, cap, st, ev, launches);
    else
        wavefront<R, false>(p, cap, st, ev, launches);
}

}  // namespace sdfgi_dev
