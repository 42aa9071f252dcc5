// select.cu — selectProbesForUpdate (probe_volume.hpp:154-198) on the device.
//
// The reference scores every probe of every cascade, std::stable_sorts the
// candidates (forced first, oldest first among forced, highest priority first
// otherwise) and keeps the first `budget`. Here one thread scores one probe (FP64,
// -fmad=false: the priority rounds exactly as the reference's), the forced and
// the other probes are split by two stable selections, and each part is ordered
// by a stable LSD radix sort (CUB) on a key whose ascending order is the
// reference's descending order — so equal keys keep the candidate order, exactly
// as std::stable_sort does. Only the selected (cascade, index) pairs go back to
// the host (budget x 8 bytes).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>

#include "kernels.cuh"

namespace sdfgi_dev {

// Ascending order of the result = descending order of the double (any sign).
__device__ __forceinline__ unsigned long long descendingKey(double v) {
    unsigned long long u = static_cast<unsigned long long>(__double_as_longlong(v));
    u = (u >> 63) ? ~u : (u | 0x8000000000000000ull);  // ascending-orderable bits
    return ~u;
}

__global__ void __launch_bounds__(256) k_select_score(SelectParams P) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= P.total) return;
    int ci = 0;
    for (int k = 1; k < P.pc.nCas; ++k)
        if (g >= P.pc.cas[k].base) ci = k;
    const CascadeDev& c = P.pc.cas[ci];
    const double* pp = P.pc.probes.pos + 3 * static_cast<size_t>(g);
    const V3<double> d = mk(pp[0], pp[1], pp[2]) - mk(P.camPos[0], P.camPos[1], P.camPos[2]);
    const double dist = length(d);
    const int staleness = P.frame - P.pc.probes.lastFrame[g];
    double angular = 0.25;
    if (dist > 1e-9) angular += 0.75 * smax(0.0, dot(d / dist, mk(P.camFwd[0], P.camFwd[1], P.camFwd[2])));
    double priority = (1.0 / (1.0 + dist / c.spacing)) * angular * static_cast<double>(staleness);
    if (P.pc.probes.reject[g]) priority *= 4.0;
    const bool forced = staleness >= P.forceAge;
    P.forced[g] = forced ? 1 : 0;
    P.other[g] = forced ? 0 : 1;
    P.ids[g] = g;
    // forced: oldest first (staleness >= forceAge >= 1, so 0x7fffffff - staleness >= 0)
    P.keyForced[g] = forced ? static_cast<unsigned int>(0x7fffffff - staleness) : 0u;
    P.keyOther[g] = descendingKey(priority);
}

__global__ void k_select_gather(const unsigned int* keyF, const unsigned long long* keyO, const int* idsF,
                                const int* idsO, const int* counts, unsigned int* outKF, unsigned long long* outKO,
                                int total) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < counts[0]) outKF[i] = keyF[idsF[i]];
    if (i < counts[1]) outKO[i] = keyO[idsO[i]];
    (void)total;
}

// (cascade level, index) pairs of the first n ids of [forced sorted, other sorted].
__global__ void k_select_emit(SelectParams P, const int* idsF, const int* idsO, const int* counts, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int nF = counts[0];
    const int g = i < nF ? idsF[i] : idsO[i - nF];
    int ci = 0;
    for (int k = 1; k < P.pc.nCas; ++k)
        if (g >= P.pc.cas[k].base) ci = k;
    P.outRefs[2 * i] = P.pc.cas[ci].level;
    P.outRefs[2 * i + 1] = g - P.pc.cas[ci].base;
}

size_t select_scratch_bytes(int total) {
    size_t a = 0, b = 0, c = 0;
    cub::DeviceSelect::Flagged(nullptr, a, static_cast<const int*>(nullptr), static_cast<const char*>(nullptr),
                               static_cast<int*>(nullptr), static_cast<int*>(nullptr), total);
    cub::DeviceRadixSort::SortPairs(nullptr, b, static_cast<const unsigned int*>(nullptr),
                                    static_cast<unsigned int*>(nullptr), static_cast<const int*>(nullptr),
                                    static_cast<int*>(nullptr), total);
    cub::DeviceRadixSort::SortPairs(nullptr, c, static_cast<const unsigned long long*>(nullptr),
                                    static_cast<unsigned long long*>(nullptr), static_cast<const int*>(nullptr),
                                    static_cast<int*>(nullptr), total);
    return std::max(a, std::max(b, c));
}

// Returns the number of selected probes (written to P.outRefs on the device).
int launch_select(const SelectParams& P, int budget, cudaStream_t st, long long* launches) {
    const int total = P.total;
    const int blocks = (total + 255) / 256;
    k_select_score<<<blocks, 256, 0, st>>>(P);
    size_t tmp = P.tempBytes;
    // stable splits: forced ids and the others, each in candidate order
    cub::DeviceSelect::Flagged(P.temp, tmp, P.ids, P.forced, P.idsF, P.counts + 0, total, st);
    tmp = P.tempBytes;
    cub::DeviceSelect::Flagged(P.temp, tmp, P.ids, P.other, P.idsO, P.counts + 1, total, st);
    int counts[2] = {0, 0};
    cudaMemcpyAsync(counts, P.counts, sizeof(counts), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    k_select_gather<<<blocks, 256, 0, st>>>(P.keyForced, P.keyOther, P.idsF, P.idsO, P.counts, P.kF, P.kO, total);
    // stable LSD radix sorts (equal keys keep the candidate order)
    if (counts[0] > 0) {
        tmp = P.tempBytes;
        cub::DeviceRadixSort::SortPairs(P.temp, tmp, P.kF, P.kF2, P.idsF, P.idsF2, counts[0], 0, 32, st);
    }
    const int n = budget < total ? budget : total;
    if (counts[0] < n && counts[1] > 0) {
        tmp = P.tempBytes;
        cub::DeviceRadixSort::SortPairs(P.temp, tmp, P.kO, P.kO2, P.idsO, P.idsO2, counts[1], 0, 64, st);
    }
    if (n > 0) k_select_emit<<<(n + 255) / 256, 256, 0, st>>>(P, P.idsF2, P.idsO2, P.counts, n);
    if (launches) *launches += 4 + (counts[0] > 0) + (counts[0] < n && counts[1] > 0) + (n > 0);
    return n;
}

struct NonNegative {
    __device__ __forceinline__ bool operator()(int x) const { return x >= 0; }
};
size_t compact_hits(const int* hitAt, int* hitList, unsigned long long* count, int n, void* temp, size_t tempBytes,
                    cudaStream_t st) {
    size_t need = 0;
    cub::DeviceSelect::If(nullptr, need, hitAt, hitList, count, n, NonNegative(), st);
    if (temp == nullptr) return need;
    cub::DeviceSelect::If(temp, tempBytes, hitAt, hitList, count, n, NonNegative(), st);
    return need;
}

size_t scan_ints(const int* in, int* out, int n, void* temp, size_t tempBytes, cudaStream_t st) {
    size_t need = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, need, in, out, n, st);
    if (temp == nullptr) return need;
    cub::DeviceScan::ExclusiveSum(temp, tempBytes, in, out, n, st);
    return need;
}

}  // namespace sdfgi_dev
