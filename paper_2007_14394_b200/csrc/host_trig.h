// host_trig.h — the transcendental parts of the reference's direction sampling,
// evaluated on the host with the same C library (glibc libm) the reference calls,
// so that every FP64 ray direction on the device is bit-identical to the
// reference's. The device only does the IEEE-exact arithmetic around them
// (+, *, /, sqrt with -fmad=false), which reproduces the reference bit for bit.
//
// glibc's sin/cos/tan are not correctly rounded (measured: ~0.1% of results one ulp
// away from the correctly rounded value), and libdevice's differ from glibc's in
// other places; an ulp in a direction can flip the owner of a hit that ties at a
// box corner. Hence tables:
//   * fibTable      sphericalFibonacci (sampling.hpp:11-17), one table per ray count;
//   * probeQuats    randomRotation's quaternion (rng.hpp:72-90) per probe per pass,
//                   keyed as sampleDirections (sampling.hpp:23-31);
//   * contactLocal  cosineHemisphereDir's r*cos(phi), r*sin(phi) (rng.hpp:58-69) per
//                   Contact GI (pixel, sample), keyed Rng(seed, 0xc0417ff, pixel)
//                   (shading.hpp:451): frame-invariant by the reference's own keying;
//   * tanHalf       Camera::rayDir / project (camera.hpp:30,42).
// The translation unit is compiled with -ffp-contract=off (build.py) so no product
// is fused into an FMA, as in the flag-pinned reference build (oracle/Makefile).
#pragma once

#include <cstdint>
#include <functional>

namespace sdfgi_host {

void fibTable(int n, double* out);  // 3n doubles: x, y, z per sample
// qx, qy, qz, qw per probe (4n doubles); keys[i] = probeKey(cascade level, index)
void probeQuats(uint64_t seed, int frame, bool rotatePerFrame, const uint64_t* keys, int n, double* out);
// lx, ly per (pixel, sample), pixel-major (2 * w * h * samples doubles)
void contactLocal(uint64_t seed, int w, int h, int samples, double* out);
double tanHalf(double fovYDeg);
uint64_t probeKey(int cascadeLevel, int index);  // probe_update.hpp:156-159
// run body(begin, end) over [0, n) on the host pool (the calling thread included)
void parallelFor(long long n, long long grain, const std::function<void(long long, long long)>& body);

}  // namespace sdfgi_host
