// kernels_f64.cu — FP64 parity-mode instantiations. Compiled with -fmad=false so
// every product and sum rounds separately, matching the reference built with
// -ffp-contract=off (SURVEY §7 hard part 1); sqrt and division are IEEE.
#include "kernels_impl.cuh"
#include "gather_impl.cuh"

namespace sdfgi_dev {

__global__ void __launch_bounds__(128) k_query_points(QueryParams P) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P.n) return;
    Counters c;
    V3<double> p = mk(P.pts[3 * i], P.pts[3 * i + 1], P.pts[3 * i + 2]);
    double init = P.init ? P.init[i] : INFINITY;
    int owner = -1;
    P.outD[i] = query<double, false>(P.scene, p, init, &owner, &c);
    P.outOwner[i] = owner >= 0 ? P.scene.orig[owner] : -1;
}

// Multi-GPU: every rank marks every updated probe of the pass (probe_update.hpp:
// 208-209: rejectHistory = false, lastUpdateFrame = frame for every alive probe the
// pass updated), so the replicated probe state stays identical on every rank
// without exchanging it. ids = the pass's global probe ids (null: 0..n-1).
__global__ void __launch_bounds__(256) k_mark_updated(const int* ids, int n, int frame, const int* alive, int* reject,
                                                      int* lastFrame) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int g = ids ? ids[i] : i;
    if (!alive[g]) return;
    reject[g] = 0;
    lastFrame[g] = frame;
}

// The nearest primitive at each brick centre (exact query; the seed of its cells').
__global__ void __launch_bounds__(128) k_grid_seed(GridBuildParams P, int nbricks) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nbricks) return;
    const int bx = b % P.bdim[0], by = (b / P.bdim[0]) % P.bdim[1], bz = b / (P.bdim[0] * P.bdim[1]);
    const double hb = 0.5 * kBrick * P.h;
    V3<double> c = mk(P.lo[0] + bx * kBrick * P.h + hb, P.lo[1] + by * kBrick * P.h + hb, P.lo[2] + bz * kBrick * P.h + hb);
    Counters cnt;
    int owner = -1;
    query<double, false>(P.scene, c, INFINITY, &owner, &cnt);
    P.bSeed[b] = owner;
}

__global__ void __launch_bounds__(128) k_grid_bound(GridBuildParams P, int ncells) {
    const int cell = blockIdx.x * blockDim.x + threadIdx.x;
    if (cell >= ncells) return;
    const int ix = cell % P.dim[0], iy = (cell / P.dim[0]) % P.dim[1], iz = cell / (P.dim[0] * P.dim[1]);
    V3<double> c = mk(P.lo[0] + (ix + 0.5) * P.h, P.lo[1] + (iy + 0.5) * P.h, P.lo[2] + (iz + 0.5) * P.h);
    Counters cnt;
    // exact whatever the seed (the walk breaks ties by CSR position)
    const int seed = P.bSeed[ix / kBrick + P.bdim[0] * (iy / kBrick + P.bdim[1] * (iz / kBrick))];
    double f = query<double, false>(P.scene, c, INFINITY, nullptr, &cnt, seed);
    double half = 0.5 * sqrt(3.0) * (P.h + 2.0 * P.pad);
    P.U[cell] = f + half * (1.0 + 1e-12) + P.margin;
}

__global__ void __launch_bounds__(128) k_brick_clusters(GridBuildParams P, int nbricks, int fill) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nbricks) return;
    const int bx = b % P.bdim[0], by = (b / P.bdim[0]) % P.bdim[1], bz = b / (P.bdim[0] * P.bdim[1]);
    const int c0[3] = {bx * kBrick, by * kBrick, bz * kBrick};
    int c1[3];
    for (int a = 0; a < 3; ++a) c1[a] = min(c0[a] + kBrick, P.dim[a]);
    // the largest cell reach in the brick, and the union of its padded cells
    double rmax = 0.0;
    for (int z = c0[2]; z < c1[2]; ++z)
        for (int y = c0[1]; y < c1[1]; ++y)
            for (int x = c0[0]; x < c1[0]; ++x)
                rmax = fmax(rmax, fmax(P.U[x + P.dim[0] * (y + P.dim[1] * z)], 0.0));
    const double r = rmax + P.margin;
    const double r2 = isinf(r) ? INFINITY : r * r;
    double lo[3], hi[3];
    for (int a = 0; a < 3; ++a) {
        lo[a] = P.lo[a] + c0[a] * P.h - P.pad;
        hi[a] = P.lo[a] + c1[a] * P.h + P.pad;
    }
    int n = 0;
    const int out = fill ? P.bStart[b] : 0;
    for (int k = 0; k < P.scene.n_clusters; ++k) {
        const DCluster<double>& cl = P.scene.clusters[k];
        bool keep = cl.unbounded != 0;
        if (!keep) {
            double g2 = 0;
            for (int a = 0; a < 3; ++a) {
                double g = fmax(fmax(cl.lo[a] - hi[a], lo[a] - cl.hi[a]), 0.0);
                g2 += g * g;
            }
            keep = g2 <= r2;
        }
        if (keep) {
            if (fill) P.bList[out + n] = k;
            ++n;
        }
    }
    if (!fill) P.bCounts[b] = n;
}

__global__ void __launch_bounds__(128) k_grid_list(GridBuildParams P, int ncells, int fill) {
    const int cell = blockIdx.x * blockDim.x + threadIdx.x;
    if (cell >= ncells) return;
    const int ix = cell % P.dim[0], iy = (cell / P.dim[0]) % P.dim[1], iz = cell / (P.dim[0] * P.dim[1]);
    const double lo[3] = {P.lo[0] + ix * P.h - P.pad, P.lo[1] + iy * P.h - P.pad, P.lo[2] + iz * P.h - P.pad};
    const double hi[3] = {lo[0] + P.h + 2 * P.pad, lo[1] + P.h + 2 * P.pad, lo[2] + P.h + 2 * P.pad};
    const double U = P.U[cell];
    const double r = fmax(U, 0.0) + P.margin;
    const double r2 = isinf(r) ? INFINITY : r * r;
    auto gap2 = [&](const double* blo, const double* bhi) {
        double g2 = 0;
        for (int a = 0; a < 3; ++a) {
            double g = fmax(fmax(blo[a] - hi[a], lo[a] - bhi[a]), 0.0);
            g2 += g * g;
        }
        return g2;
    };
    // Lower bounds of candidate j's SDF: every primitive SDF is an exact signed
    // distance (primitives.hpp:42-65), hence 1-Lipschitz, so SDF_j(p) >=
    // SDF_j(centre) - |p - centre| (the query's bound) >= SDF_j(centre) - (half
    // padded diagonal) (the cell's); the build margin covers the evaluation's
    // rounding (and the FP32 mode's). Much tighter than the distance to j's
    // bounding box, so queries stop earlier.
    const V3<double> centre = mk(0.5 * (lo[0] + hi[0]), 0.5 * (lo[1] + hi[1]), 0.5 * (lo[2] + hi[2]));
    const double half = 0.5 * sqrt(3.0) * (P.h + 2.0 * P.pad);
    // centre value E_j = SDF_j(centre) - margin (what the entry stores: a query at p
    // bounds j by E_j - |p - centre|); E_j - half bounds j over the whole cell
    auto centreValue = [&](int j) { return evalPrim<double>(P.scene.prims[j], centre) - P.margin; };
    // candidate PRIMITIVES: members of nearby clusters (or of an unbounded one) whose
    // bounding box is within r of the cell and whose lower bound does not exceed the
    // cell's upper bound U on the scene SDF — only those can attain (or tie) the
    // minimum at some point of the cell
    // f(j, box bound) -> false: j is not needed exactly (its bound may stay the box
    // bound: the lower bound of j's SDF from its bounding box, valid when the cell
    // centre is outside the box). f returns true to stop the walk.
    const int brick = ix / kBrick + P.bdim[0] * (iy / kBrick + P.bdim[1] * (iz / kBrick));
    auto forEach = [&](auto&& f) {
        for (int i = P.bStart[brick]; i < P.bStart[brick + 1]; ++i) {  // ascending cluster order
            const int k = P.bList[i];
            const DCluster<double>& cl = P.scene.clusters[k];
            if (!cl.unbounded && gap2(cl.lo, cl.hi) > r2) continue;
            for (int j = P.scene.cstart[k]; j < P.scene.cstart[k + 1]; ++j) {
                const double* b = P.primBox + 6 * static_cast<size_t>(j);
                if (!(cl.unbounded || isinf(b[0]) || gap2(b, b + 3) <= r2)) continue;
                // the box bound at the centre (<= SDF_j(centre) when the centre is
                // outside j's box): box distance - margin
                double boxE = -INFINITY;
                if (!isinf(b[0])) {
                    const double gx = fmax(fmax(b[0] - centre.x, centre.x - b[3]), 0.0);
                    const double gy = fmax(fmax(b[1] - centre.y, centre.y - b[4]), 0.0);
                    const double gz = fmax(fmax(b[2] - centre.z, centre.z - b[5]), 0.0);
                    const double g2 = gx * gx + gy * gy + gz * gz;
                    if (g2 > 0) boxE = sqrt(g2) - P.margin;
                }
                if (boxE - half > U) continue;  // its SDF bound (>= the box bound) exceeds U too
                if (f(j, boxE)) return;
            }
        }
    };
    const int K = P.maxList;
    if (!fill) {  // the list length, min(n, K + 1): the walk stops at K + 1
        int n = 0;
        forEach([&](int j, double) {
            if (centreValue(j) - half <= U) ++n;
            return n > K;
        });
        P.counts[cell] = n;
        return;
    }
    // entries sorted by their bound (rounded down into float, so `bound > d` proves
    // the candidate cannot reach or tie d); order does not affect results (queries
    // break ties towards the lowest CSR position). Insertion into the sorted prefix,
    // keeping at most K; the smallest bound pushed out (or never admitted) bounds
    // every omitted candidate and goes to the sentinel.
    const int out = P.start[cell];
    const int slots = P.start[cell + 1] - out;
    const bool truncated = slots == K + 1;
    int2* E = P.entry + out;
    int m = 0;
    float tail = INFINITY;
    forEach([&](int v, double boxE) {
        if (m == K) {
            // a full list: a candidate whose box bound is already no better than the
            // K-th entry's is pushed out without its (costlier) SDF value; the box
            // bound, below its SDF value, still bounds it in the sentinel
            const float kl = __int_as_float(E[K - 1].x);
            const float kb = __double2float_rd(boxE);
            if (!(kb < kl)) {
                tail = fminf(tail, kb);  // (conservative even if v fails the U test)
                return false;
            }
        }
        const double cv = centreValue(v);
        if (!(cv - half <= U)) return false;
        const float kv = __double2float_rd(cv);
        if (m == K) {
            const float kl = __int_as_float(E[K - 1].x);
            if (!(kv < kl)) {
                tail = fminf(tail, kv);
                return false;
            }
            tail = fminf(tail, kl);
            --m;
        }
        int b = m - 1;
        while (b >= 0 && __int_as_float(E[b].x) > kv) {
            E[b + 1] = E[b];
            --b;
        }
        E[b + 1] = make_int2(__float_as_int(kv), v);
        ++m;
        return false;
    });
    if (truncated)  // sentinel: a query still open here walks the cluster hierarchy
        E[m] = make_int2(__float_as_int(tail), -1);
}

// The per-cell records (GridDev::cell): list range and first entry.
__global__ void __launch_bounds__(256) k_grid_cells(const int* start, const int2* entry, int4* cell, int ncells) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= ncells) return;
    const int b = start[c], e = start[c + 1];
    const int2 f = b < e ? entry[b] : make_int2(__float_as_int(INFINITY), -1);
    cell[c] = make_int4(b, e, f.x, f.y);
}
__global__ void __launch_bounds__(256) k_grid_remap(int2* entry, long long n, const int* map) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int2 e = entry[i];
    if (e.y >= 0) entry[i].y = map[e.y];
}

void launch_grid_remap(int2* entry, long long n, const int* map, cudaStream_t st) {
    if (n > 0) k_grid_remap<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(entry, n, map);
}

void launch_grid_cells(const int* start, const int2* entry, int4* cell, int ncells, cudaStream_t st) {
    k_grid_cells<<<(ncells + 255) / 256, 256, 0, st>>>(start, entry, cell, ncells);
}

void launch_grid_seed(const GridBuildParams& p, int nbricks, cudaStream_t st) {
    k_grid_seed<<<(nbricks + 127) / 128, 128, 0, st>>>(p, nbricks);
}

void launch_grid_bound(const GridBuildParams& p, int ncells, cudaStream_t st) {
    k_grid_bound<<<(ncells + 127) / 128, 128, 0, st>>>(p, ncells);
}
void launch_brick_clusters(const GridBuildParams& p, int nbricks, bool fill, cudaStream_t st) {
    k_brick_clusters<<<(nbricks + 127) / 128, 128, 0, st>>>(p, nbricks, fill ? 1 : 0);
}
void launch_grid_list(const GridBuildParams& p, int ncells, bool fill, cudaStream_t st) {
    k_grid_list<<<(ncells + 127) / 128, 128, 0, st>>>(p, ncells, fill ? 1 : 0);
}

void launch_relocate(const RelocParams& p, int nProbes, bool stats, cudaStream_t st) {
    const int blocks = (nProbes + kRelocLanes - 1) / kRelocLanes;
    if (stats)
        k_relocate<true><<<blocks, 128, 0, st>>>(p);
    else
        k_relocate<false><<<blocks, 128, 0, st>>>(p);
}

__global__ void __launch_bounds__(256) k_probes_reset(ProbesView pv, int base, int rx, int ry, int rz, double ox,
                                                     double oy, double oz, double sp) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= rx * ry * rz) return;
    const int ix = i % rx, iy = (i / rx) % ry, iz = i / (rx * ry);
    // restingAt (probe_volume.hpp:37-39), the host's operation order (-fmad=false)
    const double r[3] = {ox + ix * sp, oy + iy * sp, oz + iz * sp};
    const size_t g = static_cast<size_t>(base) + i;
    for (int k = 0; k < 3; ++k) {
        pv.rest[3 * g + k] = r[k];
        pv.pos[3 * g + k] = r[k];
        pv.last[3 * g + k] = r[k];
    }
    pv.alive[g] = 1;
    pv.reject[g] = 1;
    pv.lastFrame[g] = -1;
}
__global__ void __launch_bounds__(256) k_probes_unpack(ProbesView pv, int base, int n, const double* aos) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double* a = aos + 11 * static_cast<size_t>(i);
    const int* ai = reinterpret_cast<const int*>(a + 9);
    const size_t g = static_cast<size_t>(base) + i;
    for (int k = 0; k < 3; ++k) {
        pv.rest[3 * g + k] = a[k];
        pv.pos[3 * g + k] = a[3 + k];
        pv.last[3 * g + k] = a[6 + k];
    }
    pv.reject[g] = ai[0];
    pv.alive[g] = ai[1];
    pv.lastFrame[g] = ai[2];
}
__global__ void __launch_bounds__(256) k_probes_pack(ProbesView pv, int base, int n, double* aos) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double* a = aos + 11 * static_cast<size_t>(i);
    int* ai = reinterpret_cast<int*>(a + 9);
    const size_t g = static_cast<size_t>(base) + i;
    for (int k = 0; k < 3; ++k) {
        a[k] = pv.rest[3 * g + k];
        a[3 + k] = pv.pos[3 * g + k];
        a[6 + k] = pv.last[3 * g + k];
    }
    ai[0] = pv.reject[g];
    ai[1] = pv.alive[g];
    ai[2] = pv.lastFrame[g];
    ai[3] = 0;
}
void launch_probes_reset(ProbesView pv, int base, const int res[3], const double origin[3], double spacing,
                         cudaStream_t st) {
    const int n = res[0] * res[1] * res[2];
    if (n > 0)
        k_probes_reset<<<(n + 255) / 256, 256, 0, st>>>(pv, base, res[0], res[1], res[2], origin[0], origin[1],
                                                         origin[2], spacing);
}
void launch_probes_unpack(ProbesView pv, int base, int n, const double* aos, cudaStream_t st) {
    if (n > 0) k_probes_unpack<<<(n + 255) / 256, 256, 0, st>>>(pv, base, n, aos);
}
void launch_probes_pack(ProbesView pv, int base, int n, double* aos, cudaStream_t st) {
    if (n > 0) k_probes_pack<<<(n + 255) / 256, 256, 0, st>>>(pv, base, n, aos);
}

void launch_mark_updated(const int* ids, int n, int frame, const int* alive, int* reject, int* lastFrame,
                         cudaStream_t st) {
    if (n > 0) k_mark_updated<<<(n + 255) / 256, 256, 0, st>>>(ids, n, frame, alive, reject, lastFrame);
}

void launch_query_points(const QueryParams& p, cudaStream_t st) {
    k_query_points<<<(p.n + 127) / 128, 128, 0, st>>>(p);
}

template void launch_wavefront<double>(const WaveParams<double>&, int, bool, cudaStream_t, const cudaEvent_t*,
                                       long long*);

template void launch_gather<double>(const GatherParams<double>&, int, bool, cudaStream_t);
template void launch_contact<double>(const WaveParams<double>&, bool, cudaStream_t, long long*);
template void launch_compose<double>(const WaveParams<double>&, bool, cudaStream_t, long long*);
template void launch_batch<double>(const WaveParams<double>&, int, bool, cudaStream_t, long long*);

// convolveIrradiance (probe_update.hpp:25-34): E(D) = (4 pi / N) sum max(0, D.d_i) L_i,
// each channel summed in the samples' order; one thread per texel direction.
__global__ void __launch_bounds__(128) k_convolve_batch(const double* sdir, const double* srad, int ns,
                                                        const double* tdir, int nt, double* out) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nt) return;
    const V3<double> D = mk(tdir[3 * t], tdir[3 * t + 1], tdir[3 * t + 2]);
    V3<double> acc = mk(0.0, 0.0, 0.0);
    for (int i = 0; i < ns; ++i) {
        const double w = dot(D, mk(sdir[3 * i], sdir[3 * i + 1], sdir[3 * i + 2]));
        if (w > 0) acc = acc + mk(srad[3 * i], srad[3 * i + 1], srad[3 * i + 2]) * w;
    }
    const V3<double> e = acc * (4.0 * kPi / ns);
    out[3 * t] = e.x;
    out[3 * t + 1] = e.y;
    out[3 * t + 2] = e.z;
}

void launch_convolve_batch(const double* sdir, const double* srad, int ns, const double* tdir, int nt, double* out,
                           cudaStream_t st) {
    if (nt > 0) k_convolve_batch<<<(nt + 127) / 128, 128, 0, st>>>(sdir, srad, ns, tdir, nt, out);
}

// interpolationStencil (probe_volume.hpp:224-310) per point: meta = (cascade slot or
// -1, count, crossCascade, skyFallback, usedMvc)
__global__ void __launch_bounds__(128) k_stencil_batch(ProbeCommon pc, const double* pts, int n, double mvcFrac,
                                                       int* idx, double* w, int* meta) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const V3<double> p = mk(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]);
    const StencilCell sc = stencilCell(pc.cas, pc.nCas, pc.probes, p, mvcFrac);
    const Stencil st = interpolationStencil<double>(pc.cas, pc.nCas, pc.probes, p, mvcFrac);
    for (int k = 0; k < 8; ++k) {
        idx[8 * i + k] = st.count ? st.probe[k] : 0;
        w[8 * i + k] = st.count ? st.w[k] : 0.0;
    }
    int* m = meta + 5 * i;
    m[0] = st.cascade;
    m[1] = st.count;
    m[2] = sc.chosen < 0 ? 1 : (sc.boundary ? 1 : 0);  // no cascade: crossCascade = true (:249-252)
    m[3] = st.sky;
    m[4] = st.usedMvc;
}

void launch_stencil_batch(const ProbeCommon& pc, const double* pts, int n, double mvcFrac, int* idx, double* w,
                          int* meta, cudaStream_t st) {
    if (n > 0) k_stencil_batch<<<(n + 127) / 128, 128, 0, st>>>(pc, pts, n, mvcFrac, idx, w, meta);
}

}  // namespace sdfgi_dev
