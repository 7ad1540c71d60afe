// Tour-length pass of one warp (warp_tour_length, instance.hpp:120-127) on a 200K-city tour,
// as at the end of a full C5 construction: the tour was just written by the same warp, the
// coordinates are an L2-resident 3.2 MB table. Variants: the engine's pass (U positions per
// lane per pass, two tour loads and two gathers per position), and a pass that loads each
// position once and takes position p+1's coordinates from the next lane (shuffles).
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -fmad=false -I../../paper_1709_03187_b200/csrc ub_tour_length.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <algorithm>
#include "device.cuh"
using namespace pacob200;

template <int U>
__device__ long long len_shfl(const uint32_t* out, uint32_t n, const double2* __restrict__ xy, uint32_t lane) {
    long long len = 0;
    double2 carry = make_double2(0, 0);  // coordinates of the previous pass's last position
    for (uint32_t b = 0; b < n; b += 32 * U) {
        uint32_t c[U];
        double2 x[U];
#pragma unroll
        for (int j = 0; j < U; ++j) { const uint32_t p = b + 32 * j + lane; c[j] = p < n ? out[p] : 0u; }
#pragma unroll
        for (int j = 0; j < U; ++j) x[j] = xy[c[j]];
        double d2[U + 1];
        bool ok = true;
#pragma unroll
        for (int j = 0; j < U; ++j) {
            // position p's successor p + 1: the next lane, or lane 0 of the next group
            double nx = __shfl_down_sync(kFull, x[j].x, 1), ny = __shfl_down_sync(kFull, x[j].y, 1);
            if (j + 1 < U) {
                const double ax = __shfl_sync(kFull, x[j + 1].x, 0), ay = __shfl_sync(kFull, x[j + 1].y, 0);
                if (lane == 31) { nx = ax; ny = ay; }
            }
            const uint32_t p = b + 32 * j + lane;
            const bool has = p + 1 < n && !(j + 1 == U && lane == 31);
            d2[j] = has ? sq_dist(x[j], make_double2(nx, ny)) : 0.0;
            ok &= sqrt_fast_ok(d2[j]);
        }
        // the previous pass's last position to this pass's first (lane 0)
        d2[U] = (b > 0 && lane == 0) ? sq_dist(carry, x[0]) : 0.0;
        ok &= sqrt_fast_ok(d2[U]);
        carry.x = __shfl_sync(kFull, x[U - 1].x, 31); carry.y = __shfl_sync(kFull, x[U - 1].y, 31);
        if (__all_sync(kFull, ok)) {
#pragma unroll
            for (int j = 0; j <= U; ++j) len += (int32_t)__dadd_rn(sqrt_rn_fast(d2[j]), 0.5);
        } else {
#pragma unroll
            for (int j = 0; j <= U; ++j) len += (int32_t)__dadd_rn(__dsqrt_rn(d2[j]), 0.5);
        }
        // zero-length terms add 0 (sqrt(0) + 0.5 truncates to 0)
    }
    // closing edge (n - 1, 0) by lane 0: the last position's coordinates from its lane
    if (lane == 0) len += euc2d(xy[out[n - 1]], xy[out[0]]);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) len += __shfl_xor_sync(kFull, len, off);
    return len;
}

template <int V>
__global__ void k(const uint32_t* tours, uint32_t n, const double2* xy, long long* res, long long* cyc, uint32_t reps) {
    const uint32_t lane = threadIdx.x;
    const uint32_t* out = tours + (size_t)blockIdx.x * n;
    long long s = 0;
    const long long t0 = clock64();
    for (uint32_t r = 0; r < reps; ++r) {
        if (V == 0) s += warp_tour_length(out, n, xy, lane);
        if (V == 1) s += len_shfl<8>(out, n, xy, lane);
        if (V == 2) s += len_shfl<16>(out, n, xy, lane);
    }
    const long long t1 = clock64();
    if (lane == 0) { res[blockIdx.x] = s / reps; cyc[blockIdx.x] = (t1 - t0) / reps; }
}

int main() {
    const uint32_t n = 200000, m = 148;
    std::mt19937 rng(3);
    std::vector<double2> xy(n);
    for (auto& p : xy) p = make_double2((double)(rng() % 10000000), (double)(rng() % 10000000));
    // tours: a locally shuffled identity (consecutive cities near in id = near in space, as Morton)
    std::vector<uint32_t> t((size_t)m * n);
    for (uint32_t a = 0; a < m; ++a) {
        uint32_t* o = t.data() + (size_t)a * n;
        for (uint32_t i = 0; i < n; ++i) o[i] = i;
        for (uint32_t i = 0; i + 64 <= n; i += 64) std::shuffle(o + i, o + i + 64, rng);
    }
    double2* dxy; uint32_t* dt; long long *res, *cyc;
    cudaMalloc(&dxy, n * 16); cudaMemcpy(dxy, xy.data(), n * 16, cudaMemcpyHostToDevice);
    cudaMalloc(&dt, t.size() * 4); cudaMemcpy(dt, t.data(), t.size() * 4, cudaMemcpyHostToDevice);
    cudaMalloc(&res, m * 8); cudaMalloc(&cyc, m * 8);
    for (uint32_t mm : {1u, 148u}) {
        long long ref = -1;
        auto run = [&](auto kern, const char* name) {
            kern<<<mm, 32>>>(dt, n, dxy, res, cyc, 1);
            kern<<<mm, 32>>>(dt, n, dxy, res, cyc, 3);
            cudaDeviceSynchronize();
            std::vector<long long> r(mm), c(mm);
            cudaMemcpy(r.data(), res, mm * 8, cudaMemcpyDeviceToHost);
            cudaMemcpy(c.data(), cyc, mm * 8, cudaMemcpyDeviceToHost);
            if (ref < 0) ref = r[0];
            double mc = 0; for (auto v : c) mc += v; mc /= mm;
            printf("%-28s warps=%-4u %8.2f Mcycles per pass  length %lld %s %s\n", name, mm, mc / 1e6, r[0],
                   r[0] == ref ? "same" : "DIFFERENT", cudaGetErrorString(cudaGetLastError()));
        };
        run(k<0>, "engine (U=8, 2 loads+2 gathers)");
        run(k<1>, "shuffled successor U=8");
        run(k<2>, "shuffled successor U=16");
    }
    return 0;
}
