// Measured on-chip gather ceiling for the Joseph operators (VERDICT r1 item 4 / missing 5).
//
// The f32 Ax takes one bilinear sample per (ray, slice): 4 taps (h, z), (h, z+1), (h+1, z),
// (h+1, z+1) from the z-fastest layout, a warp = 32 detector rows of one column, i.e. each tap
// load of the warp is one contiguous z run starting at an arbitrary float.  This program
// times, on an L1-resident buffer (no L2/HBM traffic), warp loads of the shapes that pattern
// produces and reports them as loads/s and samples/s:
//   line    32 lanes, one aligned 128-byte line per load               (1 wavefront)
//   run2    32 lanes, a 32-float run starting anywhere                 (2 lines)
//   ax4     the Ax sample: 4 loads, runs at (r, z0..z0+31) and (r, z0+1..z0+32) for two rows
//           r and r + pitch                                            (4 loads / sample)
//   lds     shared-memory loads, 32 consecutive floats                  (1 wavefront)
// Usage: gather_peak [iters]  -> one JSON line per pattern.
#include <cstdio>
#include <cstdlib>

#include <cuda_runtime.h>

#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e = (x);                                                                    \
        if (e != cudaSuccess) {                                                                 \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));          \
            exit(1);                                                                            \
        }                                                                                       \
    } while (0)

constexpr int kN = 8192;  // floats: 32 KB, L1-resident next to a 4-CTA/SM working set
constexpr int kPitch = 544;  // row pitch of the ax4 pattern (a padded z run, as the layout)

// Each iteration draws one warp-uniform random start and issues R independent load groups at
// fixed offsets from it (distinct lines), so address arithmetic is ~1 instruction per load and
// the LSU, not issue, is the limit.
constexpr int R = 8;
template <int P>
__global__ void __launch_bounds__(256) k_gather(const float* __restrict__ buf, float* out, int iters) {
    const int lane = threadIdx.x & 31;
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    unsigned s = 2654435761u * (w + 1);
    float acc0 = 0.f, acc1 = 0.f, acc2 = 0.f, acc3 = 0.f;
    for (int it = 0; it < iters; ++it) {
        s = s * 1664525u + 1013904223u;  // warp-uniform pseudo-random start
        if (P == 0) {
            const float* p = buf + (int((s >> 8) & (kN / 2 - 1)) & ~31) + lane;
#pragma unroll
            for (int r = 0; r < R; ++r) acc0 += __ldg(p + r * 512);
        } else if (P == 1) {
            const float* p = buf + (int((s >> 8) & (kN / 2 - 1)) | 1) + lane;  // never 32-aligned: 2 lines
#pragma unroll
            for (int r = 0; r < R; ++r) acc0 += __ldg(p + r * 512);
        } else {
            const float* p = buf + (int((s >> 8) & 511) | 1) + lane;
#pragma unroll
            for (int r = 0; r < R; ++r) {  // R samples: rows 2r, 2r+1 of a kPitch-strided plane
                const float* q = p + 2 * r * kPitch;
                acc0 += __ldg(q);
                acc1 += __ldg(q + 1);
                acc2 += __ldg(q + kPitch);
                acc3 += __ldg(q + kPitch + 1);
            }
        }
    }
    const float a = acc0 + acc1 + acc2 + acc3;
    if (a == 1234.5f) out[0] = a;  // keeps the loads live
}

__global__ void __launch_bounds__(256) k_lds(float* out, int iters) {
    __shared__ float sm[kN / 2];
    for (int i = threadIdx.x; i < kN / 2; i += blockDim.x) sm[i] = float(i);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    unsigned s = 2654435761u * (threadIdx.x / 32 + 1);
    float acc = 0.f, acc1 = 0.f;
    for (int it = 0; it < iters; ++it) {
        s = s * 1664525u + 1013904223u;
        const float* p = sm + (int((s >> 8) & (kN / 4 - 1)) & ~31) + lane;
#pragma unroll
        for (int r = 0; r < R; ++r) (r & 1 ? acc1 : acc) += p[r * 256];
    }
    if (acc + acc1 == 1234.5f) out[0] = acc;
}

int main(int argc, char** argv) {
    const int iters = argc > 1 ? atoi(argv[1]) : 1024;
    int dev = 0, sms = 0, clk = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
    float *buf, *out;
    CK(cudaMalloc(&buf, (kN + 2 * R * kPitch + 1024) * sizeof(float)));
    CK(cudaMemset(buf, 0, (kN + 2 * R * kPitch + 1024) * sizeof(float)));
    CK(cudaMalloc(&out, sizeof(float)));
    const int blocks = sms * 8, threads = 256;  // 64 warps per SM
    const double warps = double(blocks) * threads / 32;
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    const char* names[] = {"line", "run2", "ax4", "lds"};
    for (int p = 0; p < 4; ++p) {
        float best = 1e30f;
        for (int rep = 0; rep < 5; ++rep) {
            CK(cudaEventRecord(e0));
            if (p == 0) k_gather<0><<<blocks, threads>>>(buf, out, iters);
            if (p == 1) k_gather<1><<<blocks, threads>>>(buf, out, iters);
            if (p == 2) k_gather<2><<<blocks, threads>>>(buf, out, iters);
            if (p == 3) k_lds<<<blocks, threads>>>(out, iters);
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            if (rep > 0 && ms < best) best = ms;
        }
        const double loads = warps * iters * R * (p == 2 ? 4 : 1);  // warp-level load instructions
        const double per_s = loads / (best * 1e-3);
        const double samples = p == 2 ? warps * iters * R * 32 / (best * 1e-3) : 0.0;
        printf("{\"pattern\": \"%s\", \"ms\": %.4f, \"warp_loads_per_s\": %.4e, \"warp_loads_per_sm_clk\": %.4f, "
               "\"samples_per_s\": %.4e, \"sms\": %d, \"clock_mhz_attr\": %d}\n",
               names[p], best, per_s, per_s / (double(sms) * clk * 1e3), samples, sms, clk / 1000);
    }
    return 0;
}
