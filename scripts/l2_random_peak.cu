// Random-access ceiling of the B200 memory system for the sampled update pass's
// access pattern: 8-byte gathers and float2 reductions at uniformly random indices
// of an L2-resident array (the C4 level-0 positions: 1.728 M float2 = 13.8 MB), at
// full occupancy with many independent accesses in flight per thread.  Reports
// accesses per second; apply_kernel's rate (14 such accesses per step) is compared
// against it in DESIGN.md.  Diagnostics only:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/l2peak scripts/l2_random_peak.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t hash(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7feb352dU;
    x ^= x >> 15;
    x *= 0x846ca68bU;
    x ^= x >> 16;
    return x;
}

// MODE 3: gathers from y, reductions to a SECOND array z (never read): the deferred
// form of the negatives (read-only snapshot, write-only delta array).
// MODE 4: the deferred step's mix per 14 accesses: 5 gathers from the snapshot y,
// 5 reductions to the delta z, 2 gathers + 2 reductions on a third, live array w.
template <int MODE>
__global__ void __launch_bounds__(256) probe2(const float2 *__restrict__ y, float2 *z, float2 *w,
                                              uint32_t n, int per_thread, float *sink) {
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    float acc = 0.f;
    for (int k = 0; k < per_thread; k += 8) {
        uint32_t idx[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) idx[u] = hash(tid * 0x9e3779b9u + (uint32_t)(k + u)) % n;
        float2 v[8];
        if (MODE == 3) {
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = __ldg(y + idx[u]);
#pragma unroll
            for (int u = 0; u < 8; ++u) acc += v[u].x + v[u].y;
#pragma unroll
            for (int u = 0; u < 8; ++u)
                atomicAdd(z + idx[(u + 3) & 7], make_float2(1e-9f, acc * 1e-30f));
        } else if (MODE == 5) {   // snapshot reads only: 5 gathers from y, 2 gathers + 7
                                  // reductions on the live array w
#pragma unroll
            for (int u = 0; u < 5; ++u) v[u] = __ldg(y + idx[u]);
#pragma unroll
            for (int u = 5; u < 7; ++u) v[u] = __ldcg(w + idx[u]);
#pragma unroll
            for (int u = 0; u < 7; ++u) acc += v[u].x + v[u].y;
#pragma unroll
            for (int u = 0; u < 7; ++u)
                atomicAdd(w + idx[(u + 3) % 7], make_float2(1e-9f, acc * 1e-30f));
        } else {   // 7 accesses pairs: 5 snapshot/delta, 2 live (one spare index unused)
#pragma unroll
            for (int u = 0; u < 5; ++u) v[u] = __ldg(y + idx[u]);
#pragma unroll
            for (int u = 5; u < 7; ++u) v[u] = __ldcg(w + idx[u]);
#pragma unroll
            for (int u = 0; u < 7; ++u) acc += v[u].x + v[u].y;
#pragma unroll
            for (int u = 0; u < 5; ++u)
                atomicAdd(z + idx[(u + 3) % 5], make_float2(1e-9f, acc * 1e-30f));
#pragma unroll
            for (int u = 5; u < 7; ++u)
                atomicAdd(w + idx[u], make_float2(1e-9f, acc * 1e-30f));
        }
    }
    if (acc == 123.456f) *sink = acc;
}

template <int MODE>   // 0 gather, 1 red, 2 gather + red (1:1)
__global__ void __launch_bounds__(256) probe(float2 *y, uint32_t n, int per_thread, float *sink) {
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    float acc = 0.f;
    for (int k = 0; k < per_thread; k += 8) {
        uint32_t idx[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) idx[u] = hash(tid * 0x9e3779b9u + (uint32_t)(k + u)) % n;
        if (MODE == 0 || MODE == 2) {
            float2 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = __ldcg(y + idx[u]);
#pragma unroll
            for (int u = 0; u < 8; ++u) acc += v[u].x + v[u].y;
        }
        if (MODE == 1 || MODE == 2) {
#pragma unroll
            for (int u = 0; u < 8; ++u) atomicAdd(y + idx[(u + 3) & 7], make_float2(1e-9f, acc * 1e-30f));
        }
    }
    if (acc == 123.456f) *sink = acc;
}

// Size sweep (argv[1] == "sweep"): random 8-byte gathers over arrays from 13.8 MB to
// 512 MB at 2048 threads/SM -- where the rate falls off shows the L2 capacity that
// uniformly shared random data really gets (both dies' SMs read every line).
int sweep() {
    const uint32_t sizes[] = {1728000, 4000000, 6000000, 8000000, 10000000, 12500000,
                              16777216, 67108864};
    float2 *y;
    float *sink;
    cudaMalloc(&y, sizeof(float2) * 67108864u);
    cudaMalloc(&sink, 4);
    cudaMemset(y, 0, sizeof(float2) * 67108864u);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int grid = sms * 8, per_thread = 256;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (uint32_t n : sizes) {
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(a);
            probe<0><<<grid, 256>>>(y, n, per_thread, sink);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            if (rep == 2)
                printf("{\"mode\": \"gather 8B\", \"array_MB\": %.1f, \"ms\": %.3f, "
                       "\"G_accesses_per_s\": %.1f}\n",
                       n * 8.0 / 1e6, ms, (double)grid * 256 * per_thread / (ms * 1e-3) / 1e9);
        }
    }
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

int main(int argc, char **argv) {
    if (argc > 1 && argv[1][0] == 's') return sweep();
    const uint32_t n = 1728000;
    float2 *y;
    float *sink;
    cudaMalloc(&y, sizeof(float2) * n);
    cudaMalloc(&sink, 4);
    cudaMemset(y, 0, sizeof(float2) * n);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int per_thread = 256;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const char *names[3] = {"gather 8B", "float2 red", "gather+red 1:1"};
    for (int blocks_per_sm : {2, 4, 8}) {
        const int grid = sms * blocks_per_sm;
        for (int mode = 0; mode < 3; ++mode) {
            for (int rep = 0; rep < 2; ++rep) {
                cudaEventRecord(a);
                if (mode == 0) probe<0><<<grid, 256>>>(y, n, per_thread, sink);
                if (mode == 1) probe<1><<<grid, 256>>>(y, n, per_thread, sink);
                if (mode == 2) probe<2><<<grid, 256>>>(y, n, per_thread, sink);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms = 0;
                cudaEventElapsedTime(&ms, a, b);
                const double accesses = (double)grid * 256 * per_thread * (mode == 2 ? 2 : 1);
                if (rep == 1)
                    printf("{\"mode\": \"%s\", \"threads_per_sm\": %d, \"ms\": %.3f, "
                           "\"G_accesses_per_s\": %.1f}\n",
                           names[mode], blocks_per_sm * 256, ms, accesses / (ms * 1e-3) / 1e9);
            }
        }
    }
    {   // deferred-negatives mixes over separate arrays
        float2 *z, *w;
        cudaMalloc(&z, sizeof(float2) * n);
        cudaMalloc(&w, sizeof(float2) * n);
        cudaMemset(z, 0, sizeof(float2) * n);
        cudaMemset(w, 0, sizeof(float2) * n);
        for (int blocks_per_sm : {2, 4, 8}) {
            const int grid = sms * blocks_per_sm;
            for (int mode = 3; mode <= 5; ++mode) {
                for (int rep = 0; rep < 2; ++rep) {
                    cudaEventRecord(a);
                    if (mode == 3) probe2<3><<<grid, 256>>>(y, z, w, n, per_thread, sink);
                    else if (mode == 4) probe2<4><<<grid, 256>>>(y, z, w, n, per_thread, sink);
                    else probe2<5><<<grid, 256>>>(y, z, w, n, per_thread, sink);
                    cudaEventRecord(b);
                    cudaEventSynchronize(b);
                    float ms = 0;
                    cudaEventElapsedTime(&ms, a, b);
                    const double accesses = (double)grid * 256 * per_thread * (mode == 3 ? 2.0 : 14.0 / 8.0);
                    if (rep == 1)
                        printf("{\"mode\": \"%s\", \"threads_per_sm\": %d, \"ms\": %.3f, "
                               "\"G_accesses_per_s\": %.1f}\n",
                               mode == 3 ? "gather(A)+red(B) 1:1" : mode == 4 ? "deferred step mix 5gA+5rB+2g2rC" : "snapshot-read mix 5gA+2g7rC",
                               blocks_per_sm * 256, ms, accesses / (ms * 1e-3) / 1e9);
                }
            }
        }
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        printf("error %s\n", cudaGetErrorString(e));
        return 1;
    }
    return 0;
}
