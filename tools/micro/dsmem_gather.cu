// Random 8 B gather throughput per SM: the PageRank pass-A question of whether
// the renumbered graph's hub values (the top ~128K ids hold ~57% of C2's
// gathers) would be served faster from distributed shared memory spread over
// a cluster than through L1/L2.
//   (g) global gathers over an array of S doubles (S = 128K: L2-resident hub
//       table; S = 16M: C2's whole contrib array), through L1
//   (d) DSMEM gathers over a 128K-double table split across a cluster of 8
//       CTAs (16K doubles = 128 KB of shared memory each), loaded once
//   (l) local shared-memory gathers over a 16K-double table (the floor)
// Indices come from a per-thread xorshift (no index traffic); 8 independent
// gathers per loop iteration, as a pass-A lane issues them.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dg dsmem_gather.cu && /tmp/dg
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

constexpr int kThreads = 1024;
constexpr int kSlice = 16384;  // doubles per CTA (128 KB)
constexpr int kCluster = 8;

__device__ __forceinline__ uint32_t xs(uint32_t& s) {
    s ^= s << 13;
    s ^= s >> 17;
    s ^= s << 5;
    return s;
}

__global__ void __launch_bounds__(256) k_global(const double* __restrict__ a, uint32_t mask,
                                                int iters, double* out) {
    uint32_t s = 0x9E3779B9u * (blockIdx.x * blockDim.x + threadIdx.x + 1);
    double acc = 0.0;
    for (int it = 0; it < iters; ++it) {
        double v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = __ldg(a + (xs(s) & mask));
#pragma unroll
        for (int k = 0; k < 8; ++k) acc += v[k];
    }
    if (acc == 1.2345) out[0] = acc;
}

__global__ void __cluster_dims__(kCluster, 1, 1) __launch_bounds__(kThreads)
    k_dsmem(const double* __restrict__ a, int iters, double* out) {
    extern __shared__ double tab[];
    cg::cluster_group cl = cg::this_cluster();
    const int r = int(cl.block_rank());
    for (int i = threadIdx.x; i < kSlice; i += kThreads) tab[i] = a[r * kSlice + i];
    cl.sync();
    const double* peer[kCluster];
#pragma unroll
    for (int q = 0; q < kCluster; ++q) peer[q] = cl.map_shared_rank(tab, q);
    uint32_t s = 0x9E3779B9u * (blockIdx.x * blockDim.x + threadIdx.x + 1);
    double acc = 0.0;
    for (int it = 0; it < iters; ++it) {
        double v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const uint32_t x = xs(s) & (kCluster * kSlice - 1);
            const double* p;
            switch (x >> 14) {  // peer table pointer without local-memory indexing
                case 0: p = peer[0]; break;
                case 1: p = peer[1]; break;
                case 2: p = peer[2]; break;
                case 3: p = peer[3]; break;
                case 4: p = peer[4]; break;
                case 5: p = peer[5]; break;
                case 6: p = peer[6]; break;
                default: p = peer[7]; break;
            }
            v[k] = p[x & (kSlice - 1)];
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) acc += v[k];
    }
    cl.sync();  // no CTA exits while its table is read
    if (acc == 1.2345) out[0] = acc;
}

__global__ void __launch_bounds__(kThreads) k_local(const double* __restrict__ a, int iters,
                                                     double* out) {
    extern __shared__ double tab[];
    for (int i = threadIdx.x; i < kSlice; i += kThreads) tab[i] = a[i];
    __syncthreads();
    uint32_t s = 0x9E3779B9u * (blockIdx.x * blockDim.x + threadIdx.x + 1);
    double acc = 0.0;
    for (int it = 0; it < iters; ++it) {
        double v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = tab[xs(s) & (kSlice - 1)];
#pragma unroll
        for (int k = 0; k < 8; ++k) acc += v[k];
    }
    if (acc == 1.2345) out[0] = acc;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t big = size_t(1) << 24;
    double *a, *out;
    cudaMalloc(&a, big * sizeof(double));
    cudaMalloc(&out, 8);
    cudaMemset(a, 0, big * sizeof(double));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 2000;
    auto report = [&](const char* name, double gathers) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        const double per_clk_sm = gathers / (ms * 1e-3) / sms / 1.965e9;
        printf("%-44s %8.3f ms  %7.1f Ggather/s  %.2f gathers/clk/SM  (%s)\n", name, ms,
               gathers / (ms * 1e-3) / 1e9, per_clk_sm, cudaGetErrorString(cudaGetLastError()));
    };
    for (uint32_t mask : {uint32_t(kCluster * kSlice - 1), uint32_t(big - 1)}) {
        const int grid = sms * 8;
        k_global<<<grid, 256>>>(a, mask, 10, out);
        cudaEventRecord(e0);
        k_global<<<grid, 256>>>(a, mask, iters, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        char name[64];
        snprintf(name, sizeof name, "global, %u doubles (L1/L2)", mask + 1);
        report(name, double(grid) * 256 * iters * 8);
    }
    {
        cudaFuncSetAttribute(k_dsmem, cudaFuncAttributeMaxDynamicSharedMemorySize, kSlice * 8);
        const int grid = (sms / kCluster) * kCluster;
        k_dsmem<<<grid, kThreads, kSlice * 8>>>(a, 10, out);
        cudaEventRecord(e0);
        k_dsmem<<<grid, kThreads, kSlice * 8>>>(a, iters, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        report("DSMEM, 128K doubles over a cluster of 8", double(grid) * kThreads * iters * 8);
    }
    {
        cudaFuncSetAttribute(k_local, cudaFuncAttributeMaxDynamicSharedMemorySize, kSlice * 8);
        const int grid = sms;
        k_local<<<grid, kThreads, kSlice * 8>>>(a, 10, out);
        cudaEventRecord(e0);
        k_local<<<grid, kThreads, kSlice * 8>>>(a, iters, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        report("local shared, 16K doubles", double(grid) * kThreads * iters * 8);
    }
    return 0;
}
