// Floor of a BC level step: cost of cluster.sync() for 64 clusters of 2 x 1024
// threads, alone and after a global store / global atomic / L2 load chain.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/cs cluster_sync.cu && /tmp/cs
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

template <int MODE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(1024) k(int iters, int* buf, double* acc, int n) {
    cg::cluster_group cl = cg::this_cluster();
    const int tid = cl.block_rank() * 1024 + threadIdx.x;
    int* mine = buf + (blockIdx.x / 2) * (1 << 20);
    int x = tid;
    for (int it = 0; it < iters; ++it) {
        if (MODE == 1 || MODE == 5) mine[(tid * 97 + it * 131) & ((1 << 20) - 1)] = it;          // store
        if (MODE == 2 || MODE == 6) atomicAdd(&acc[(tid * 7919 + it * 104729) % n], 1.0);        // red
        if (MODE == 3) x = mine[(x * 97 + it) & ((1 << 20) - 1)] & 1023;             // 1 L2 load
        if (MODE == 4) {                                                             // 3 dep loads
            x = mine[(x * 97 + it) & ((1 << 20) - 1)] & 1023;
            x = mine[(x * 31 + it + 7) & ((1 << 20) - 1)] & 1023;
            x = mine[(x * 13 + it + 5) & ((1 << 20) - 1)] & 1023;
        }
        if (MODE >= 5) {  // relaxed arrive (no release of the prior stores) + wait
            asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
        } else {
            cl.sync();
        }
    }
    if (x == -5) buf[0] = x;
}

template <int MODE>
float run(int iters, int* buf, double* acc, int n) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k<MODE><<<128, 1024>>>(10, buf, acc, n);
    cudaEventRecord(a);
    k<MODE><<<128, 1024>>>(iters, buf, acc, n);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms * 1e3f / iters;
}

int main() {
    int* buf;
    double* acc;
    const int n = 24000000;
    cudaMalloc(&buf, 64ll * (1 << 20) * 4);
    cudaMalloc(&acc, size_t(n) * 8);
    cudaMemset(buf, 0, 64ll * (1 << 20) * 4);
    cudaMemset(acc, 0, size_t(n) * 8);
    const int it = 20000;
    printf("cluster.sync only        : %.2f us\n", run<0>(it, buf, acc, n));
    printf("store + sync             : %.2f us\n", run<1>(it, buf, acc, n));
    printf("global red.f64 + sync    : %.2f us\n", run<2>(it, buf, acc, n));
    printf("1 dependent load + sync  : %.2f us\n", run<3>(it, buf, acc, n));
    printf("3 dependent loads + sync : %.2f us\n", run<4>(it, buf, acc, n));
    printf("store + relaxed arrive    : %.2f us\n", run<5>(it, buf, acc, n));
    printf("red + relaxed arrive      : %.2f us\n", run<6>(it, buf, acc, n));
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
