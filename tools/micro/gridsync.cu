// Microbenchmark: cost of cooperative grid.sync() on this GPU for several grid
// shapes (informs the per-round/per-level overhead of the persistent kernels).
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_sync(int iters, unsigned* sink) {
    cg::grid_group g = cg::this_grid();
    unsigned x = 0;
    for (int i = 0; i < iters; ++i) {
        x += threadIdx.x ^ i;
        g.sync();
    }
    if (x == 0xdeadbeef) *sink = x;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned* sink;
    cudaMalloc(&sink, 4);
    int shapes[][2] = {{1, 256}, {1, 1024}, {2, 256}, {4, 256}, {5, 256}, {8, 256}};
    for (auto& sh : shapes) {
        int per = sh[0], bs = sh[1], occ = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_sync, bs, 0);
        if (occ < per) continue;
        int grid = per * sms, iters = 2000;
        void* args[] = {&iters, &sink};
        cudaLaunchCooperativeKernel((void*)k_sync, grid, bs, args, 0, 0);
        cudaDeviceSynchronize();
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel((void*)k_sync, grid, bs, args, 0, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("grid %d x %d threads: %.3f us per grid.sync\n", grid, bs, ms * 1e3 / iters);
    }
    return 0;
}
