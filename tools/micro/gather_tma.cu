// Microbenchmark: random 8-byte gathers (PageRank's contrib[rev_srcs[e]])
// through the LSU (LDG) versus the TMA engine (cp.async.bulk.tensor
// tile::gather4, 16-byte rows) versus a split of the two.  Sums the gathered
// values per warp so nothing is dead code; checks every variant against LDG.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_tma gather_tma.cu
//   ./gather_tma [n_log2=24] [m=268435456] [skew=3]
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                        \
    do {                                                                             \
        cudaError_t e = (x);                                                         \
        if (e != cudaSuccess) {                                                      \
            printf("%s:%d %s -> %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); \
            exit(1);                                                                 \
        }                                                                            \
    } while (0)

__device__ inline uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

// idx = floor(n * u^skew): skew 1 = uniform, larger = hub-heavy (RMAT-like)
__global__ void k_gen(int64_t m, int32_t n, int skew, int32_t* idx, double* vals) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
         i += (int64_t)gridDim.x * blockDim.x) {
        double u = (mix64(i) >> 11) * 0x1.0p-53, p = u;
        for (int k = 1; k < skew; ++k) p *= u;
        idx[i] = int32_t(p * n) % n;
        if (i < n) vals[i] = double(i % 1000) * 0.001;
    }
}

__device__ inline uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int ITEMS>
__global__ void __launch_bounds__(256) k_ldg(int64_t m, const int32_t* __restrict__ idx,
                                             const double* __restrict__ vals, double* out) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t e0 = t * ITEMS;
    double s = 0.0;
    if (e0 + ITEMS <= m) {
        int32_t j[ITEMS];
#pragma unroll
        for (int k = 0; k < ITEMS; k += 4) {
            int4 q = *reinterpret_cast<const int4*>(idx + e0 + k);
            j[k] = q.x, j[k + 1] = q.y, j[k + 2] = q.z, j[k + 3] = q.w;
        }
        double v[ITEMS];
#pragma unroll
        for (int k = 0; k < ITEMS; ++k) v[k] = __ldg(vals + j[k]);
#pragma unroll
        for (int k = 0; k < ITEMS; ++k) s += v[k];
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) out[t >> 5] = s;
}

// Each warp handles 32*ITEMS edges per tile: every lane issues ITEMS/4
// gather4 copies (4 rows of 16 B each) into the warp's smem buffer; then every
// lane sums its ITEMS values out of shared memory.  LDG_SHARE of every ITEMS
// items per lane are instead loaded through the LSU.
template <int ITEMS, int LDG_ITEMS>
__global__ void __launch_bounds__(128) k_tma(int64_t m, const int32_t* __restrict__ idx,
                                             const double* __restrict__ vals,
                                             const __grid_constant__ CUtensorMap map, double* out) {
    constexpr int TMA_ITEMS = ITEMS - LDG_ITEMS;
    static_assert(TMA_ITEMS % 4 == 0, "");
    __shared__ __align__(128) double buf[4][32 * (TMA_ITEMS > 0 ? TMA_ITEMS : 1) * 4];  // 128 B per gather4
    __shared__ __align__(8) uint64_t bar[4];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t e0 = t * ITEMS;
    double s = 0.0;
    if (lane == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[w])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    const bool ok = e0 + ITEMS <= m;
    int32_t j[ITEMS];
#pragma unroll
    for (int k = 0; k < ITEMS; k += 4) {
        int4 q = ok ? *reinterpret_cast<const int4*>(idx + e0 + k) : make_int4(0, 0, 0, 0);
        j[k] = q.x, j[k + 1] = q.y, j[k + 2] = q.z, j[k + 3] = q.w;
    }
    if (TMA_ITEMS > 0) {
        if (lane == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                             smem_u32(&bar[w])),
                         "r"(uint32_t(32 * TMA_ITEMS * 16))
                         : "memory");
        __syncwarp();
#pragma unroll
        for (int k = 0; k < TMA_ITEMS; k += 4) {
            double* dst = &buf[w][(lane * TMA_ITEMS + k) * 4];
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
                "l"(&map), "r"(0), "r"(j[k] >> 1), "r"(j[k + 1] >> 1), "r"(j[k + 2] >> 1),
                "r"(j[k + 3] >> 1), "r"(smem_u32(&bar[w]))
                : "memory");
        }
    }
    double v[LDG_ITEMS > 0 ? LDG_ITEMS : 1];
#pragma unroll
    for (int k = 0; k < LDG_ITEMS; ++k) v[k] = __ldg(vals + j[TMA_ITEMS + k]);
#pragma unroll
    for (int k = 0; k < LDG_ITEMS; ++k) s += v[k];
    if (TMA_ITEMS > 0) {
        uint32_t done = 0;
        while (!done)
            asm volatile(
                "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
                "selp.u32 %0, 1, 0, p;\n\t}"
                : "=r"(done)
                : "r"(smem_u32(&bar[w]))
                : "memory");
#pragma unroll
        for (int k = 0; k < TMA_ITEMS; ++k) s += buf[w][(lane * TMA_ITEMS + (k & ~3)) * 4 + (k & 3) * 2 + (j[k] & 1)];
    }
    if (!ok) s = 0.0;
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) out[t >> 5] = s;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                             CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                             CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
    const int nlog = argc > 1 ? atoi(argv[1]) : 24;
    const int64_t m = argc > 2 ? atoll(argv[2]) : (int64_t(1) << 28);
    const int skew = argc > 3 ? atoi(argv[3]) : 3;
    const int32_t n = 1 << nlog;
    int32_t* idx;
    double *vals, *out, *ref;
    CK(cudaMalloc(&idx, m * 4 + 64));
    CK(cudaMalloc(&vals, size_t(n) * 8 + 64));
    const int64_t nw = m / 32 + 64;
    CK(cudaMalloc(&out, nw * 8));
    CK(cudaMalloc(&ref, nw * 8));
    k_gen<<<4096, 256>>>(m, n, skew, idx, vals);
    CK(cudaDeviceSynchronize());

    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    CUtensorMap map;
    cuuint64_t gdim[2] = {2, cuuint64_t(n / 2)};
    cuuint64_t gstride[1] = {16};
    int boxrows = argc > 4 ? atoi(argv[4]) : 1;
    cuuint32_t box[2] = {2, cuuint32_t(boxrows)};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = ((EncodeFn)fn)(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, vals, gdim, gstride, box,
                                estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                CU_TENSOR_MAP_L2_PROMOTION_NONE,
                                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode (box rows %d) -> %d\n", boxrows, int(r));

    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    std::vector<double> h_ref(nw), h_out(nw);
    auto bench = [&](const char* name, auto launch, bool is_ref) {
        launch();
        CK(cudaDeviceSynchronize());
        cudaEventRecord(a);
        const int reps = 5;
        for (int i = 0; i < reps; ++i) launch();
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        ms /= reps;
        CK(cudaMemcpy(is_ref ? h_ref.data() : h_out.data(), out, (m / 32) * 8,
                      cudaMemcpyDeviceToHost));
        double maxd = 0;
        if (!is_ref)
            for (int64_t i = 0; i < m / 32 / 8; ++i) {
                double d = fabs(h_out[i] - h_ref[i]);
                if (d > maxd) maxd = d;
            }
        printf("%-28s %.3f ms  %.1f Ggather/s  maxdiff %.3g\n", name, ms, m / (ms * 1e-3) / 1e9,
               maxd);
    };
    const int T = 128;
    bench("ldg items=8", [&] { k_ldg<8><<<(m / 8 + T - 1) / T, T>>>(m, idx, vals, out); }, true);
    bench("ldg items=16", [&] { k_ldg<16><<<(m / 16 + T - 1) / T, T>>>(m, idx, vals, out); }, false);
    bench("tma items=8 (all tma)",
          [&] { k_tma<8, 0><<<(m / 8 + T - 1) / T, T>>>(m, idx, vals, map, out); }, false);
    bench("tma 4 + ldg 4",
          [&] { k_tma<8, 4><<<(m / 8 + T - 1) / T, T>>>(m, idx, vals, map, out); }, false);
    bench("tma 8 + ldg 8",
          [&] { k_tma<16, 8><<<(m / 16 + T - 1) / T, T>>>(m, idx, vals, map, out); }, false);
    bench("tma 4 + ldg 12",
          [&] { k_tma<16, 12><<<(m / 16 + T - 1) / T, T>>>(m, idx, vals, map, out); }, false);
    return 0;
}
