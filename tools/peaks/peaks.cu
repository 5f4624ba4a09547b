// peaks.cu -- measured roofline denominators for the kernels of this repo on one B200:
//   * tcgen05.mma.cta_group::1 kind::i8 (u8 x u8 -> s32) at M=128, N=256 (the centre-scan /
//     dense-correlation instruction, k_tc.cu), and kind::tf32 at the same shape;
//   * FP32 FFMA and DP4A (u8x4 dot -> u32, the packed R_co walk, k_autocorr.cu) issue peaks.
// MEASURED_PEAKS.json (driver-written) has only the HBM copy and cuBLAS bf16 figures.
//
// One CTA per SM (148), operands resident in shared memory, one elected thread issuing
// back-to-back MMAs into one TMEM accumulator, a commit + wait at the end; time with CUDA
// events over all CTAs.  Ops counted as 2*M*N*K per instruction (K = 32 bytes / element).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o peaks peaks.cu && ./peaks > peaks.json
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x)                                                                   \
    do {                                                                        \
        cudaError_t e_ = (x);                                                   \
        if (e_ != cudaSuccess) {                                                \
            std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
            std::exit(1);                                                       \
        }                                                                       \
    } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// no-swizzle K-major descriptor (LBO between the two 16-byte K halves of a 32-byte K step,
// SBO between 8-row core-matrix groups), sm_100 version bit 46
__device__ __forceinline__ uint64_t make_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return uint64_t((addr >> 4) & 0x3FFF) | (uint64_t((lbo >> 4) & 0x3FFF) << 16) |
           (uint64_t((sbo >> 4) & 0x3FFF) << 32) | (uint64_t(1) << 46);
}
// instruction descriptor: c_format bits 4-5, a/b format bits 7-9 / 10-12, N>>3 at 17,
// M>>4 at 24 (cute/arch/mma_sm100_desc.hpp InstrDescriptor)
__host__ __device__ constexpr uint32_t idesc(int cfmt, int abfmt, int M, int N) {
    return (uint32_t(cfmt) << 4) | (uint32_t(abfmt) << 7) | (uint32_t(abfmt) << 10) |
           (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}

constexpr int kM = 128, kN = 256, kKB = 128;  // K bytes staged: four 32-byte K steps

template <int KIND>  // 0 = kind::i8, 1 = kind::tf32
__global__ void __launch_bounds__(128) k_mma(int iters, const uint8_t* src, int* sink) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_base;
    uint8_t* sA = sm;
    uint8_t* sB = sm + kM * kKB;
    for (int i = threadIdx.x; i < (kM + kN) * kKB; i += blockDim.x) sm[i] = src[i & 4095] & 0x3F;
    asm volatile("fence.proxy.async.shared::cta;");
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(&tmem_base)), "r"(256));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_base;
    if (threadIdx.x == 0) {
        const uint32_t id = KIND == 0 ? idesc(2, 0, kM, kN) : idesc(1, 2, kM, kN);
        const uint32_t sbo = 128 * (kKB / 16);
        for (int it = 0; it < iters; ++it)
#pragma unroll
            for (int s = 0; s < kKB / 32; ++s) {
                const uint64_t ad = make_desc(smem_u32(sA) + 256 * s, 128, sbo);
                const uint64_t bd = make_desc(smem_u32(sB) + 256 * s, 128, sbo);
                const uint32_t acc = (it | s) ? 1u : 0u;
                if (KIND == 0)
                    asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                                 " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                                 ::"r"(tmem), "l"(ad), "l"(bd), "r"(id), "r"(acc));
                else
                    asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                                 " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n"
                                 ::"r"(tmem), "l"(ad), "l"(bd), "r"(id), "r"(acc));
            }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                     ::"r"(smem_u32(&bar)));
    }
    __syncwarp();
    uint32_t ok = 0;
    while (!ok)
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                     " selp.u32 %0, 1, 0, p;\n}\n" : "=r"(ok) : "r"(smem_u32(&bar)), "r"(0));
    asm volatile("tcgen05.fence::after_thread_sync;");
    uint32_t v;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v)
                 : "r"(tmem + (uint32_t((threadIdx.x >> 5) * 32) << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    if (v == 0x7fffffffu) sink[0] = int(v);
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

__global__ void __launch_bounds__(256) k_ffma(int iters, float a, float* sink) {
    float x[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = threadIdx.x * 1e-3f + j;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int r = 0; r < 16; ++r)
#pragma unroll
            for (int j = 0; j < 8; ++j) x[j] = fmaf(x[j], a, 0.5f);
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += x[j];
    if (s == 1234.5f) sink[0] = s;
}

__global__ void __launch_bounds__(256) k_dp4a(int iters, unsigned a, unsigned* sink) {
    unsigned x[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = threadIdx.x + j;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int r = 0; r < 16; ++r)
#pragma unroll
            for (int j = 0; j < 8; ++j) x[j] = __dp4a(x[j] | 0x01010101u, a, x[j]);
    unsigned s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += x[j];
    if (s == 12345u) sink[0] = s;
}

template <class F>
float time_ms(F f) {
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    f();  // warm-up
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
        CK(cudaEventRecord(a));
        f();
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        best = ms < best ? ms : best;
    }
    return best;
}

int main() {
    int dev = 0, sms = 0, clk = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
    uint8_t* src;
    int* sink;
    CK(cudaMalloc(&src, 4096));
    CK(cudaMemset(src, 0x5A, 4096));
    CK(cudaMalloc(&sink, 64));
    const size_t smem = size_t(kM + kN) * kKB;
    CK(cudaFuncSetAttribute(k_mma<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    CK(cudaFuncSetAttribute(k_mma<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    const int iters = 20000;
    const double mmas = double(sms) * iters * (kKB / 32);
    const float ms_i8 = time_ms([&] { k_mma<0><<<sms, 128, smem>>>(iters, src, sink); });
    const float ms_tf = time_ms([&] { k_mma<1><<<sms, 128, smem>>>(iters, src, sink); });
    const double i8_tops = mmas * 2.0 * kM * kN * 32 / (ms_i8 * 1e-3) / 1e12;
    const double tf32_tflops = mmas * 2.0 * kM * kN * 8 / (ms_tf * 1e-3) / 1e12;
    const int fit = 4000, blocks = sms * 8;
    const float ms_f = time_ms([&] { k_ffma<<<blocks, 256>>>(fit, 1.0001f, (float*)sink); });
    const float ms_d = time_ms([&] { k_dp4a<<<blocks, 256>>>(fit, 0x01020304u, (unsigned*)sink); });
    const double lanes = double(blocks) * 256 * fit * 16 * 8;
    const double ffma_tflops = lanes * 2.0 / (ms_f * 1e-3) / 1e12;
    const double dp4a_tops = lanes * 8.0 / (ms_d * 1e-3) / 1e12;  // 4 MACs = 8 ops
    CK(cudaGetLastError());
    std::printf("{\"sms\": %d, \"sm_clock_mhz_attr\": %.0f,\n"
                " \"i8_tops\": %.1f, \"i8_shape\": \"tcgen05.mma cta_group::1 kind::i8 M=128 N=256 K=32\",\n"
                " \"tf32_tflops\": %.1f, \"tf32_shape\": \"tcgen05.mma cta_group::1 kind::tf32 M=128 N=256 K=8\",\n"
                " \"ffma_tflops\": %.1f, \"dp4a_tops\": %.1f,\n"
                " \"ms\": {\"i8\": %.3f, \"tf32\": %.3f, \"ffma\": %.3f, \"dp4a\": %.3f}}\n",
                sms, clk / 1e3, i8_tops, tf32_tflops, ffma_tflops, dp4a_tops, ms_i8, ms_tf, ms_f,
                ms_d);
    return 0;
}
