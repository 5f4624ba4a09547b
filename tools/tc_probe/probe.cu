// tcgen05 kind::i8 probe: validates the shared-memory descriptor encoding (canonical
// no-swizzle K-major, and the overlapping "Toeplitz" A view with LBO=16 B / SBO=128 B),
// the instruction descriptor for u8 x u8 -> s32, TMEM alloc/ld and commit->mbarrier.
// Standalone: nvcc -gencode arch=compute_100a,code=sm_100a -o probe probe.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <unistd.h>
#include <vector>
#include <chrono>
#include <thread>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t make_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return uint64_t((addr >> 4) & 0x3FFF) | (uint64_t((lbo >> 4) & 0x3FFF) << 16) |
           (uint64_t((sbo >> 4) & 0x3FFF) << 32) | (uint64_t(1) << 46);
}
__host__ __device__ constexpr uint32_t make_idesc_i8(int M, int N) {
    return (2u << 4)                        // D format: s32
           | (0u << 7) | (0u << 10)        // A, B: unsigned 8-bit
           | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ bool mbar_wait(uint64_t* bar, uint32_t phase) {
    uint32_t ok = 0;
    for (long it = 0; it < 20000000L; ++it) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            " selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(phase));
        if (ok) return true;
    }
    return false;
}
__device__ __forceinline__ void mma_i8(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                       uint32_t acc) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
        smem_u32(bar)));
}

// case 0: canonical A (128 x K), case 1: Toeplitz A over a row S (A[a][k] = S[16a+k]).
// B: N x K canonical.  K = 32*ksteps.
__global__ void k_probe(const uint8_t* gA, const uint8_t* gB, int N, int ksteps, int toeplitz,
                        int* out, int* status) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_base;
    const int K = 32 * ksteps;
    uint8_t* sA = sm;                       // up to 128*K or 2048+K bytes
    uint8_t* sB = sm + 128 * 1024;          // N x K canonical
    const int tid = threadIdx.x, warp = tid >> 5;
    // fill smem operands
    if (toeplitz) {
        for (int i = tid; i < 2048 + K; i += blockDim.x) sA[i] = gA[i];
    } else {
        // canonical K-major: (a,k) -> (a/8)*SBO + (a%8)*16 + (k/16)*128 + k%16, SBO = 128*(K/16)
        for (int i = tid; i < 128 * K; i += blockDim.x) {
            const int a = i / K, k = i % K;
            sA[(a / 8) * (128 * (K / 16)) + (a % 8) * 16 + (k / 16) * 128 + (k % 16)] = gA[i];
        }
    }
    for (int i = tid; i < N * K; i += blockDim.x) {
        const int r = i / K, k = i % K;
        sB[(r / 8) * (128 * (K / 16)) + (r % 8) * 16 + (k / 16) * 128 + (k % 16)] = gB[i];
    }
    asm volatile("fence.proxy.async.shared::cta;");
    if (tid == 0) {
        mbar_init(&bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(&tmem_base)),
                     "r"(256));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_base;
    if (tid == 0) {
        const uint32_t idesc = make_idesc_i8(128, N);
        for (int s = 0; s < ksteps; ++s) {
            uint64_t ad = toeplitz ? make_desc(smem_u32(sA) + 32 * s, 16, 128)
                                   : make_desc(smem_u32(sA) + 256 * s, 128, 128 * (K / 16));
            uint64_t bd = make_desc(smem_u32(sB) + 256 * s, 128, 128 * (K / 16));
            mma_i8(tmem, ad, bd, idesc, s > 0 ? 1u : 0u);
        }
        mma_commit(&bar);
    }
    __syncwarp();
    const bool ok = mbar_wait(&bar, 0);
    if (!ok && tid == 0) atomicExch(status, 2);
    asm volatile("tcgen05.fence::after_thread_sync;");
    // lane = tid (warp w reads lanes 32w..32w+31), columns 0..N-1 in chunks of 16
    for (int c0 = 0; c0 < N; c0 += 16) {
        uint32_t v[16];
        const uint32_t addr = tmem + (uint32_t(warp * 32) << 16) + uint32_t(c0);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
              "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
              "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
            : "r"(addr));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        for (int j = 0; j < 16; ++j) out[tid * N + c0 + j] = int(v[j]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}


// Throughput: `iters` x ksteps MMAs on resident operands; one commit at the end.
__global__ void k_bench(int N, int ksteps, int mode, int iters, long long* cycles, int nacc) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_base;
    const int K = 32 * ksteps;
    uint8_t* sA = sm;
    uint8_t* sB = sm + 128 * 1024;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < 100 * 1024; i += blockDim.x) sm[i] = uint8_t(i * 7);
    asm volatile("fence.proxy.async.shared::cta;");
    if (tid == 0) {
        mbar_init(&bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(&tmem_base)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_base;
    if (tid == 0) {
        const uint32_t idesc = make_idesc_i8(128, N);
        int acc_i = 0;
        const long long t0 = clock64();
        for (int it = 0; it < iters; ++it)
            for (int s = 0; s < ksteps; ++s) {
                uint64_t ad;
                if (mode == 0) ad = make_desc(smem_u32(sA) + 256 * s, 128, 128 * (K / 16));  // canonical
                else if (mode == 1) ad = make_desc(smem_u32(sA) + 32 * s, 16, 128);          // Toeplitz
                else ad = make_desc(smem_u32(sA) + 128 * (s / 4) + 0, 8192, 128);             // 8 phase copies
                uint64_t bd = make_desc(smem_u32(sB) + 256 * s, 128, 128 * (K / 16));
                mma_i8(tmem + uint32_t(acc_i * N), ad, bd, idesc, 1u);
                if (++acc_i == nacc) acc_i = 0;
            }
        mma_commit(&bar);
        mbar_wait(&bar, 0);
        cycles[0] = clock64() - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

static void run_bench(int N, int ksteps, int mode, int nacc) {
    long long* d;
    cudaMalloc(&d, 8);
    cudaFuncSetAttribute(k_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    const int iters = 2000;
    k_bench<<<1, 128, 200 * 1024>>>(N, ksteps, mode, iters, d, nacc);
    cudaError_t e = cudaDeviceSynchronize();
    long long c = 0;
    cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    printf("bench N=%3d nacc=%d ksteps=%d mode=%s: %.1f cycles/MMA (%s)\n", N, nacc, ksteps,
           mode == 0 ? "canonical" : (mode == 1 ? "toeplitz " : "phasecopy"),
           double(c) / (iters * ksteps), cudaGetErrorString(e));
    cudaFree(d);
}


// Row-loop mimic: per "row" [optional fence], 3 MMAs (Toeplitz A in ring slot, B window),
// [optional commit to a ring of mbarriers].  Warp-uniform issue with elect.sync.
__global__ void k_rowbench(int N, int rows, int fence, int commit, long long* cycles) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bars[64];
    __shared__ uint32_t tmem_base;
    uint8_t* sA = sm;
    uint8_t* sB = sm + 160 * 1024;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < 190 * 1024; i += blockDim.x) sm[i] = uint8_t(i * 7);
    asm volatile("fence.proxy.async.shared::cta;");
    if (tid == 0) {
        for (int i = 0; i < 64; ++i) mbar_init(&bars[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(&tmem_base)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_base;
    if (warp == 0) {
        const uint32_t idesc = make_idesc_i8(128, N);
        const uint64_t a0 = make_desc(smem_u32(sA), 16, 128);
        const uint64_t b0 = make_desc(smem_u32(sB), 128, 128 * 6);
        const long long t0 = clock64();
        for (int r = 0; r < rows; ++r) {
            if (fence) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            uint64_t ad = a0 + uint64_t((r % 60) * 144);   // 2304-byte slots
            uint64_t bd = b0 + uint64_t((r % 8) * 96);      // 1536-byte entries
            for (int ks = 0; ks < 3; ++ks) {
                asm volatile(
                    "{\n .reg .pred e, acc;\n elect.sync _|e, 0xffffffff;\n setp.ne.b32 acc, 1, 0;\n"
                    " @e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, acc;\n}\n" ::"r"(tmem + 16 * (r % 4)),
                    "l"(ad), "l"(bd), "r"(idesc));
                ad += 2;
                bd += 16;
            }
            if (commit)
                asm volatile(
                    "{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
                    " @e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(
                        smem_u32(&bars[r % 64])));
        }
        asm volatile(
            "{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
            " @e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(
                smem_u32(&bars[63])));
        if (tid == 0) cycles[0] = clock64() - t0;
    }
    __syncthreads();
    // drain: wait until the last commit landed (phase parity depends on counts; just sleep)
    if (tid == 0) { long long t = clock64(); while (clock64() - t < 2000000) {} }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

static void run_rowbench(int N, int fence, int commit) {
    long long* d;
    cudaMalloc(&d, 8);
    cudaFuncSetAttribute(k_rowbench, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    const int rows = 2000;
    k_rowbench<<<1, 128, 200 * 1024>>>(N, rows, fence, commit, d);
    cudaError_t e = cudaDeviceSynchronize();
    long long c = 0;
    cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    printf("rowbench N=%3d fence=%d commit=%d: %.1f cycles/row issue (%s)\n", N, fence, commit,
           double(c) / rows, cudaGetErrorString(e));
    cudaFree(d);
}


// Replays the centre-scan band schedule (sr, m, R rows, Kx=96): per image row dx, one MMA
// chain with N = 16*(k_hi-k_lo+1) into D columns 16*k_lo.., B window at entry(i_top).
__global__ void k_schedbench(int sr, int m, int R, int bands, int commit, long long* cycles, int variant, int variant_spin_sleep) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bars[64];
    __shared__ uint32_t tmem_base;
    // variant >= 10: the production kernel's layout (B at 18 KB, 50-slot A ring after B)
    uint8_t* sA = variant >= 10 ? sm + 18 * 1024 + 96 * 1024 : sm;
    uint8_t* sB = variant >= 10 ? sm + 18 * 1024 : sm + 100 * 1024;
    const int nslot = variant >= 10 ? 40 : 40;
    const int slot_b = variant >= 10 ? 2176 : 2176;
    variant = variant % 10;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < 200 * 1024; i += blockDim.x) sm[i] = uint8_t(i * 7);
    asm volatile("fence.proxy.async.shared::cta;");
    if (tid == 0) {
        for (int i = 0; i < 64; ++i) mbar_init(&bars[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(&tmem_base)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_base;
    long long nmma = 0;
    __shared__ int stop_spin;
    __shared__ int4 tab[256];
    int ntab = 0;
    if (tid == 0) {
        for (int dx = 0; dx < sr * (R - 1) + m; ++dx) {
            const int lo_num = dx - m + 1;
            const int k_lo = lo_num <= 0 ? 0 : (lo_num + sr - 1) / sr;
            const int k_hi = min(R - 1, dx / sr);
            if (k_lo > k_hi) continue;
            const int i_top = dx - sr * k_lo;
            const int entry = (i_top % sr) * ((m + sr - 1) / sr) + (m - 1 - i_top) / sr;
            tab[ntab++] = make_int4(dx, k_lo, k_hi, entry);
        }
        tab[255].x = ntab;
        stop_spin = 0;
    }
    __syncthreads();
    ntab = tab[255].x;
    if (warp > 0) {  // waiters like the production kernel's producer/epilogue warps
        uint32_t ok = 0;
        while (!*(volatile int*)&stop_spin) {
            asm volatile(
                "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                " selp.u32 %0, 1, 0, p;\n}\n"
                : "=r"(ok) : "r"(smem_u32(&bars[62])), "r"(0u) : "memory");
            if (variant_spin_sleep > 0) __nanosleep(variant_spin_sleep);
        }
    }
    if (warp == 0) {
        const uint64_t a0 = make_desc(smem_u32(sA), 16, 128);
        const uint64_t b0 = make_desc(smem_u32(sB), 128, 768);
        const long long t0 = clock64();
        int slot = 0;
        for (int b = 0; b < bands; ++b)
            for (int e = 0; e < ntab; ++e) {
                const int4 row = tab[e];
                const int k_lo = row.y, k_hi = row.z, entry = row.w;
                uint64_t ad = a0 + uint64_t(slot * (slot_b / 16));
                uint64_t bd = b0 + uint64_t(entry * 96);
                const int nfix = variant == 1 || variant == 3 ? R : (k_hi - k_lo + 1);
                const int kfix = variant == 1 || variant == 2 ? 0 : k_lo;
                const uint32_t idesc = make_idesc_i8(128, 16 * nfix);
                const uint32_t d = tmem + (b & 1) * 256 + 16 * kfix;
                for (int ks = 0; ks < 3; ++ks) {
                    asm volatile(
                        "{\n .reg .pred e, acc;\n elect.sync _|e, 0xffffffff;\n setp.ne.b32 acc, 1, 0;\n"
                        " @e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, acc;\n}\n" ::"r"(d),
                        "l"(ad), "l"(bd), "r"(idesc));
                    ad += 2;
                    bd += 16;
                    ++nmma;
                }
                if (commit)
                    asm volatile(
                        "{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
                        " @e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(
                            smem_u32(&bars[slot % 64])));
                slot = (slot + 1) % nslot;
            }
        if (tid == 0) {
            cycles[blockIdx.x * 2] = clock64() - t0;
            cycles[blockIdx.x * 2 + 1] = nmma;
            *(volatile int*)&stop_spin = 1;
        }
    }
    __syncthreads();
    if (tid == 0) { long long t = clock64(); while (clock64() - t < 3000000) {} }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

static void run_sched(int sr, int m, int R, int grid, int commit, int variant, int threads = 128,
                      int sleep_ns = 0) {
    long long* d;
    cudaMalloc(&d, 2 * 8 * 148);
    cudaFuncSetAttribute(k_schedbench, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    const int bands = 5;
    k_schedbench<<<grid, threads, 200 * 1024>>>(sr, m, R, bands, commit, d, variant, sleep_ns);
    cudaError_t e = cudaDeviceSynchronize();
    long long c[2] = {0, 0};
    cudaMemcpy(c, d, 16, cudaMemcpyDeviceToHost);
    const int rows = bands * (sr * (R - 1) + m);
    printf("sched sr=%d m=%d R=%2d threads=%d sleep=%d: %.1f cycles/row, %.1f cycles/MMA (%s)\n", sr, m,
           R, threads, sleep_ns, double(c[0]) / rows, double(c[0]) / c[1], cudaGetErrorString(e));
    cudaFree(d);
}

static int run_case(int N, int ksteps, int toeplitz) {
    const int K = 32 * ksteps;
    const int asz = toeplitz ? 2048 + K : 128 * K;
    std::vector<uint8_t> A(asz), B(N * K);
    srand(1234 + N + ksteps * 7 + toeplitz);
    for (auto& x : A) x = uint8_t(rand() & 255);
    for (auto& x : B) x = uint8_t(rand() & 255);
    uint8_t *dA, *dB;
    int *dO, *dS;
    cudaMalloc(&dA, asz);
    cudaMalloc(&dB, N * K);
    cudaMalloc(&dO, 128 * N * 4);
    cudaMalloc(&dS, 4);
    cudaMemcpy(dA, A.data(), asz, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), N * K, cudaMemcpyHostToDevice);
    cudaMemset(dO, 0xff, 128 * N * 4);
    cudaMemset(dS, 0, 4);
    cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    k_probe<<<1, 128, 200 * 1024>>>(dA, dB, N, ksteps, toeplitz, dO, dS);
    cudaError_t e = cudaGetLastError();
    auto t0 = std::chrono::steady_clock::now();
    while ((e = cudaStreamQuery(0)) == cudaErrorNotReady) {
        if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(10)) {
            printf("case N=%d ks=%d toe=%d: TIMEOUT\n", N, ksteps, toeplitz);
            fflush(stdout);
            _exit(3);
        }
        std::this_thread::sleep_for(std::chrono::milliseconds(1));
    }
    if (e != cudaSuccess) {
        printf("case N=%d ks=%d toe=%d: CUDA error %s\n", N, ksteps, toeplitz, cudaGetErrorString(e));
        _exit(4);
    }
    std::vector<int> O(128 * N);
    int st = 0;
    cudaMemcpy(O.data(), dO, 128 * N * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(&st, dS, 4, cudaMemcpyDeviceToHost);
    long bad = 0;
    int shown = 0;
    for (int a = 0; a < 128; ++a)
        for (int nn = 0; nn < N; ++nn) {
            long ref = 0;
            for (int k = 0; k < K; ++k) {
                const int av = toeplitz ? A[16 * a + k] : A[a * K + k];
                ref += long(av) * B[nn * K + k];
            }
            if (ref != O[a * N + nn]) {
                if (shown++ < 4)
                    printf("  mismatch a=%d n=%d got %d want %ld\n", a, nn, O[a * N + nn], ref);
                ++bad;
            }
        }
    printf("case N=%d ksteps=%d toeplitz=%d: status=%d mismatches=%ld / %d\n", N, ksteps, toeplitz,
           st, bad, 128 * N);
    fflush(stdout);
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(dO);
    cudaFree(dS);
    return bad == 0 && st == 0 ? 0 : 1;
}

int main() {
    int fails = 0;
    fails += run_case(16, 1, 0);
    fails += run_case(16, 1, 1);
    fails += run_case(16, 3, 1);
    fails += run_case(256, 3, 1);
    fails += run_case(64, 2, 0);
    printf("fails=%d\n", fails);
    // variant 0: as scheduled; 1: fixed N=16R, D offset 0; 2: varying N, D offset 0;
    // 3: fixed N=16R, D offset 16*k_lo (N range clipped at 512 columns)
    for (int R : {4, 16}) {
        run_sched(3, 64, R, 148, 1, 10, 32, 0);
        run_sched(3, 64, R, 148, 1, 10, 320, 0);
        run_sched(3, 64, R, 148, 1, 10, 320, 64);
        run_sched(3, 64, R, 148, 1, 10, 320, 256);
    }
    return fails ? 1 : 0;
}
