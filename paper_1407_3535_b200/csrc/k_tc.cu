// k_tc.cu -- integer tensor-core correlation (tcgen05.mma kind::i8, sm_100a).
//
// window_dot (detail.hpp:32-41) on 8-bit data is a sum of u8*u8 products; the 5th-gen
// tensor cores compute it exactly (s32 accumulation, m*n*255^2 < 2^31), so the dot that
// feeds the FP64 zncc_at epilogue (detail.hpp:45-51) is bit-identical to the CUDA-core
// path and to the reference.
//
// Formulation.  For an output row r and a 2048-column tile c0, write the column as
// c = c0 + 16a + phi (a < 128 = MMA M, phi < 16).  Then
//     out[r, c] = sum_i sum_t I[r+i, c0 + 16a + t] * T[i, t - phi]     (t < Kx)
// so for image row x = r+i the A operand A_x[a, t] = I[x, c0 + 16a + t] is a Toeplitz
// view of ONE staged image row: a no-swizzle K-major shared-memory descriptor with core
// matrix rows 16 B apart (LBO = 16 B between K halves, SBO = 128 B between 8-row groups)
// reads row a at byte 16a -- no im2col is materialised.  B[(i, phi), t] = T[i, t - phi]
// holds the template rows at the 16 column phases (built once per template).
// A CTA owns a band of R output rows r_k = r0 + sr*k (sr = group height for the centre
// scan, 1 for dense work) and accumulates D[a, (k, phi)] in TMEM; image row x feeds every
// k with 0 <= x - r_k < m in ONE MMA chain whose N = 16 * (#k): the B rows it needs are
// T rows x - r_k, descending by sr, which is one contiguous window when B is stored
// grouped by (row mod sr) in descending row order.
//
// Roles (one CTA per SM, persistent over (band, column tile) tiles):
//   warp 0      producer: cp.async.bulk of image rows (from a 16-byte pitched copy) into a
//               ring of shared-memory slots, and of the B chunk; mbarrier expect_tx.
//   warp 1      TMEM allocation; one elected thread issues the MMAs and commits.
//   warps 2..5  epilogue: tcgen05.ld of the exact s32 dots, FP64 ZNCC, argmax / outputs;
//               re-zero the TMEM buffer and hand it back (double buffered).
//
// Split planes (MODE 3; the north star's "3x" tensor-core variant for non-integer search
// images, e.g. OptA's blurred image).  A pixel v in [0, 256) is cut into three bytes of
// floor(v * 2^16) (tc_split_image); each plane runs the same Toeplitz MMA chains against
// the same B into its own TMEM slots, so  dot_a = D0 + D1/2^8 + D2/2^16  is an EXACT
// integer combination with  0 <= dot_true - dot_a < 2^-16 * sum(T).  kind::i8 slices are
// used instead of 3xTF32 because the s32 accumulation has no rounding at all (a rigorous
// radius; 3xTF32 accumulates in FP32, ~K*2^-24) and the i8 pipe has 4x the TF32 peak.
// The reference's FP64 window_dot (detail.hpp:32-41) rounds in sequence and cannot be
// reproduced by any re-associated sum, so this mode SCREENS: it brackets every rho
// (detail.hpp:45-51 evaluated on the bracketed dot), keeps the largest lower bound and
// lists the few locations whose upper bound reaches it; those are evaluated exactly by the
// FP64 replica (k_list_f64).  Results stay bit-identical to the reference.
#include <algorithm>
#include <cstdio>
#include <vector>

#include "kernels.hpp"
#include "tm_common.cuh"

namespace tmk {

namespace {

Grid to_grid(GridDesc d) {
    return Grid::make(d.er, d.ec, d.h, d.w, d.tr, d.tc, d.ti_lo, d.ti_hi);
}

constexpr int kTcThreads = 320;  // producer, MMA, 8 epilogue warps
constexpr int kTcMaxStages = 64;
constexpr int kTcBarBytes = 2048;  // barriers + TMEM slot at the start of shared memory
constexpr int kTcSchedBytes = 16 * 1024;  // staged row schedule
// Epilogue staging: a warp's 512 output columns of one row (window statistics, visit codes)
// are loaded coalesced and transposed through shared memory to the TMEM layout (lane a owns
// columns 16a..16a+15); 17-element lane pitch = conflict-free both ways.
constexpr int kEpiWarpDoubles = 512 + 32;
constexpr int kEpiBytes = 8 * kEpiWarpDoubles * 8;
constexpr int kTcCols = 2048;  // output columns per tile (M=128 rows x 16 phases)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// shared-memory matrix descriptor, no swizzle, SM100 version field = 1
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return uint64_t((addr >> 4) & 0x3FFF) | (uint64_t((lbo >> 4) & 0x3FFF) << 16) |
           (uint64_t((sbo >> 4) & 0x3FFF) << 32) | (uint64_t(1) << 46);
}

// instruction descriptor: kind::i8, u8 x u8 -> s32, K-major A and B, M = 128
__device__ __forceinline__ uint32_t idesc_i8(int n) {
    return (2u << 4) | (uint32_t(n >> 3) << 17) | (uint32_t(128 >> 4) << 24);
}

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
                 "r"(bytes));
}

__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)));
}

// bounded wait: a protocol error traps (kernel error) instead of hanging the device.
// Waiters off the MMA critical path back off with nanosleep so their polling does not
// steal issue slots from the MMA warp on the same SM sub-partition.
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity, int sleep_ns = 0) {
    uint32_t ok = 0;
    for (long long it = 0;; ++it) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            " selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(ok)
            : "r"(smem_u32(b)), "r"(parity)
            : "memory");
        if (ok) return;
        if (sleep_ns) __nanosleep(sleep_ns);
        if (it > (1ll << 26)) __trap();
    }
}

__device__ __forceinline__ void mbar_wait_t(uint64_t* b, uint32_t parity, long long* acc,
                                            int sleep_ns = 0) {
    if (!acc) {
        mbar_wait(b, parity, sleep_ns);
        return;
    }
    const long long t0 = clock64();
    mbar_wait(b, parity, sleep_ns);
    *acc += clock64() - t0;
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(b))
        : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t addr, uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
          "=r"(v[14]), "=r"(v[15])
        : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void tmem_zero16(uint32_t addr) {
    const uint32_t z = 0;
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(
            addr),
        "r"(z)
        : "memory");
}

template <int MODE>
__global__ void __launch_bounds__(kTcThreads, 1) k_tc_corr(TcJob job, TcTask task, CellH* partials) {
    pdl_wait();
    extern __shared__ __align__(1024) uint8_t sm[];
    const TcPlan& P = job.plan;
    constexpr int NPL = MODE >= 3 ? kTcSplitPlanes : 1;  // image planes per output row
    // a ring stage holds kRows consecutive scheduled image rows (kRows slots of a_slot bytes):
    // one expect_tx, one full-wait and one commit per stage instead of per row
    constexpr int kRows = 4;
    const int kTcStages = P.stages / kRows;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm);
    int4* ssched = reinterpret_cast<int4*>(sm + kTcBarBytes);  // staged row schedule
    uint8_t* sB = sm + P.header;                // B chunk (P.b_smem bytes)
    uint8_t* sA = sB + P.b_smem;                // ring of P.stages image-row slots
    uint64_t* full = bars;                      // [kTcMaxStages]
    uint64_t* empty = bars + kTcMaxStages;      // [kTcMaxStages]
    uint64_t* bfull = bars + 2 * kTcMaxStages;
    uint64_t* bempty = bfull + 1;
    uint64_t* dfull = bfull + 2;                // [2]
    uint64_t* dempty = bfull + 4;               // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bfull + 6);
    __shared__ Cell scratch[8];

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int ntiles = task.nbands * task.ntc;
    // mode 2 with tile flags: tasks whose 16-row x 2048-column blocks hold no survivor are
    // skipped by all three roles alike (same read-only flags)
    auto tile_on = [&](int t) -> bool {
        if (MODE != 2 || !task.tf.p) return true;
        const TcBand bd = task.bands[t / task.ntc];
        const int cblk = t % task.ntc;  // kTcCols == 2048: one flag column per tile
        const int b0 = bd.r0 >> 4, b1 = (bd.r0 + bd.sr * (bd.cnt - 1)) >> 4;
        for (int b = b0; b <= b1; ++b)
            if (task.tf.p[size_t(b) * task.tf.cols + cblk]) return true;
        return false;
    };
    if (task.gate && *task.gate == 0) {  // not selected on the device (survivor_dispatch)
        if (tid == 0) partials[blockIdx.x] = CellH{0.0, -1, -1, 2};
        return;
    }

    if (tid == 0) {
        for (int s = 0; s < kTcStages; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, 1);
        }
        mbar_init(bfull, 1);
        mbar_init(bempty, 1);
        for (int b = 0; b < 2; ++b) {
            mbar_init(dfull + b, 1);
            mbar_init(dempty + b, 256);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    const bool sched_smem = task.sched_total * 16 <= kTcSchedBytes;
    if (sched_smem)
        for (int i = tid; i < task.sched_total; i += blockDim.x) ssched[i] = __ldg(task.sched + i);
    const int4* sched = sched_smem ? ssched : task.sched;
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ============================ producer ============================
        if (lane == 0) {
            long long w_empty = 0, w_bempty = 0;
            const long long t_start = clock64();
            long long* pe = task.dbg ? &w_empty : nullptr;
            long long* pb = task.dbg ? &w_bempty : nullptr;
            uint32_t it = 0;   // ring uses
            uint32_t bl = 0;   // B loads
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
                if (!tile_on(t)) continue;
                const TcBand bd = task.bands[t / task.ntc];
                const int c0 = (t % task.ntc) * kTcCols;
                for (int ch = 0; ch < P.nch; ++ch) {
                    if (P.nch > 1 || bl == 0) {
                        if (bl > 0) mbar_wait_t(bempty, (bl - 1) & 1, pb, 128);
                        const uint32_t bytes = uint32_t(P.b_bytes[ch]);
                        mbar_expect_tx(bfull, bytes);
                        const uint8_t* src = job.bglob + P.b_off[ch];
                        for (uint32_t o = 0; o < bytes; o += 32768)
                            bulk_g2s(sB + o, src + o, min(32768u, bytes - o), bfull);
                        ++bl;
                    }
                    const int4* sc = sched + task.sched_off[ch];
                    const int ns = task.sched_len[ch];
                    for (int pl = 0; pl < NPL; ++pl)
                    for (int e0 = 0; e0 < ns; e0 += kRows) {
                        int dx[kRows];
                        int nr = 0;  // rows are in k_lo order: the valid ones are a prefix
#pragma unroll
                        for (int j = 0; j < kRows; ++j) {
                            const int4 row = e0 + j < ns ? sc[e0 + j] : make_int4(0, 1 << 30, 0, 0);
                            dx[j] = row.x;
                            if (row.y < bd.cnt && nr == j) nr = j + 1;
                        }
                        if (nr == 0) break;
                        const int s = int(it % kTcStages);
                        const uint32_t par = ((it / kTcStages) & 1) ^ 1;
                        mbar_wait_t(empty + s, par, pe, 64);
                        if (task.dbg_flags & 1) {  // timing experiment: no copy
                            mbar_arrive(full + s);
                        } else {
                            mbar_expect_tx(full + s, uint32_t(nr * P.a_bytes));
                            for (int j = 0; j < nr; ++j)
                                bulk_g2s(sA + (size_t(s) * kRows + j) * P.a_slot,
                                         job.imgp + (NPL > 1 ? size_t(pl) * job.plane_stride : size_t(0)) +
                                             size_t(bd.r0 + dx[j]) * job.pitch + c0,
                                         uint32_t(P.a_bytes), full + s);
                        }
                        ++it;
                        if (nr < kRows) break;
                    }
                }
            }
            if (task.dbg) {
                long long* d = task.dbg + blockIdx.x * 8;
                d[0] = clock64() - t_start;
                d[1] = w_empty;
                d[2] = w_bempty;
                d[3] = it;
            }
        }
    } else if (warp == 1) {
        // ============================ MMA issuer ==========================
        // The whole warp runs the (warp-uniform) loop so descriptors live in uniform
        // registers; one elected lane issues.  Descriptors are built once and advanced by
        // adds (16-byte units): A +2 per K-step (32 B), B +16 per K-step (two 128 B core
        // matrices), N field of idesc at bit 17 in units of 8.
        long long w_full = 0, w_dempty = 0, w_bfull = 0, w_issue = 0;
        const long long t_start = clock64();
        long long* pf = task.dbg && lane == 0 ? &w_full : nullptr;
        long long* pd = task.dbg && lane == 0 ? &w_dempty : nullptr;
        long long* pbf = task.dbg && lane == 0 ? &w_bfull : nullptr;
        uint32_t it = 0, bl = 0, tl = 0;
        const uint32_t b_sbo = 128u * uint32_t(P.kx / 16);
        const uint32_t entry16 = uint32_t(P.kx);  // entry bytes / 16
        const uint32_t slot16 = uint32_t(P.a_slot) >> 4;
        const uint64_t a_desc0 = sdesc(smem_u32(sA), 16, 128);
        const uint64_t b_desc0 = sdesc(smem_u32(sB), 128, b_sbo);
        const uint32_t idesc0 = idesc_i8(0);
        const int ksteps = P.kx / 32;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
            if (!tile_on(t)) continue;
            const TcBand bd = task.bands[t / task.ntc];
            const uint32_t buf = tl & 1;
            ++tl;
            mbar_wait_t(dempty + buf, ((tl - 1) >> 1) & 1, pd);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t dbase = tmem + buf * 256;
            for (int ch = 0; ch < P.nch; ++ch) {
                if (P.nch > 1 || bl == 0) {
                    mbar_wait_t(bfull, bl & 1, pbf);
                    ++bl;
                }
                const int4* sc = sched + task.sched_off[ch];
                const int ns = task.sched_len[ch];
                // one ring stage = up to kRows scheduled rows: one wait, their MMAs, one commit
                for (int pl = 0; pl < NPL; ++pl)
                for (int e0 = 0; e0 < ns; e0 += kRows) {
                    int4 rows[kRows];
                    int nr = 0;
#pragma unroll
                    for (int j = 0; j < kRows; ++j) {
                        rows[j] = e0 + j < ns ? sc[e0 + j] : make_int4(0, 1 << 30, 0, 0);
                        if (rows[j].y < bd.cnt && nr == j) nr = j + 1;
                    }
                    if (nr == 0) break;
                    const int s = int(it % kTcStages);
                    const uint32_t par = (it / kTcStages) & 1;
                    if (!(task.dbg_flags & 8)) mbar_wait_t(full + s, par, pf);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const long long t_iss = pf ? clock64() : 0;
#pragma unroll
                    for (int j = 0; j < kRows; ++j) {
                        if (j >= nr) break;
                        const int k_hi = min(rows[j].z, bd.cnt - 1);
                        uint64_t ad = a_desc0 + uint64_t(uint32_t(s * kRows + j) * slot16);
                        uint64_t bdsc = b_desc0 + uint64_t(uint32_t(rows[j].w) * entry16);
                        const uint32_t idesc = idesc0 | (uint32_t(k_hi - rows[j].y + 1) << 18);
                        const uint32_t d =
                            dbase + uint32_t(16 * (rows[j].y + (NPL > 1 ? pl * task.kp : 0)));
                        for (int ks = 0; ks < ksteps; ++ks) {
                            asm volatile(
                                "{\n .reg .pred e, acc;\n elect.sync _|e, 0xffffffff;\n"
                                " setp.ne.b32 acc, 1, 0;\n"
                                " @e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, acc;\n}\n" ::"r"(d),
                                "l"(ad), "l"(bdsc), "r"(idesc));
                            ad += 2;
                            bdsc += 16;
                        }
                    }
                    if (pf) w_issue += clock64() - t_iss;
                    asm volatile(
                        "{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
                        " @e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(
                            smem_u32(empty + s)));
                    ++it;
                    if (nr < kRows) break;
                }
                if (P.nch > 1)
                    asm volatile(
                        "{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
                        " @e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(
                            smem_u32(bempty)));
            }
            asm volatile(
                "{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
                " @e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(
                    smem_u32(dfull + buf)));
        }
        if (task.dbg && lane == 0) {
            long long* dd = task.dbg + blockIdx.x * 8;
            dd[4] = clock64() - t_start;
            dd[5] = w_full;
            dd[6] = w_dempty;
            dd[7] = w_bfull;
            dd[3] = w_issue;  // (overrides the producer's row count slot)
        }
        __syncwarp();
    } else {
        // ============================ epilogue ============================
        // 8 warps: group eg = 0/1 handles output rows k of parity eg; the four warps of a
        // group cover the four TMEM lane quarters (warp w may only touch lanes 32*(w%4)..).
        const int ew = warp - 2;
        const int eg = ew >> 2;
        const int q4 = warp & 3;
        const int a = q4 * 32 + lane;  // MMA row = TMEM lane
        const uint32_t lane_addr = uint32_t(q4 * 32) << 16;
        // zero this group's columns (k of parity eg) of both buffers, hand them over
        for (int b = 0; b < 2; ++b)
            for (int k = eg; k < 16; k += 2) tmem_zero16(tmem + lane_addr + b * 256 + 16 * k);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        mbar_arrive(dempty + 0);
        mbar_arrive(dempty + 1);

        const TStats ts = TStats{job.ts.mu, job.ts.omega, job.ts.mn, job.ts.flat};
        const DevStats st = job.st;
        Cell best = no_cell();
        // dense modes without a rho surface: FP32 pre-test against the thread's exact best
        const bool can_skip = (MODE == 0 || MODE == 2) && !task.out_rho && !(task.dbg_flags & 4);
        bool best_ok = false;
        float best_f = -INFINITY;
        const double tmean = __dmul_rn(ts.mn, ts.mu);  // detail.hpp:49 mn * ts.mu
        uint32_t tl = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
            if (!tile_on(t)) continue;
            const TcBand bd = task.bands[t / task.ntc];
            const int c0 = (t % task.ntc) * kTcCols;
            const uint32_t buf = tl & 1;
            ++tl;
            const int cb = c0 + 16 * a;  // this thread's 16 consecutive columns
            // MODE 1: which of the 16 columns are group centres (constant over the tile)
            uint32_t cmask = 0;
            int tj0 = 0, ph_last = -1;
            if (MODE == 1 || MODE == 4) {
                const int d0 = cb - task.cbase;
                int first = d0 <= 0 ? -d0 : (d0 % task.cstep == 0 ? 0 : task.cstep - d0 % task.cstep);
                tj0 = (cb + first - task.cbase) / task.cstep;
                for (int ph = first, tj = tj0; ph < 16 && tj < task.nc; ph += task.cstep, ++tj)
                    cmask |= 1u << ph;
                // the clipped last group column (irregular centre), stored at tj = tc - 1
                if (task.c_last >= cb && task.c_last < cb + 16) ph_last = task.c_last - cb;
            } else {
                for (int ph = 0; ph < 16; ++ph)
                    if (cb + ph < task.c_lim) cmask |= 1u << ph;
            }
            mbar_wait(dfull + buf, ((tl - 1) >> 1) & 1, 256);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            for (int k = eg; k < bd.cnt && !(task.dbg_flags & 2); k += 2) {
                uint32_t v[16];
                const uint32_t addr = tmem + lane_addr + buf * 256 + uint32_t(16 * k);
                tmem_ld16(addr, v);
                tmem_zero16(addr);
                const int r = bd.r0 + bd.sr * k;
                if (MODE == 3) {
                    // split planes: v = plane 0 (integer parts); planes 1, 2 sit kp and 2 kp
                    // slots further.  dot_a is exact; the bracket of the reference's rho:
                    //   dot_ref in [dot_a (1 - gamma), (dot_a + delta)(1 + gamma)]
                    uint32_t v1[16], v2[16];
                    tmem_ld16(addr + uint32_t(16 * task.kp), v1);
                    tmem_zero16(addr + uint32_t(16 * task.kp));
                    tmem_ld16(addr + uint32_t(32 * task.kp), v2);
                    tmem_zero16(addr + uint32_t(32 * task.kp));
                    const size_t rb = size_t(r) * st.ec + cb;
#pragma unroll
                    for (int ph = 0; ph < 16; ++ph) {
                        if (!((cmask >> ph) & 1u)) continue;
                        const size_t kk = rb + ph;
                        // masked (scan-2 survivors only): the other locations never compete
                        if (st.flat[kk] || (task.mask && task.mask[kk] != 2)) {
                            task.out_ub[kk] = -2.0f;
                            continue;
                        }
                        const double dot_a = double(int(v[ph])) + double(int(v1[ph])) * 0.00390625 +
                                             double(int(v2[ph])) * 0.0000152587890625;
                        const double half = 0.5 * job.scr_delta;
                        const double rad = half + job.scr_gamma * (dot_a + job.scr_delta);
                        const double den = __dmul_rn(ts.omega, st.omega[kk]);
                        const double num = (dot_a + half) - __dmul_rn(tmean, st.mu[kk]);
                        const double rho_m = num / den;
                        const double e = (rad / den) * 1.000001 + 1e-14 + fabs(rho_m) * 1e-14;
                        const double lb = dclamp(rho_m - e, -1.0, 1.0);
                        const double ub = dclamp(rho_m + e, -1.0, 1.0);
                        task.out_ub[kk] = __double2float_ru(ub);
                        const Cell cand = make_cell(r, cb + ph, lb, false);
                        if (better(cand, best)) best = cand;
                    }
                    continue;
                }
                if (MODE == 1 || MODE == 4) {
                    // centres: the exact dot goes to a compact per-group array; the FP64
                    // epilogue runs in k_centre_epi (coalesced statistics loads).  MODE 4
                    // (split planes): dot_a = D0 + D1/2^8 + D2/2^16, exact in FP64; the
                    // bracket is taken by k_split_centre_epi.
                    uint32_t v1[16], v2[16];
                    if (MODE == 4) {
                        tmem_ld16(addr + uint32_t(16 * task.kp), v1);
                        tmem_zero16(addr + uint32_t(16 * task.kp));
                        tmem_ld16(addr + uint32_t(32 * task.kp), v2);
                        tmem_zero16(addr + uint32_t(32 * task.kp));
                    }
                    double* row_out = task.out_rho + size_t(bd.yi0 + k) * task.tc;
                    int tj = tj0;
#pragma unroll
                    for (int ph = 0; ph < 16; ++ph) {
                        double d = double(int(v[ph]));
                        if (MODE == 4)
                            d = d + double(int(v1[ph])) * 0.00390625 +
                                double(int(v2[ph])) * 0.0000152587890625;
                        if (ph == ph_last) row_out[task.tc - 1] = d;
                        if (!((cmask >> ph) & 1u)) continue;
                        row_out[tj++] = d;
                    }
                    continue;
                }
                const size_t rb = size_t(r) * st.ec + cb;
                const size_t rowb = size_t(r) * st.ec;
                const int cw = c0 + 512 * q4;  // the warp's first column (lane: cw + 16*lane)
                double* wd = reinterpret_cast<double*>(sm + kTcBarBytes + kTcSchedBytes) +
                             size_t(ew) * kEpiWarpDoubles;
                uint8_t* wb = reinterpret_cast<uint8_t*>(wd);
                // MODE 2: the visit codes first (coalesced, transposed through shared memory);
                // a warp whose 512 columns hold no survivor skips the row
                uint32_t on2 = cmask;
                bool staged = true;
                if (MODE == 2) {
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        const int idx = j * 32 + lane, col = cw + idx;
                        wb[idx + (idx >> 4)] = col < task.c_lim ? __ldg(task.mask + rowb + col)
                                                                : uint8_t(0);
                    }
                    __syncwarp();
                    on2 = 0u;
#pragma unroll
                    for (int ph = 0; ph < 16; ++ph)
                        if (((cmask >> ph) & 1u) && wb[17 * lane + ph] == 2) on2 |= 1u << ph;
                    __syncwarp();
                    const unsigned nsurv = __reduce_add_sync(0xffffffffu, unsigned(__popc(on2)));
                    if (nsurv == 0u) continue;
                    staged = nsurv >= 96u;  // sparse rows: gather only the survivors' statistics
                }
                uint8_t fl[16];
                double mu[16], om[16];
                if (staged) {
                    // the warp's 512 columns of flat / mu / omega: coalesced loads (all issued
                    // first), then one array at a time through the warp's staging buffer
                    uint8_t gf[16];
                    double gm[16], go[16];
                    // row pointers at this lane's first column: element j is 32*j further
                    const uint8_t* pf = st.flat + rowb + cw + lane;
                    const double* pm = st.mu + rowb + cw + lane;
                    const double* po = st.omega + rowb + cw + lane;
                    const int left = task.c_lim - cw - lane;  // columns j with 32*j < left exist
                    if (left > 480) {  // warp-uniform for all but the last column tile
#pragma unroll
                        for (int j = 0; j < 16; ++j) {
                            gf[j] = __ldg(pf + 32 * j);
                            gm[j] = __ldg(pm + 32 * j);
                            go[j] = __ldg(po + 32 * j);
                        }
                    } else {
#pragma unroll
                        for (int j = 0; j < 16; ++j) {
                            const bool in = 32 * j < left;
                            gf[j] = in ? __ldg(pf + 32 * j) : uint8_t(1);
                            gm[j] = in ? __ldg(pm + 32 * j) : 0.0;
                            go[j] = in ? __ldg(po + 32 * j) : 0.0;
                        }
                    }
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        const int idx = j * 32 + lane;
                        wb[idx + (idx >> 4)] = gf[j];
                    }
                    __syncwarp();
#pragma unroll
                    for (int ph = 0; ph < 16; ++ph) fl[ph] = wb[17 * lane + ph];
                    __syncwarp();
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        const int idx = j * 32 + lane;
                        wd[idx + (idx >> 4)] = gm[j];
                    }
                    __syncwarp();
#pragma unroll
                    for (int ph = 0; ph < 16; ++ph) mu[ph] = wd[17 * lane + ph];
                    __syncwarp();
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        const int idx = j * 32 + lane;
                        wd[idx + (idx >> 4)] = go[j];
                    }
                    __syncwarp();
#pragma unroll
                    for (int ph = 0; ph < 16; ++ph) om[ph] = wd[17 * lane + ph];
                    __syncwarp();
                } else {
                    // all loads first (independent, predicated), then the FP64 epilogues
#pragma unroll
                    for (int ph = 0; ph < 16; ++ph) {
                        const bool on = (on2 >> ph) & 1u;
                        const size_t kk = on ? rb + ph : 0;
                        fl[ph] = on ? st.flat[kk] : uint8_t(1);
                        mu[ph] = on ? st.mu[kk] : 0.0;
                        om[ph] = on ? st.omega[kk] : 0.0;
                    }
                }
                uint32_t need = on2;
                if (can_skip && best_ok) {
                    // argmax only: a location whose FP32 quotient is below the warp's best
                    // (non-degenerate, exact) rho by more than the quotient's error (< 1e-6
                    // for |q| < 2; margin 2e-5) cannot win -- no FP64 division.  Branch-free:
                    // the locations that still need the exact epilogue are collected in a mask
                    uint32_t skip = 0u;
#pragma unroll
                    for (int ph = 0; ph < 16; ++ph) {
                        const double num =
                            __dsub_rn(double(int(v[ph])), __dmul_rn(tmean, mu[ph]));
                        const float q = __fdividef(__double2float_rn(num),
                                                   __double2float_rn(__dmul_rn(ts.omega, om[ph])));
                        const bool sk = fl[ph] != 0 || (fabsf(q) < 2.f && q + 2e-5f < best_f);
                        skip |= (sk ? 1u : 0u) << ph;
                    }
                    need &= ~skip;
                }
                if (need)
#pragma unroll
                for (int ph = 0; ph < 16; ++ph) {
                    if (!((need >> ph) & 1u)) continue;
                    const int c = cb + ph;
                    const bool wflat = fl[ph];
                    const double rho = zncc_epilogue(double(int(v[ph])), ts, mu[ph], om[ph], wflat);
                    const bool deg = ts.flat || wflat;
                    if (task.out_rho) task.out_rho[rb + ph] = rho;
                    const Cell cand = make_cell(r, c, rho, deg);
                    if (better(cand, best)) {
                        best = cand;
                        if (!deg) {
                            best_ok = true;
                            best_f = fmaxf(best_f, __double2float_rd(rho));
                        }
                    }
                }
                if (can_skip) {
                    // the pre-test limit is shared by the warp after every row (any exact
                    // non-degenerate rho found so far bounds the final maximum from below)
                    const int bits = __float_as_int(best_ok ? best_f : -INFINITY);
                    const int key = bits >= 0 ? bits : bits ^ 0x7fffffff;  // order-preserving
                    const int top = __reduce_max_sync(0xffffffffu, key);
                    const float lim = __int_as_float(top >= 0 ? top : top ^ 0x7fffffff);
                    if (lim > -INFINITY) {
                        best_ok = true;
                        best_f = lim;
                    }
                }
            }
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            mbar_arrive(dempty + buf);
        }
        // block best over the 8 epilogue warps
        best = warp_best(best);
        if (lane == 0) scratch[ew] = best;
        asm volatile("bar.sync 1, 256;" ::: "memory");
        if (ew == 0 && lane == 0) {
            Cell b = scratch[0];
            for (int w = 1; w < 8; ++w)
                if (better(scratch[w], b)) b = scratch[w];
            partials[blockIdx.x] = CellH{b.rho, b.row, b.col, b.flags};
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

// B chunk layout: entry e (16 rows = the 16 column phases of one template row i) x Kx
// bytes, canonical no-swizzle K-major: byte (row rho, t) at
// (rho/8)*SBO + (rho%8)*16 + (t/16)*128 + t%16, SBO = 128*Kx/16.
__global__ void k_tc_build_b(const float* __restrict__ tf, int npad, int m, int n, TcPlan P,
                             uint8_t* __restrict__ out, const int* __restrict__ gate) {
    pdl_wait();
    if (gate && !*gate) return;  // the pass this B feeds is gated off (survivor_dispatch)
    const int ch = blockIdx.y;
    const int i0 = P.i0[ch], i1 = P.i1[ch];
    const int entries = i1 - i0;
    uint8_t* o = out + P.b_off[ch];
    const int sbo = 128 * (P.kx / 16);
    const int nk16 = P.kx / 16;
    // one thread per 16-byte run of one (entry, phase) row: the run is contiguous in the
    // core-matrix layout ((t/16)*128 + t%16) and in the template row, one 16-byte store
    const unsigned total = unsigned(entries) * 16u * unsigned(nk16);
    for (unsigned idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += gridDim.x * blockDim.x) {
        const unsigned eph = idx / unsigned(nk16);
        const int t16 = int(idx - eph * unsigned(nk16));
        const int e = int(eph >> 4), ph = int(eph & 15u);
        // entry e -> (class, position) -> template row i
        int cls = 0;
        while (cls + 1 < P.sr && P.cls_off[ch][cls + 1] <= e) ++cls;
        const int i = P.cls_max[ch][cls] - P.sr * (e - P.cls_off[ch][cls]);
        const bool row_ok = i >= i0 && i < i1;
        const float* trow = tf + size_t(row_ok ? i : 0) * npad;
        unsigned w[4] = {0u, 0u, 0u, 0u};
#pragma unroll
        for (int bb = 0; bb < 16; ++bb) {
            const int j = t16 * 16 + bb - ph;
            const unsigned v = (row_ok && j >= 0 && j < n) ? unsigned(trow[j]) : 0u;
            w[bb >> 2] |= v << (8 * (bb & 3));
        }
        const int row = e * 16 + ph;
        *reinterpret_cast<uint4*>(o + size_t(row / 8) * sbo + (row % 8) * 16 + t16 * 128) =
            make_uint4(w[0], w[1], w[2], w[3]);
    }
}

__global__ void k_tc_pitch(const uint8_t* __restrict__ img, int p, int q, uint8_t* __restrict__ out,
                           int pitch, int rows) {
    const int cpr = pitch >> 4;  // chunks per row
    const size_t total = size_t(rows) * cpr;
    const bool vec = (q & 15) == 0;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < total;
         i += size_t(gridDim.x) * blockDim.x) {
        const int r = int(i / cpr), c = int(i - size_t(r) * cpr) << 4;
        uint4 v = make_uint4(0u, 0u, 0u, 0u);
        if (r < p && c < q) {
            const uint8_t* src = img + size_t(r) * q + c;
            if (vec) {
                v = __ldg(reinterpret_cast<const uint4*>(src));
            } else {
                unsigned w[4] = {0u, 0u, 0u, 0u};
                const int nb = min(16, q - c);
                for (int b = 0; b < nb; ++b) w[b >> 2] |= unsigned(__ldg(src + b)) << (8 * (b & 3));
                v = make_uint4(w[0], w[1], w[2], w[3]);
            }
        }
        *reinterpret_cast<uint4*>(out + size_t(r) * pitch + c) = v;
    }
}

// floor(v * 2^16) of a non-integer image cut into three byte planes (16-byte pitched, zero
// padded like k_tc_pitch): plane 0 = integer part, planes 1, 2 = the next two bytes.
__global__ void k_tc_split(const double* __restrict__ img, int p, int q, uint8_t* __restrict__ out,
                           int pitch, int rows, size_t plane_stride, int* __restrict__ bad) {
    const int cpr = pitch >> 4;
    const size_t total = size_t(rows) * cpr;
    int any_bad = 0;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < total;
         i += size_t(gridDim.x) * blockDim.x) {
        const int r = int(i / cpr), c = int(i - size_t(r) * cpr) << 4;
        unsigned w[3][4] = {};
        if (r < p && c < q) {
            const double* src = img + size_t(r) * q + c;
            const int nb = min(16, q - c);
            for (int b = 0; b < nb; ++b) {
                const double v = __ldg(src + b);
                if (!(v >= 0.0 && v < 256.0)) {
                    any_bad = 1;
                    continue;
                }
                const unsigned u = __double2uint_rd(v * 65536.0);  // exact scaling
                w[0][b >> 2] |= (u >> 16) << (8 * (b & 3));
                w[1][b >> 2] |= ((u >> 8) & 255u) << (8 * (b & 3));
                w[2][b >> 2] |= (u & 255u) << (8 * (b & 3));
            }
        }
#pragma unroll
        for (int pl = 0; pl < 3; ++pl)
            *reinterpret_cast<uint4*>(out + pl * plane_stride + size_t(r) * pitch + c) =
                make_uint4(w[pl][0], w[pl][1], w[pl][2], w[pl][3]);
    }
    if (any_bad) atomicOr(bad, 1);
}

// Locations whose upper bound reaches the largest lower bound (any order: the exact
// evaluation that follows reduces with better_candidate's total order).
__global__ void k_tc_screen_compact(const float* __restrict__ ub, int er, int ec,
                                    const CellH* __restrict__ best, int2* __restrict__ locs,
                                    unsigned long long* __restrict__ count,
                                    unsigned long long max_count) {
    pdl_wait();
    const double lim = best->rho;
    const size_t E = size_t(er) * ec;
    for (size_t k = blockIdx.x * size_t(blockDim.x) + threadIdx.x; k < E;
         k += size_t(gridDim.x) * blockDim.x) {
        const float u = __ldg(ub + k);
        if (u >= -1.5f && double(u) >= lim) {
            const unsigned long long at = atomicAdd(count, 1ull);
            if (at < max_count) locs[at] = make_int2(int(k / size_t(ec)), int(k % size_t(ec)));
        }
    }
}

// ---- split centre scan (scan 1 of a search on a non-integer image) ----------------------
// The bracket of one rho from the exact split dot (same model as MODE 3 of k_tc_corr).
__device__ __forceinline__ void split_bracket(double dot_a, const SplitModel& sm, const TStats& ts,
                                              double mu_w, double omega_w, double& rho_m,
                                              double& e) {
    const double half = 0.5 * sm.delta;
    const double rad = half + sm.gamma * (dot_a + sm.delta);
    const double den = __dmul_rn(ts.omega, omega_w);
    const double num = (dot_a + half) - __dmul_rn(__dmul_rn(ts.mn, ts.mu), mu_w);
    rho_m = num / den;
    e = (rad / den) * 1.000001 + 1e-14 + fabs(rho_m) * 1e-14;
}

// Per centre: provisional rho_c = clamp(rho_m), radius rad_c (0 = exact), deg_c; partials =
// the best LOWER bound among non-degenerate centres (or the first degenerate centre).
__global__ void __launch_bounds__(256)
    k_split_centre_epi(Grid g, const double* __restrict__ dot, DevStats st, TStatsH tsh,
                       SplitModel sm, double* __restrict__ rho_c, double* __restrict__ rad_c,
                       uint8_t* __restrict__ deg_c, CellH* partials) {
    pdl_wait();
    __shared__ Cell scratch[8];
    const TStats ts = TStats{tsh.mu, tsh.omega, tsh.mn, tsh.flat};
    const size_t G = size_t(g.tr) * g.tc;
    Cell best = no_cell();
    for (size_t gi = blockIdx.x * size_t(blockDim.x) + threadIdx.x; gi < G;
         gi += size_t(gridDim.x) * blockDim.x) {
        const int ti = int(gi / size_t(g.tc)), tj = int(gi - size_t(ti) * g.tc);
        const int r = g.center_row(ti), c = g.center_col(tj);
        const size_t kk = size_t(r) * g.ec + c;
        if (st.flat[kk]) {
            rho_c[gi] = 0.0;
            rad_c[gi] = 0.0;
            deg_c[gi] = 1;
            const Cell cand = make_cell(r, c, 0.0, true);
            if (better(cand, best)) best = cand;
            continue;
        }
        double rho_m, e;
        split_bracket(dot[gi], sm, ts, st.mu[kk], st.omega[kk], rho_m, e);
        rho_c[gi] = dclamp(rho_m, -1.0, 1.0);
        rad_c[gi] = e;
        deg_c[gi] = 0;
        const Cell cand = make_cell(r, c, dclamp(rho_m - e, -1.0, 1.0), false);
        if (better(cand, best)) best = cand;
    }
    best = block_best(best, scratch);
    if (threadIdx.x == 0)
        partials[blockIdx.x] = CellH{best.rho, best.row, best.col, best.flags};
}

__device__ __forceinline__ void split_append(int2* locs, int* gidx, unsigned long long* count,
                                             int r, int c, size_t gi) {
    const unsigned long long at = atomicAdd(count, 1ull);
    locs[at] = make_int2(r, c);  // capacity G: a centre is listed at most once per pass
    gidx[at] = int(gi);
}

// Centres that still need their exact rho.  mode 0: the candidates for the best centre
// (upper bound >= the largest lower bound in *lim; a degenerate *lim lists that centre
// alone).  mode 1: the seeding decision rho_c >= thr - margin (k_seed_members) is not
// settled by the bracket.
__global__ void __launch_bounds__(256)
    k_split_pick(Grid g, const double* __restrict__ rho_c, const double* __restrict__ rad_c,
                 const uint8_t* __restrict__ deg_c, int mode, const CellH* __restrict__ lim,
                 const double* __restrict__ thr, double margin, int2* locs, int* gidx,
                 unsigned long long* count) {
    pdl_wait();
    const size_t G = size_t(g.tr) * g.tc;
    for (size_t gi = blockIdx.x * size_t(blockDim.x) + threadIdx.x; gi < G;
         gi += size_t(gridDim.x) * blockDim.x) {
        const int ti = int(gi / size_t(g.tc)), tj = int(gi - size_t(ti) * g.tc);
        const int r = g.center_row(ti), c = g.center_col(tj);
        bool pick = false;
        if (mode == 0) {
            if (lim->flags & 2)
                pick = (lim->flags & 1) && lim->row == r && lim->col == c;
            else
                pick = !deg_c[gi] && rho_c[gi] + rad_c[gi] >= lim->rho;
        } else {
            const double e = rad_c[gi];
            const double x = *thr - margin;
            pick = e > 0.0 && !deg_c[gi] && fabs(rho_c[gi] - x) <= e + 1e-12;
        }
        if (pick) split_append(locs, gidx, count, r, c, gi);
    }
}

// Exact values back into the per-group arrays.
__global__ void k_split_scatter(const double* __restrict__ rho, const int* __restrict__ gidx,
                                const unsigned long long* __restrict__ count,
                                double* __restrict__ rho_c, double* __restrict__ rad_c) {
    pdl_wait();
    const unsigned long long n = *count;
    for (unsigned long long i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
         i += size_t(gridDim.x) * blockDim.x) {
        rho_c[gidx[i]] = rho[i];
        rad_c[gidx[i]] = 0.0;
    }
}

// Groups whose members' bound test (k_sec_rows: sec_holds(min(T, 1), rho_c, R_co),
// bounds.cpp:41-46) is not settled by the centre's bracket [rho - e, rho + e].  The bound
// rho*R + sqrt(1 - rho^2) sqrt(1 - R^2) is monotone in rho on either side of rho = R, so its
// range over the bracket is spanned by the endpoint values unless R lies inside; brackets
// reaching |rho| ~ 1 (where the FP64 square root amplifies rounding) are listed outright.
// A non-finite / below -1 threshold eliminates nothing at T; with a moving threshold those
// members are re-tested later, so every bracketed group is listed.
__global__ void __launch_bounds__(256)
    k_split_sec_uncertain(Grid g, const double* __restrict__ map, const double* __restrict__ rho_c,
                          const double* __restrict__ rad_c, const uint8_t* __restrict__ deg_c,
                          const uint8_t* __restrict__ flat, const double* __restrict__ thr_ptr,
                          const uint8_t* __restrict__ seeded, uint8_t* __restrict__ gflag,
                          int2* locs, int* gidx, unsigned long long* count, int moving) {
    pdl_wait();
    const double T = *thr_ptr;
    if (!(T >= -1.0) && !moving) return;  // nothing is eliminated: no decision reads rho_c
    const bool none = !(T >= -1.0);
    const double tb = dmin(T, 1.0);
    const size_t E = size_t(g.er) * g.ec;
    for (size_t k = blockIdx.x * size_t(blockDim.x) + threadIdx.x; k < E;
         k += size_t(gridDim.x) * blockDim.x) {
        int r, c;
        g.rc(k, r, c);
        const int ti = g.tile_r(r), tj = g.tile_c(c);
        const size_t gi = size_t(ti) * g.tc + tj;
        const double e = rad_c[gi];
        if (e == 0.0 || deg_c[gi] || gflag[gi]) continue;
        if (seeded && seeded[gi]) continue;
        const int cr = g.center_row(ti), cc = g.center_col(tj);
        if ((cr == r && cc == c) || flat[k]) continue;
        const double a = rho_c[gi];
        const double lo = a - e, hi = a + e;
        const double b = dclamp(map[k], -1.0, 1.0);
        bool unsure = none || hi >= 0.9999995 || lo <= -0.9999995 || (b >= lo && b <= hi);
        if (!unsure) {
            const double f_lo = __dadd_rn(__dmul_rn(lo, b), half_gap(lo, b));
            const double f_hi = __dadd_rn(__dmul_rn(hi, b), half_gap(hi, b));
            const double fmax = dmax(f_lo, f_hi), fmin = dmin(f_lo, f_hi);
            // moving (sequential policy): the threshold only rises from T, so a member
            // certainly eliminated now stays eliminated; every other member may be re-tested
            // at a later threshold and needs the exact rho_c
            unsure = !(tb >= fmax + 1e-12 || (!moving && tb < fmin - 1e-12));
        }
        if (unsure) {
            // one listing per group: byte flags claimed through a 32-bit atomicOr
            const unsigned bit = 1u << (8 * unsigned(gi & 3));
            const unsigned old = atomicOr(reinterpret_cast<unsigned*>(gflag) + (gi >> 2), bit);
            if (!(old & bit)) split_append(locs, gidx, count, cr, cc, gi);
        }
    }
}

}  // namespace

namespace {
__global__ void k_survivor_dispatch(const Tally* tally, unsigned long long E, int* dense_flag,
                                    unsigned long long* list_count,
                                    const unsigned long long* gate) {
    pdl_wait();
    if (gate && !*gate) {  // speculative launch not confirmed: the passes behind it do nothing
        *dense_flag = 0;
        *list_count = 0ull;
        return;
    }
    const unsigned long long n = tally->survivors;
    const bool dense = n * kDenseDiv > E;
    *dense_flag = dense ? 1 : 0;
    *list_count = dense ? 0ull : n;
}

}  // namespace

cudaError_t survivor_dispatch(const Tally* tally, unsigned long long E, int* dense_flag,
                              unsigned long long* list_count, cudaStream_t s,
                              const unsigned long long* gate) {
    launch_pdl(k_survivor_dispatch, dim3(1), dim3(1), 0, s, tally, E, dense_flag, list_count,
               gate);
    return cudaGetLastError();
}

bool tc_supported(int m, int n) {
    // exact s32 dots; Kx <= 256 bytes per MMA chain; at least one template row per chunk
    return double(m) * double(n) * 65025.0 < 2147483648.0 && n + 15 <= 256;
}

TcPlan tc_plan(int m, int n, int sr, size_t smem_budget) {
    TcPlan P{};
    P.kx = ((n + 15) + 31) / 32 * 32;
    P.sr = std::max(1, sr);
    P.a_bytes = ((2032 + P.kx) + 15) / 16 * 16;
    P.a_slot = (P.a_bytes + 127) / 128 * 128;
    // header: barriers + up to 16 KB of staged row schedule; at least 16 ring stages; B
    // gets the rest (the ring grows back into what B leaves)
    P.header = kTcBarBytes + kTcSchedBytes + kEpiBytes;
    const size_t fixed = size_t(16) * P.a_slot + P.header;
    const size_t entry = size_t(16) * P.kx;
    const int per_chunk = int((smem_budget - fixed) / entry);
    if (per_chunk < 1) return TcPlan{};
    P.nch = (m + per_chunk - 1) / per_chunk;
    if (P.nch > kTcMaxChunks || P.sr > kTcMaxClasses) return TcPlan{};
    const int rows = (m + P.nch - 1) / P.nch;
    size_t off = 0, bmax = 0;
    for (int ch = 0; ch < P.nch; ++ch) {
        P.i0[ch] = ch * rows;
        P.i1[ch] = std::min(m, (ch + 1) * rows);
        int e = 0;
        for (int c = 0; c < P.sr; ++c) {
            P.cls_off[ch][c] = e;
            // largest i in [i0, i1) with i % sr == c
            int hi = P.i1[ch] - 1;
            while (hi >= P.i0[ch] && hi % P.sr != c) --hi;
            P.cls_max[ch][c] = hi;
            if (hi >= P.i0[ch]) e += (hi - P.i0[ch]) / P.sr + 1;
        }
        P.b_off[ch] = off;
        P.b_bytes[ch] = size_t(e) * entry;
        off += P.b_bytes[ch];
        bmax = std::max(bmax, P.b_bytes[ch]);
    }
    P.total_bytes = off;
    P.b_smem = (bmax + 1023) / 1024 * 1024;
    const size_t left = smem_budget - P.header - P.b_smem;
    P.stages = int(std::min<size_t>(kTcMaxStages, left / P.a_slot));
    P.smem = P.header + P.b_smem + size_t(P.stages) * P.a_slot;
    return P;
}

std::vector<int> tc_schedule(const TcPlan& P, int rmax, int* off, int* len) {
    // per chunk, rows dx = x - r0 of a band of rmax rows at stride P.sr that feed at least
    // one output row: {dx, k_lo, k_hi, B entry of T row dx - sr*k_lo}, in increasing dx
    // (so k_lo is non-decreasing: a band with fewer rows stops at k_lo >= cnt).
    std::vector<int> out;
    for (int ch = 0; ch < P.nch; ++ch) {
        off[ch] = int(out.size() / 4);
        const int i0 = P.i0[ch], i1 = P.i1[ch];
        for (int dx = i0; dx < P.sr * (rmax - 1) + i1; ++dx) {
            const int lo_num = dx - i1 + 1;
            const int k_lo = lo_num <= 0 ? 0 : (lo_num + P.sr - 1) / P.sr;
            const int k_hi = std::min(rmax - 1, (dx - i0) / P.sr);
            if (k_lo > k_hi) continue;
            const int i_top = dx - P.sr * k_lo;
            const int cls = i_top % P.sr;
            const int pos = (P.cls_max[ch][cls] - i_top) / P.sr;
            out.push_back(dx);
            out.push_back(k_lo);
            out.push_back(k_hi);
            out.push_back(P.cls_off[ch][cls] + pos);
        }
        len[ch] = int(out.size() / 4) - off[ch];
    }
    return out;
}

int tc_pitch(int q, int ec) {
    const int ntc = (ec + kTcCols - 1) / kTcCols;
    return ((std::max(q, ntc * kTcCols + 256) + 15) / 16) * 16;
}

int tc_tile_cols() { return kTcCols; }

cudaError_t tc_pitch_image(const uint8_t* img, int p, int q, uint8_t* out, int pitch, int rows,
                           cudaStream_t s) {
    const size_t chunks = size_t(rows) * (pitch / 16);
    const int blocks = int(std::min<size_t>((chunks + 255) / 256, 148 * 8));
    k_tc_pitch<<<blocks, 256, 0, s>>>(img, p, q, out, pitch, rows);
    return cudaGetLastError();
}

cudaError_t tc_split_image(const double* img, int p, int q, uint8_t* out, int pitch, int rows,
                           size_t plane_stride, int* bad, cudaStream_t s) {
    const size_t chunks = size_t(rows) * (pitch / 16);
    const int blocks = int(std::min<size_t>((chunks + 255) / 256, 148 * 8));
    k_tc_split<<<blocks, 256, 0, s>>>(img, p, q, out, pitch, rows, plane_stride, bad);
    return cudaGetLastError();
}

cudaError_t tc_screen_compact(const float* ub, int er, int ec, const CellH* best, int2* locs,
                              unsigned long long* count, unsigned long long max_count,
                              cudaStream_t s) {
    launch_pdl(k_tc_screen_compact, dim3(148 * 8), dim3(256), 0, s, ub, er, ec, best, locs, count,
               max_count);
    return cudaGetLastError();
}

cudaError_t split_centre_epilogue(GridDesc g, const double* dot, DevStats st, TStatsH ts,
                                  SplitModel sm, double* rho_c, double* rad_c, uint8_t* deg_c,
                                  CellH* partials, int n_partials, cudaStream_t s) {
    launch_pdl(k_split_centre_epi, dim3(n_partials), dim3(256), 0, s, to_grid(g), dot, st, ts, sm,
               rho_c, rad_c, deg_c, partials);
    return cudaGetLastError();
}

cudaError_t split_pick(GridDesc g, const double* rho_c, const double* rad_c, const uint8_t* deg_c,
                       int mode, const CellH* lim, const double* thr, double margin, int2* locs,
                       int* gidx, unsigned long long* count, cudaStream_t s) {
    const size_t G = size_t(g.tr) * g.tc;
    const int blocks = int(std::min<size_t>((G + 255) / 256, 148 * 8));
    launch_pdl(k_split_pick, dim3(blocks), dim3(256), 0, s, to_grid(g), rho_c, rad_c, deg_c, mode,
               lim, thr, margin, locs, gidx, count);
    return cudaGetLastError();
}

cudaError_t split_scatter(const double* rho, const int* gidx, const unsigned long long* count,
                          double* rho_c, double* rad_c, cudaStream_t s) {
    launch_pdl(k_split_scatter, dim3(64), dim3(256), 0, s, rho, gidx, count, rho_c, rad_c);
    return cudaGetLastError();
}

cudaError_t split_sec_uncertain(GridDesc g, const double* map, const double* rho_c,
                                const double* rad_c, const uint8_t* deg_c, const uint8_t* flat,
                                const double* thr, const uint8_t* seeded, uint8_t* gflag,
                                int2* locs, int* gidx, unsigned long long* count, cudaStream_t s,
                                int moving) {
    const size_t E = size_t(g.er) * g.ec;
    const int blocks = int(std::min<size_t>((E + 255) / 256, 148 * 8));
    launch_pdl(k_split_sec_uncertain, dim3(blocks), dim3(256), 0, s, to_grid(g), map, rho_c, rad_c,
               deg_c, flat, thr, seeded, gflag, locs, gidx, count, moving);
    return cudaGetLastError();
}

cudaError_t tc_build_b(const float* tf, int npad, int m, int n, const TcPlan& plan, uint8_t* out,
                       cudaStream_t s, const int* gate) {
    dim3 grid(64, plan.nch);
    launch_pdl(k_tc_build_b, dim3(grid), dim3(256), 0, s, tf, npad, m, n, plan, out, gate);
    return cudaGetLastError();
}

cudaError_t tc_corr(const TcJob& job, const TcTask& task, CellH* partials, int* nparts,
                    cudaStream_t s) {
    const int ntiles = task.nbands * task.ntc;
    const int grid = std::max(1, std::min(148, ntiles));
    *nparts = grid;
    const size_t smem = job.plan.smem;
    cudaError_t e = cudaSuccess;
    static size_t attr_set[5] = {0, 0, 0, 0, 0};
    if (task.mode < 0 || task.mode > 4) return cudaErrorInvalidValue;
    if (attr_set[task.mode] < smem) {
        const void* fn = task.mode == 0 ? (const void*)k_tc_corr<0>
                        : task.mode == 1 ? (const void*)k_tc_corr<1>
                        : task.mode == 2 ? (const void*)k_tc_corr<2>
                        : task.mode == 3 ? (const void*)k_tc_corr<3> : (const void*)k_tc_corr<4>;
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        attr_set[task.mode] = smem;
    }
    switch (task.mode) {
        case 0: launch_pdl(k_tc_corr<0>, dim3(grid), dim3(kTcThreads), smem, s, job, task, partials); break;
        case 1: launch_pdl(k_tc_corr<1>, dim3(grid), dim3(kTcThreads), smem, s, job, task, partials); break;
        case 2: launch_pdl(k_tc_corr<2>, dim3(grid), dim3(kTcThreads), smem, s, job, task, partials); break;
        case 3: launch_pdl(k_tc_corr<3>, dim3(grid), dim3(kTcThreads), smem, s, job, task, partials); break;
        default: launch_pdl(k_tc_corr<4>, dim3(grid), dim3(kTcThreads), smem, s, job, task, partials); break;
    }
    e = cudaGetLastError();
    return e;
}

}  // namespace tmk
