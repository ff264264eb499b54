// score_tc.cu -- tcgen05/TMEM tensor-core cosine scan with a fused top-k epilogue (sm_100a).
//
// The similarity of a batch of queries with every cached entry (SURVEY
// 8(a) a2-a3) is the dense contraction S = Q~ X~^T (B x N, K = dim).  One output tile is
// 128 queries (M, TMEM lanes) x 256 entries (N, TMEM columns) x dim:
//
//   warp 0 (1 lane)  TMA producer: A = Q~ tile [128 x 64] and B = X~ tile [256 x 64] per
//                    64-wide K chunk (128-byte swizzle) into a 4-stage shared-memory ring
//   warp 1 (1 lane)  MMA issuer: tcgen05.mma.cta_group::1.kind::f16 (bf16 x bf16 -> fp32)
//                    M=128 N=256 K=16, accumulating in TMEM; double-buffered accumulators
//                    (2 x 256 columns) so the epilogue of tile i overlaps the MMAs of i+1
//   warps 4-7        epilogue: each thread owns one query row (one TMEM lane), reads its 256
//                    fp32 dots with tcgen05.ld, scales by the entry inv-norm (NaN = empty
//                    slot), and keeps the running top-k in registers -- no score matrix is
//                    ever written to HBM
//
// Work unit = (n-chunk, m-tile): a run of `chunk_tiles` consecutive entry tiles for one
// query tile.  Units are dealt round-robin to a persistent grid (one CTA per SM), m fastest,
// so the CTAs running at the same time share the same entry tiles (L2 reuse).  Each unit
// ends with one partial top-k record list per query -> ws[chunk][query][KMAX]; k_finalize
// merges the n_chunks lists under the same total order (R3).
#include <cstdlib>
#include <cuda.h>

#include "kernels.h"

namespace nv {
namespace tc {

constexpr int BM = 128, BN = 256, BK = 64, STAGES = 4;
constexpr int A_BYTES = BM * BK * 2;            // 16 KiB
constexpr int B_BYTES = BN * BK * 2;            // 32 KiB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;  // 48 KiB
constexpr int TMEM_COLS = 512;                  // 2 accumulators x 256 fp32 columns
constexpr int EPI_WARP0 = 4;
// Instruction descriptor, kind::f16: D=f32 (bits 4-5 = 1), A=B=bf16 (bits 7-9, 10-12 = 1),
// both K-major (bits 15,16 = 0), N>>3 at bits 17-22, M>>4 at bits 24-28.
constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                           ((uint32_t)(BM >> 4) << 24);
constexpr int SMEM_INV_OFF = STAGES * STAGE_BYTES;              // 2 x 256 floats
constexpr int SMEM_IDS_OFF = SMEM_INV_OFF + 2 * BN * 4;          // 2 x 256 entry ids
constexpr int SMEM_BAR_OFF = SMEM_IDS_OFF + 2 * BN * 4;          // 2*STAGES + 4 mbarriers
constexpr int SMEM_TMEM_OFF = SMEM_BAR_OFF + (2 * STAGES + 4) * 8;
constexpr int SMEM_XCH_OFF = SMEM_TMEM_OFF + 16;                  // half-merge exchange (128 x 16 x 12 B)
constexpr int SMEM_BYTES = SMEM_XCH_OFF + BM * 16 * 12 + 1024;   // + alignment slack

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    while (!mbar_try_wait(bar, parity)) {
    }
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, uint32_t bar, int x, int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(x), "r"(y)
        : "memory");
}

// Programmatic dependent launch: the scan is launched while the ingest kernel is still running
// (its prologue -- barrier init, TMEM allocation, tensor-map prefetch -- overlaps it) and waits
// here for the ingest's results; it lets the finalize kernel launch early in turn.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// One lane of a converged warp (elect.sync): the rest of the warp stays in uniform control flow.
__device__ __forceinline__ bool elect_one() {
    uint32_t e;
    asm volatile(
        "{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(e));
    return e != 0;
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// Shared-memory matrix descriptor: K-major, 128-byte swizzle, 8-row groups 1024 B apart.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);   // start address (bits 0-13)
    d |= (uint64_t)1 << 16;                     // leading byte offset (unused for SW128 K-major)
    d |= (uint64_t)(1024 >> 4) << 32;           // stride byte offset: 8 rows x 128 B
    d |= (uint64_t)1 << 46;                     // descriptor version 1 (sm_100)
    d |= (uint64_t)2 << 61;                     // layout: SWIZZLE_128B
    return d;
}

__device__ __forceinline__ void umma_bf16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %3, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %4, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(accum), "r"(IDESC)
        : "memory");
}

__device__ __forceinline__ void umma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
                 : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
          "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
          "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
          "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

// Wait for this thread's outstanding tcgen05.ld; the registers are tied as in/out operands
// so the compiler cannot schedule their uses above the wait.
__device__ __forceinline__ void tmem_ld_wait_regs(uint32_t (&r)[32]) {
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]),
                   "+r"(r[7]), "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]),
                   "+r"(r[14]), "+r"(r[15]), "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]),
                   "+r"(r[21]), "+r"(r[22]), "+r"(r[23]), "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]),
                   "+r"(r[28]), "+r"(r[29]), "+r"(r[30]), "+r"(r[31])
                 :
                 : "memory");
}

__device__ __forceinline__ float4 lds_f4(uint32_t addr) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
    return v;
}

// Scale one 32-column chunk by the entry inv-norms, gate on its max, offer survivors.  The
// tile's entry ids are staged in shared memory next to the inv-norms: an offer used to load
// its id from global memory, and those dependent L2 round trips (one per improving value)
// kept the epilogue holding its TMEM accumulator while the MMA waited for it (measured: the
// scan ran 11% faster with the epilogue's loads or its arithmetic alone).
template <int KMAX, bool kDense>
__device__ __forceinline__ void epi_chunk(const uint32_t (&r)[32], uint32_t inv_addr, uint32_t col0, TopK<KMAX>& tk,
                                          uint32_t ids_addr, float* dense_row) {
    float t[32];
    float mx = -INFINITY;
#pragma unroll
    for (int i = 0; i < 32; i += 4) {
        const float4 iv = lds_f4(inv_addr + 4 * i);
        t[i] = __uint_as_float(r[i]) * iv.x;
        t[i + 1] = __uint_as_float(r[i + 1]) * iv.y;
        t[i + 2] = __uint_as_float(r[i + 2]) * iv.z;
        t[i + 3] = __uint_as_float(r[i + 3]) * iv.w;
        mx = fmaxf(mx, fmaxf(fmaxf(t[i], t[i + 1]), fmaxf(t[i + 2], t[i + 3])));
    }
    if (kDense) {
        if (dense_row) {
#pragma unroll
            for (int i = 0; i < 32; i += 4)
                *reinterpret_cast<float4*>(dense_row + col0 + i) = make_float4(t[i], t[i + 1], t[i + 2], t[i + 3]);
        }
    } else if (mx >= tk.thr) {
        if constexpr (KMAX == 1) {
            // top-1: the chunk's best key is (mx, smallest id among the values equal to mx) --
            // one offer instead of a dependent chain of up to 32 (early tiles, where the row's
            // threshold is still low, used to hold the accumulator for 3-10 K cycles)
            uint32_t best_id = 0xFFFFFFFFu, best_i = 0u;
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                if (t[i] == mx) {
                    uint32_t id;
                    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(id) : "r"(ids_addr + 4 * i));
                    if (id < best_id) { best_id = id; best_i = (uint32_t)i; }
                }
            }
            tk.offer_key(make_key(mx, best_id), col0 + best_i);
        } else {
            // k > 1: a mask of the values passing the gate, then one compact loop over its set
            // bits (the value picked from registers by a constant-index select chain).  Fully
            // unrolling 32 inlined KMAX-slot insertions per chunk (x2 call sites x2 halves) blew
            // the instruction cache: the C2 top-16 scan took 7 ms.
            uint32_t mask = 0u;
#pragma unroll
            for (int i = 0; i < 32; ++i) mask |= (t[i] >= tk.thr ? 1u : 0u) << i;   // NaN fails
#pragma unroll 1
            while (mask) {
                const int i = __ffs(mask) - 1;
                mask &= mask - 1u;
                float ti = t[0];
#pragma unroll
                for (int j = 1; j < 32; ++j) ti = (i == j) ? t[j] : ti;
                if (!(ti >= tk.thr)) continue;   // the gate may have risen since the mask
                uint32_t id;
                asm volatile("ld.shared.u32 %0, [%1];" : "=r"(id) : "r"(ids_addr + 4 * i));
                tk.offer_key(make_key(ti, id), col0 + (uint32_t)i);
            }
        }
    }
}

constexpr int EPI_WARPS = 8;                       // 2 per SM sub-partition: column halves
constexpr int NUM_THREADS_TC = (EPI_WARP0 + EPI_WARPS) * 32;   // 384

// kDense = true: debug/test variant that stores the scan values t = dot * inv_e densely
// (out[q][col]) instead of reducing them -- used to check the tcgen05 main loop on its own.
template <int KMAX, bool kDense>
__global__ void __launch_bounds__(NUM_THREADS_TC, 1)
k_score_tc(const __grid_constant__ CUtensorMap tmap_q, const __grid_constant__ CUtensorMap tmap_e,
           const float* __restrict__ inv_e, const uint32_t* __restrict__ ids, int dim, int64_t B,
           int m_tiles, int n_tiles, int chunk_tiles, int n_units, Rec* __restrict__ ws,
           uint32_t* __restrict__ gk, float* __restrict__ dense, int64_t dense_ld) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + SMEM_TMEM_OFF);
    const uint32_t sbase = smem_u32(smem);
    const uint32_t inv_base = sbase + SMEM_INV_OFF;
    const uint32_t ids_base = sbase + SMEM_IDS_OFF;
    const uint32_t bar_full = sbase + SMEM_BAR_OFF, bar_empty = bar_full + STAGES * 8;
    const uint32_t bar_tfull = bar_empty + STAGES * 8, bar_tempty = bar_tfull + 2 * 8;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int kch = dim / BK;

    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_q)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_e)) : "memory");
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(bar_full + 8 * s, 1);
            mbar_init(bar_empty + 8 * s, 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(bar_tfull + 8 * a, 1);
            mbar_init(bar_tempty + 8 * a, EPI_WARPS);   // one arrive per epilogue warp
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(TMEM_COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    // The entry tiles do not depend on the ingest kernel: the producer issues the first STAGES
    // stages' entry loads (into the empty ring) before waiting for it, their query loads after.
    int pre = 0;
    if (warp == 0 && lane == 0) {
        for (int u = blockIdx.x; u < n_units && pre < STAGES; u += gridDim.x) {
            const int chunk = u / m_tiles;
            const int n0 = chunk * chunk_tiles, n1 = min(n_tiles, n0 + chunk_tiles);
            for (int n = n0; n < n1 && pre < STAGES; ++n)
                for (int kc = 0; kc < kch && pre < STAGES; ++kc, ++pre) {
                    mbar_expect_tx(bar_full + 8 * pre, STAGE_BYTES);
                    tma_load_2d(sbase + pre * STAGE_BYTES + A_BYTES, &tmap_e, bar_full + 8 * pre, kc * BK, n * BN);
                }
        }
    }
    pdl_wait();      // queries / inv-norms / gate words of the ingest kernel are visible from here
    pdl_trigger();

    if (warp == 0) {
        // ------------------------------- TMA producer -------------------------------
        if (lane == 0) {
            uint32_t stage = 0, phase = 0;
            int it = 0;
            for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
                const int chunk = u / m_tiles, m = u - chunk * m_tiles;
                const int n0 = chunk * chunk_tiles, n1 = min(n_tiles, n0 + chunk_tiles);
                for (int n = n0; n < n1; ++n) {
                    for (int kc = 0; kc < kch; ++kc, ++it) {
                        const uint32_t sa = sbase + stage * STAGE_BYTES;
                        if (it < pre) {   // entry half already in flight, stage's tx already expected
                            tma_load_2d(sa, &tmap_q, bar_full + 8 * stage, kc * BK, m * BM);
                        } else {
                            mbar_wait(bar_empty + 8 * stage, phase ^ 1);
                            mbar_expect_tx(bar_full + 8 * stage, STAGE_BYTES);
                            tma_load_2d(sa, &tmap_q, bar_full + 8 * stage, kc * BK, m * BM);
                            tma_load_2d(sa + A_BYTES, &tmap_e, bar_full + 8 * stage, kc * BK, n * BN);
                        }
                        if (++stage == STAGES) { stage = 0; phase ^= 1; }
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------- MMA issuer ---------------------------------
        // The whole warp runs the loop (warp-uniform control flow keeps the descriptor
        // arithmetic in uniform registers); one elected lane issues.  Issued from a single
        // divergent lane, every tcgen05.mma got an ELECT/R2UR.BROADCAST wrapper and the
        // ~110-instruction k-chunk loop took about as long as the 512 tensor cycles it feeds.
        const uint64_t desc0 = sw128_desc(sbase);
        uint32_t stage = 0, phase = 0, acc = 0, acc_phase = 0;
        for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
            const int chunk = u / m_tiles;
            const int n0 = chunk * chunk_tiles, n1 = min(n_tiles, n0 + chunk_tiles);
            for (int n = n0; n < n1; ++n) {
                mbar_wait(bar_tempty + 8 * acc, acc_phase ^ 1);
                tc_fence_after();
                const uint32_t d = tmem_base + acc * BN;
                for (int kc = 0; kc < kch; ++kc) {
                    mbar_wait(bar_full + 8 * stage, phase);
                    tc_fence_after();
                    const uint64_t ad = desc0 + (uint64_t)(stage * (STAGE_BYTES >> 4));
                    const uint64_t bd = ad + (uint64_t)(A_BYTES >> 4);
                    if (elect_one()) {
#pragma unroll
                        for (int k = 0; k < BK / 16; ++k)   // +32 B along K inside the swizzle atom
                            umma_bf16(d, ad + 2 * k, bd + 2 * k, (kc | k) != 0);
                        umma_commit(bar_empty + 8 * stage);  // frees the smem stage when done
                    }
                    __syncwarp();
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
                if (elect_one()) umma_commit(bar_tfull + 8 * acc);   // accumulator ready
                __syncwarp();
                acc ^= 1;
                if (acc == 0) acc_phase ^= 1;
            }
        }
    } else if (warp >= EPI_WARP0) {
        // ------------------------------- epilogue -----------------------------------
        // warp w: TMEM lane quarter w % 4 (rows 32*(w%4)..+31), column half h = (w-4)/4.
        const int ew = warp & 3;
        const int h = (warp - EPI_WARP0) >> 2;
        const int et = threadIdx.x - EPI_WARP0 * 32;        // 0..255
        const int row = 32 * ew + lane;
        uint32_t acc = 0, acc_phase = 0;
        // The gate word and the first tile's inv-norm / id of a unit are fetched during the
        // previous unit's last tile, so no global latency is exposed at a unit boundary while
        // the MMA may be waiting for this warp's accumulator release.
        auto gate_of = [&](int uu) -> uint32_t {
            const int64_t qq = (int64_t)(uu % m_tiles) * BM + row;   // unit = chunk * m_tiles + m
            return (!kDense && gk != nullptr && qq < B) ? *reinterpret_cast<volatile const uint32_t*>(gk + qq) : 0u;
        };
        float inv_next = 0.0f;
        uint32_t id_next = 0u, gk_next = 0u;
        if ((int)blockIdx.x < n_units) {
            const int64_t c0 = (int64_t)((int)blockIdx.x / m_tiles) * chunk_tiles * BN + et;
            inv_next = __ldg(inv_e + c0);
            id_next = kDense ? 0u : __ldg(ids + c0);
            gk_next = gate_of(blockIdx.x);
        }
        for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
            const int chunk = u / m_tiles, m = u - chunk * m_tiles;
            const int n0 = chunk * chunk_tiles, n1 = min(n_tiles, n0 + chunk_tiles);
            const int64_t q = (int64_t)m * BM + row;
            const int u_next = u + (int)gridDim.x;
            const int unit_div = m_tiles;
            float* dense_row = (kDense && q < B) ? dense + q * dense_ld : nullptr;
            TopK<KMAX> tk;
            tk.init();
            // Seed the gate with a global lower bound on this query's k-th best scan value:
            // the best k-th value of any finished unit (every member of the final top-k has
            // t >= it, so nothing that can reach the final top-k is ever gated out; a value
            // read a tile early is merely a weaker bound).
            if (gk_next != 0u) tk.thr = key_to_f32((unsigned long long)gk_next << 32);
            // shared gate: every unit scanning query q publishes its running k-th best t into
            // gk[q] after each tile and raises its own gate to gk[q] one tile later -- each is a
            // lower bound on q's final k-th best, so nothing that can reach the final top-k is
            // gated out.  Without it the concurrent first-wave units each started from -inf and,
            // for k > 1, inserted most of their early values one by one while holding the TMEM
            // accumulator (C2 top-16 scan 7.0 ms vs 0.37 ms for top-1).
            const bool share = !kDense && gk != nullptr && q < B;
            uint32_t g_known = gk_next;
            if (q >= B) tk.thr = INFINITY;   // padding rows of the last query tile: never offer
#pragma unroll 1
            for (int n = n0; n < n1; ++n) {
                // entry inv-norms and ids of this tile -> smem (double-buffered by accumulator);
                // the next tile's values are fetched now so their L2 latency hides behind this tile
                const uint32_t ivb = inv_base + acc * BN * 4;
                const uint32_t idb = ids_base + acc * BN * 4;
                const uint32_t g_now = share ? *reinterpret_cast<volatile const uint32_t*>(gk + q) : 0u;  // used after this tile
                {
                    const float v = inv_next;
                    const uint32_t idv = id_next;
                    if (n + 1 < n1) {
                        inv_next = __ldg(inv_e + (int64_t)(n + 1) * BN + et);
                        if (!kDense) id_next = __ldg(ids + (int64_t)(n + 1) * BN + et);
                    } else if (u_next < n_units) {   // this CTA's next unit
                        const int64_t c0 = (int64_t)(u_next / unit_div) * chunk_tiles * BN + et;
                        inv_next = __ldg(inv_e + c0);
                        if (!kDense) id_next = __ldg(ids + c0);
                        gk_next = gate_of(u_next);
                    }
                    asm volatile("st.shared.f32 [%0], %1;" ::"r"(ivb + 4 * et), "f"(v) : "memory");
                    asm volatile("st.shared.u32 [%0], %1;" ::"r"(idb + 4 * et), "r"(idv) : "memory");
                }
                asm volatile("bar.sync 1, 256;" ::: "memory");
                mbar_wait(bar_tfull + 8 * acc, acc_phase);
                tc_fence_after();
                const uint32_t taddr = tmem_base + ((uint32_t)(32 * ew) << 16) + acc * BN + h * 128;
                const uint32_t col_base = (uint32_t)(n * BN + h * 128);
                const uint32_t ivh = ivb + 4 * (h * 128);
                const uint32_t idh = idb + 4 * (h * 128);
                uint32_t ra[32], rb[32];
                tmem_ld32(taddr, ra);
                tmem_ld_wait_regs(ra);
#pragma unroll 1
                for (int c = 0; c < 128; c += 64) {
                    tmem_ld32(taddr + c + 32, rb);
                    epi_chunk<KMAX, kDense>(ra, ivh + 4 * c, col_base + c, tk, idh + 4 * c, dense_row);
                    tmem_ld_wait_regs(rb);
                    if (c + 64 < 128) tmem_ld32(taddr + c + 64, ra);
                    else {
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(bar_tempty + 8 * acc);   // TMEM columns free again
                    }
                    epi_chunk<KMAX, kDense>(rb, ivh + 4 * (c + 32), col_base + c + 32, tk, idh + 4 * (c + 32), dense_row);
                    if (c + 64 < 128) tmem_ld_wait_regs(ra);
                }
                if (share) {
                    if (tk.k[KMAX - 1] != 0ull) {
                        const uint32_t mine = (uint32_t)(tk.k[KMAX - 1] >> 32);
                        if (mine > g_known) { atomicMax(gk + q, mine); g_known = mine; }
                    }
                    if (g_now > g_known) {
                        g_known = g_now;
                        tk.thr = fmaxf(tk.thr, key_to_f32((unsigned long long)g_now << 32));
                    }
                }
                acc ^= 1;
                if (acc == 0) acc_phase ^= 1;
            }
            if (!kDense) {
                // merge the two column halves of each row through shared memory (the inv buffer
                // region is free: every thread has passed this unit's last bar.sync)
                unsigned long long* mk = reinterpret_cast<unsigned long long*>(smem + SMEM_XCH_OFF);
                uint32_t* ms = reinterpret_cast<uint32_t*>(smem + SMEM_XCH_OFF + BM * KMAX * 8);
                if (h == 1) {
#pragma unroll
                    for (int i = 0; i < KMAX; ++i) { mk[row * KMAX + i] = tk.k[i]; ms[row * KMAX + i] = tk.s[i]; }
                }
                asm volatile("bar.sync 2, 256;" ::: "memory");
                if (h == 0) {
#pragma unroll 1
                    for (int i = 0; i < KMAX; ++i)
                        if (mk[row * KMAX + i]) tk.offer_key(mk[row * KMAX + i], ms[row * KMAX + i]);
                    if (q < B) {
                        if (gk != nullptr && tk.k[KMAX - 1] != 0ull)
                            atomicMax(gk + q, (uint32_t)(tk.k[KMAX - 1] >> 32));
                        Rec* o = ws + ((int64_t)chunk * B + q) * KMAX;
#pragma unroll
                        for (int i = 0; i < KMAX; ++i) {
                            Rec rr;
                            rr.key = tk.k[i];
                            rr.slot = tk.s[i];
                            rr.pad = 0;
                            o[i] = rr;
                        }
                    }
                }
                asm volatile("bar.sync 2, 256;" ::: "memory");
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 1) {
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS)
                     : "memory");
    }
}

// =========================================================================================
// CTA-pair variant (cta_group::2).  A cluster of 2 CTAs on one TPC computes a 256-query x
// 256-entry tile per MMA: CTA r holds query rows [128r, 128r+128) of the pair's A tile and
// entry rows [128r, 128r+128) of the B tile; the leader (rank 0) issues
// tcgen05.mma.cta_group::2 M256 N256 K16, whose result lands in both CTAs' TMEM (each its own
// 128 query rows x 256 entries).  Per SM and K chunk the TMA fill drops from 48 KiB to 32 KiB
// and the tensor core's shared-memory reads from 12 KiB to 8 KiB per MMA.  Both TMA halves
// signal the leader's full barrier (the peer-bit trick), MMA completion is multicast to both
// CTAs' empty / tfull barriers, and both CTAs' epilogue warps release the accumulator on the
// leader's tempty barrier.  The epilogue is the single-CTA one.
// =========================================================================================
namespace pair {
constexpr int STAGES = 6;
constexpr int A_BYTES = BM * BK * 2;            // 16 KiB: own 128 query rows
constexpr int B_BYTES = (BN / 2) * BK * 2;      // 16 KiB: own 128 entry rows
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;  // 32 KiB
constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                           ((uint32_t)(256 >> 4) << 24);   // M = 256 (the pair), N = 256
constexpr int SMEM_INV_OFF = STAGES * STAGE_BYTES;
constexpr int SMEM_IDS_OFF = SMEM_INV_OFF + 2 * BN * 4;
constexpr int SMEM_BAR_OFF = SMEM_IDS_OFF + 2 * BN * 4;
constexpr int SMEM_TMEM_OFF = SMEM_BAR_OFF + (2 * STAGES + 4) * 8;
constexpr int SMEM_XCH_OFF = SMEM_TMEM_OFF + 16;
constexpr int SMEM_BYTES = SMEM_XCH_OFF + BM * 16 * 12 + 1024;
}  // namespace pair

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t map_to_rank(uint32_t saddr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
    return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
    // default (.release.cta) semantics like CUTLASS's ClusterBarrier::arrive(cta_id): the
    // TMEM reads it publishes are ordered by tcgen05.wait::ld + fence::before_thread_sync;
    // a .cluster-scope release would add a cluster-wide memory barrier per tile
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void tma_load_2d_pair(uint32_t dst, const CUtensorMap* map, uint32_t bar, int x, int y) {
    // both CTAs of the pair signal the leader's barrier (clear the peer bit of the address)
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(bar & 0xFEFFFFFFu), "r"(x), "r"(y)
        : "memory");
}
__device__ __forceinline__ void umma_bf16_pair(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %3, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %4, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(accum), "r"(pair::IDESC)
        : "memory");
}
__device__ __forceinline__ void umma_commit_pair(uint32_t bar) {
    asm volatile(
        "{\n\t.reg .b16 m;\n\tmov.b16 m, 3;\n\t"
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n\t}" ::"r"(
            bar)
        : "memory");
}

namespace pair {   // (unqualified layout constants below resolve to pair::)
template <int KMAX, bool kDense>
__global__ void __launch_bounds__(NUM_THREADS_TC, 1)
k_score_tc2(const __grid_constant__ CUtensorMap tmap_q, const __grid_constant__ CUtensorMap tmap_e,
            const float* __restrict__ inv_e, const uint32_t* __restrict__ ids, int dim, int64_t B,
            int m_pairs, int n_tiles, int chunk_tiles, int n_units, Rec* __restrict__ ws,
            uint32_t* __restrict__ gk, float* __restrict__ dense, int64_t dense_ld) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + SMEM_TMEM_OFF);
    const uint32_t sbase = smem_u32(smem);
    const uint32_t inv_base = sbase + SMEM_INV_OFF;
    const uint32_t ids_base = sbase + SMEM_IDS_OFF;
    const uint32_t bar_full = sbase + SMEM_BAR_OFF, bar_empty = bar_full + STAGES * 8;
    const uint32_t bar_tfull = bar_empty + STAGES * 8, bar_tempty = bar_tfull + 2 * 8;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int kch = dim / BK;
    const uint32_t rank = cluster_rank();
    const int cid = blockIdx.x >> 1, n_clusters = gridDim.x >> 1;

    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_q)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_e)) : "memory");
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(bar_full + 8 * s, 1);
            mbar_init(bar_empty + 8 * s, 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(bar_tfull + 8 * a, 1);
            mbar_init(bar_tempty + 8 * a, 2 * EPI_WARPS);   // both CTAs' epilogue warps (leader's copy)
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(TMEM_COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();   // peer barriers initialised, TMEM allocated in both CTAs
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    // Entry tiles first (independent of the ingest kernel), as in the single-CTA kernel: both
    // CTAs issue their halves of the first STAGES stages' entry tiles before the PDL wait; the
    // leader's barrier expects all four loads of a stage once.
    int pre = 0;
    if (warp == 0 && lane == 0) {
        for (int u = cid; u < n_units && pre < STAGES; u += n_clusters) {
            const int chunk = u / m_pairs;
            const int n0 = chunk * chunk_tiles, n1 = min(n_tiles, n0 + chunk_tiles);
            for (int n = n0; n < n1 && pre < STAGES; ++n)
                for (int kc = 0; kc < kch && pre < STAGES; ++kc, ++pre) {
                    if (rank == 0) mbar_expect_tx(bar_full + 8 * pre, 2 * STAGE_BYTES);
                    tma_load_2d_pair(sbase + pre * STAGE_BYTES + A_BYTES, &tmap_e, bar_full + 8 * pre, kc * BK,
                                     n * BN + (int)rank * (BN / 2));
                }
        }
    }
    pdl_wait();      // queries / inv-norms / gate words of the ingest kernel are visible from here
    pdl_trigger();

    if (warp == 0) {
        // ------------------------------- TMA producer (both CTAs) ---------------------
        if (lane == 0) {
            uint32_t stage = 0, phase = 0;
            int it = 0;
            for (int u = cid; u < n_units; u += n_clusters) {
                const int chunk = u / m_pairs, mp = u - chunk * m_pairs;
                const int n0 = chunk * chunk_tiles, n1 = min(n_tiles, n0 + chunk_tiles);
                const int qrow = (2 * mp + (int)rank) * BM;
                for (int n = n0; n < n1; ++n) {
                    for (int kc = 0; kc < kch; ++kc, ++it) {
                        const uint32_t sa = sbase + stage * STAGE_BYTES;
                        if (it < pre) {   // entry half already in flight, stage's tx already expected
                            tma_load_2d_pair(sa, &tmap_q, bar_full + 8 * stage, kc * BK, qrow);
                        } else {
                            mbar_wait(bar_empty + 8 * stage, phase ^ 1);
                            if (rank == 0) mbar_expect_tx(bar_full + 8 * stage, 2 * STAGE_BYTES);
                            tma_load_2d_pair(sa, &tmap_q, bar_full + 8 * stage, kc * BK, qrow);
                            tma_load_2d_pair(sa + A_BYTES, &tmap_e, bar_full + 8 * stage, kc * BK,
                                             n * BN + (int)rank * (BN / 2));
                        }
                        if (++stage == STAGES) { stage = 0; phase ^= 1; }
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------- MMA issuer (leader only) --------------------
        // whole warp in the loop, one elected lane issues (see the single-CTA kernel)
        if (rank == 0) {
            const uint64_t desc0 = sw128_desc(sbase);
            uint32_t stage = 0, phase = 0, acc = 0, acc_phase = 0;
            for (int u = cid; u < n_units; u += n_clusters) {
                const int chunk = u / m_pairs;
                const int n0 = chunk * chunk_tiles, n1 = min(n_tiles, n0 + chunk_tiles);
                for (int n = n0; n < n1; ++n) {
                    mbar_wait(bar_tempty + 8 * acc, acc_phase ^ 1);
                    tc_fence_after();
                    const uint32_t d = tmem_base + acc * BN;
                    for (int kc = 0; kc < kch; ++kc) {
                        mbar_wait(bar_full + 8 * stage, phase);
                        tc_fence_after();
                        const uint64_t ad = desc0 + (uint64_t)(stage * (STAGE_BYTES >> 4));
                        const uint64_t bd = ad + (uint64_t)(A_BYTES >> 4);
                        if (elect_one()) {
#pragma unroll
                            for (int k = 0; k < BK / 16; ++k)
                                umma_bf16_pair(d, ad + 2 * k, bd + 2 * k, (kc | k) != 0);
                            umma_commit_pair(bar_empty + 8 * stage);   // frees the stage in both CTAs
                        }
                        __syncwarp();
                        if (++stage == STAGES) { stage = 0; phase ^= 1; }
                    }
                    if (elect_one()) umma_commit_pair(bar_tfull + 8 * acc);   // both CTAs' accumulators ready
                    __syncwarp();
                    acc ^= 1;
                    if (acc == 0) acc_phase ^= 1;
                }
            }
        }
    } else if (warp >= EPI_WARP0) {
        // ------------------------------- epilogue (both CTAs) ------------------------
        const int ew = warp & 3;
        const int h = (warp - EPI_WARP0) >> 2;
        const int et = threadIdx.x - EPI_WARP0 * 32;
        const int row = 32 * ew + lane;
        const uint32_t tempty_leader = map_to_rank(bar_tempty, 0);
        uint32_t acc = 0, acc_phase = 0;
        // next unit's gate word / first-tile inv-norm and id prefetched as in the 1-CTA kernel
        auto gate_of = [&](int uu) -> uint32_t {
            const int64_t qq = (int64_t)(2 * (uu % m_pairs) + (int)rank) * BM + row;
            return (!kDense && gk != nullptr && qq < B) ? *reinterpret_cast<volatile const uint32_t*>(gk + qq) : 0u;
        };
        float inv_next = 0.0f;
        uint32_t id_next = 0u, gk_next = 0u;
        if (cid < n_units) {
            const int64_t c0 = (int64_t)(cid / m_pairs) * chunk_tiles * BN + et;
            inv_next = __ldg(inv_e + c0);
            id_next = kDense ? 0u : __ldg(ids + c0);
            gk_next = gate_of(cid);
        }
        for (int u = cid; u < n_units; u += n_clusters) {
            const int chunk = u / m_pairs, mp = u - chunk * m_pairs;
            const int n0 = chunk * chunk_tiles, n1 = min(n_tiles, n0 + chunk_tiles);
            const int64_t q = (int64_t)(2 * mp + (int)rank) * BM + row;
            const int u_next = u + n_clusters;
            const int unit_div = m_pairs;
            float* dense_row = (kDense && q < B) ? dense + q * dense_ld : nullptr;
            TopK<KMAX> tk;
            tk.init();
            if (gk_next != 0u) tk.thr = key_to_f32((unsigned long long)gk_next << 32);
            // shared gate: every unit scanning query q publishes its running k-th best t into
            // gk[q] after each tile and raises its own gate to gk[q] one tile later -- each is a
            // lower bound on q's final k-th best, so nothing that can reach the final top-k is
            // gated out.  Without it the concurrent first-wave units each started from -inf and,
            // for k > 1, inserted most of their early values one by one while holding the TMEM
            // accumulator (C2 top-16 scan 7.0 ms vs 0.37 ms for top-1).
            const bool share = !kDense && gk != nullptr && q < B;
            uint32_t g_known = gk_next;
            if (q >= B) tk.thr = INFINITY;
#pragma unroll 1
            for (int n = n0; n < n1; ++n) {
                const uint32_t ivb = inv_base + acc * BN * 4;
                const uint32_t idb = ids_base + acc * BN * 4;
                const uint32_t g_now = share ? *reinterpret_cast<volatile const uint32_t*>(gk + q) : 0u;  // used after this tile
                {
                    const float v = inv_next;
                    const uint32_t idv = id_next;
                    if (n + 1 < n1) {
                        inv_next = __ldg(inv_e + (int64_t)(n + 1) * BN + et);
                        if (!kDense) id_next = __ldg(ids + (int64_t)(n + 1) * BN + et);
                    } else if (u_next < n_units) {   // this CTA's next unit
                        const int64_t c0 = (int64_t)(u_next / unit_div) * chunk_tiles * BN + et;
                        inv_next = __ldg(inv_e + c0);
                        if (!kDense) id_next = __ldg(ids + c0);
                        gk_next = gate_of(u_next);
                    }
                    asm volatile("st.shared.f32 [%0], %1;" ::"r"(ivb + 4 * et), "f"(v) : "memory");
                    asm volatile("st.shared.u32 [%0], %1;" ::"r"(idb + 4 * et), "r"(idv) : "memory");
                }
                asm volatile("bar.sync 1, 256;" ::: "memory");
                mbar_wait(bar_tfull + 8 * acc, acc_phase);
                tc_fence_after();
                const uint32_t taddr = tmem_base + ((uint32_t)(32 * ew) << 16) + acc * BN + h * 128;
                const uint32_t col_base = (uint32_t)(n * BN + h * 128);
                const uint32_t ivh = ivb + 4 * (h * 128);
                const uint32_t idh = idb + 4 * (h * 128);
                uint32_t ra[32], rb[32];
                tmem_ld32(taddr, ra);
                tmem_ld_wait_regs(ra);
#pragma unroll 1
                for (int c = 0; c < 128; c += 64) {
                    tmem_ld32(taddr + c + 32, rb);
                    epi_chunk<KMAX, kDense>(ra, ivh + 4 * c, col_base + c, tk, idh + 4 * c, dense_row);
                    tmem_ld_wait_regs(rb);
                    if (c + 64 < 128) tmem_ld32(taddr + c + 64, ra);
                    else {
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) {
                            if (rank == 0) mbar_arrive(bar_tempty + 8 * acc);   // own barrier
                            else mbar_arrive_cluster(tempty_leader + 8 * acc);
                        }
                    }
                    epi_chunk<KMAX, kDense>(rb, ivh + 4 * (c + 32), col_base + c + 32, tk, idh + 4 * (c + 32), dense_row);
                    if (c + 64 < 128) tmem_ld_wait_regs(ra);
                }
                if (share) {
                    if (tk.k[KMAX - 1] != 0ull) {
                        const uint32_t mine = (uint32_t)(tk.k[KMAX - 1] >> 32);
                        if (mine > g_known) { atomicMax(gk + q, mine); g_known = mine; }
                    }
                    if (g_now > g_known) {
                        g_known = g_now;
                        tk.thr = fmaxf(tk.thr, key_to_f32((unsigned long long)g_now << 32));
                    }
                }
                acc ^= 1;
                if (acc == 0) acc_phase ^= 1;
            }
            if (!kDense) {
                unsigned long long* mk = reinterpret_cast<unsigned long long*>(smem + SMEM_XCH_OFF);
                uint32_t* ms = reinterpret_cast<uint32_t*>(smem + SMEM_XCH_OFF + BM * KMAX * 8);
                if (h == 1) {
#pragma unroll
                    for (int i = 0; i < KMAX; ++i) { mk[row * KMAX + i] = tk.k[i]; ms[row * KMAX + i] = tk.s[i]; }
                }
                asm volatile("bar.sync 2, 256;" ::: "memory");
                if (h == 0) {
#pragma unroll 1
                    for (int i = 0; i < KMAX; ++i)
                        if (mk[row * KMAX + i]) tk.offer_key(mk[row * KMAX + i], ms[row * KMAX + i]);
                    if (q < B) {
                        if (gk != nullptr && tk.k[KMAX - 1] != 0ull)
                            atomicMax(gk + q, (uint32_t)(tk.k[KMAX - 1] >> 32));
                        Rec* o = ws + ((int64_t)chunk * B + q) * KMAX;
#pragma unroll
                        for (int i = 0; i < KMAX; ++i) {
                            Rec rr;
                            rr.key = tk.k[i];
                            rr.slot = tk.s[i];
                            rr.pad = 0;
                            o[i] = rr;
                        }
                    }
                }
                asm volatile("bar.sync 2, 256;" ::: "memory");
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();   // both CTAs finished with TMEM and with the leader's barriers
    tc_fence_after();
    if (warp == 1) {
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS)
                     : "memory");
    }
}
}  // namespace pair

template <int KMAX, bool kDense>
static bool launch_pair(const TcPlan& p, const CUtensorMap* tq, const CUtensorMap* te, const float* inv_e,
                        const uint32_t* ids, int dim, int64_t b, Rec* ws, uint32_t* gk, float* dense,
                        int64_t dense_ld, cudaStream_t s) {
    auto kern = pair::k_score_tc2<KMAX, kDense>;
    static bool attr_set = false;
    if (!attr_set) {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, pair::SMEM_BYTES) != cudaSuccess)
            return false;
        attr_set = true;
    }
    const int n_units = p.n_chunks * p.m_tiles;   // m_tiles of a pair plan = query-tile pairs
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)(2 * p.grid));
    cfg.blockDim = dim3(NUM_THREADS_TC);
    cfg.dynamicSmemBytes = pair::SMEM_BYTES;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    const CUtensorMap q = *tq, e = *te;
    if (cudaLaunchKernelEx(&cfg, kern, q, e, inv_e, ids, dim, b, p.m_tiles, p.n_tiles, p.chunk_tiles, n_units,
                           ws, gk, dense, dense_ld) != cudaSuccess)
        return false;
    return cudaPeekAtLastError() == cudaSuccess;
}

template <int KMAX, bool kDense>
static bool launch(const TcPlan& p, const CUtensorMap* tq, const CUtensorMap* te, const float* inv_e,
                   const uint32_t* ids, int dim, int64_t b, Rec* ws, uint32_t* gk, float* dense,
                   int64_t dense_ld, cudaStream_t s) {
    auto kern = k_score_tc<KMAX, kDense>;
    static bool attr_set = false;
    if (!attr_set) {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES) != cudaSuccess)
            return false;
        attr_set = true;
    }
    const int n_units = p.n_chunks * p.m_tiles;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)p.grid);
    cfg.blockDim = dim3(NUM_THREADS_TC);
    cfg.dynamicSmemBytes = SMEM_BYTES;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const CUtensorMap q = *tq, e = *te;
    if (cudaLaunchKernelEx(&cfg, kern, q, e, inv_e, ids, dim, b, p.m_tiles, p.n_tiles, p.chunk_tiles, n_units, ws,
                           gk, dense, dense_ld) != cudaSuccess)
        return false;
    return cudaPeekAtLastError() == cudaSuccess;
}

}  // namespace tc

bool tc_supported(int dim) { return dim % tc::BK == 0 && dim >= tc::BK && dim <= kMaxDim; }

// Chunk size: minimise the round-robin makespan (memoised per (b, n_slots, sm_count)) (in tiles, + a small per-unit cost for the
// record flush / pipeline refill); ties -> larger chunks (fewer partial records to merge).
// pair = true: CTA-pair kernel; m_tiles then counts 256-query tile pairs and the "CTAs" of
// the makespan model are clusters (sm_count / 2).
TcPlan tc_plan(int64_t b, int64_t n_slots, int sm_count, bool pair) {
    static thread_local int64_t mb = -1, mn = -1;
    static thread_local int ms = -1;
    static thread_local bool mp = false;
    static thread_local TcPlan memo{};
    if (b == mb && n_slots == mn && sm_count == ms && pair == mp) return memo;
    TcPlan p{};
    p.pair = pair;
    if (pair) sm_count = std::max(1, sm_count / 2);
    p.m_tiles = (int)((b + (pair ? 2 * tc::BM : tc::BM) - 1) / (pair ? 2 * tc::BM : tc::BM));
    p.n_tiles = (int)((n_slots + tc::BN - 1) / tc::BN);
    double best = 1e30;
    for (int nc = 1; nc <= std::min(p.n_tiles, 64); ++nc) {
        const int nch = (p.n_tiles + nc - 1) / nc;
        const int64_t units = (int64_t)nch * p.m_tiles;
        const int g = (int)std::min<int64_t>(sm_count, units);
        // CTA j takes units j, j+g, ...; unit u has chunk u / m_tiles
        double mk = 0;
        for (int j = 0; j < g; ++j) {
            double t = 0;
            for (int64_t u = j; u < units; u += g) {
                const int c = (int)(u / p.m_tiles);
                t += std::min(nc, p.n_tiles - c * nc) + 0.15;
            }
            mk = std::max(mk, t);
        }
        if (mk < best - 1e-9 || (mk <= best + 1e-9 && nc > p.chunk_tiles)) {
            best = mk;
            p.chunk_tiles = nc;
        }
    }
    if (const char* ev = std::getenv("NIRVANA_TC_CHUNK")) {   // experiments: fixed entry tiles per unit
        const int nc = std::atoi(ev);
        if (nc >= 1) p.chunk_tiles = std::min(nc, p.n_tiles);
    }
    p.n_chunks = (p.n_tiles + p.chunk_tiles - 1) / p.chunk_tiles;
    p.grid = (int)std::min<int64_t>(sm_count, (int64_t)p.n_chunks * p.m_tiles);
    p.parts = p.n_chunks;
    mb = b;
    mn = n_slots;
    ms = pair ? 2 * sm_count : sm_count;
    mp = pair;
    memo = p;
    return p;
}

// tmap_e: box of 256 entry rows for the single-CTA kernel, 128 rows for the CTA pair.
bool launch_score_tc(int kmax, const TcPlan& p, const void* tmap_q, const void* tmap_e, const float* inv_e,
                     const uint32_t* ids, int dim, int64_t b, Rec* ws, uint32_t* gk, cudaStream_t s) {
    const CUtensorMap* tq = static_cast<const CUtensorMap*>(tmap_q);
    const CUtensorMap* te = static_cast<const CUtensorMap*>(tmap_e);
    if (p.pair) {
        if (kmax == 1) return tc::launch_pair<1, false>(p, tq, te, inv_e, ids, dim, b, ws, gk, nullptr, 0, s);
        if (kmax == 4) return tc::launch_pair<4, false>(p, tq, te, inv_e, ids, dim, b, ws, gk, nullptr, 0, s);
        return tc::launch_pair<16, false>(p, tq, te, inv_e, ids, dim, b, ws, gk, nullptr, 0, s);
    }
    if (kmax == 1) return tc::launch<1, false>(p, tq, te, inv_e, ids, dim, b, ws, gk, nullptr, 0, s);
    if (kmax == 4) return tc::launch<4, false>(p, tq, te, inv_e, ids, dim, b, ws, gk, nullptr, 0, s);
    return tc::launch<16, false>(p, tq, te, inv_e, ids, dim, b, ws, gk, nullptr, 0, s);
}

bool launch_score_tc_dense(const TcPlan& p, const void* tmap_q, const void* tmap_e, const float* inv_e, int dim,
                           int64_t b, float* dense, int64_t dense_ld, cudaStream_t s) {
    const CUtensorMap* tq = static_cast<const CUtensorMap*>(tmap_q);
    const CUtensorMap* te = static_cast<const CUtensorMap*>(tmap_e);
    if (p.pair) return tc::launch_pair<1, true>(p, tq, te, inv_e, nullptr, dim, b, nullptr, nullptr, dense, dense_ld, s);
    return tc::launch<1, true>(p, tq, te, inv_e, nullptr, dim, b, nullptr, nullptr, dense, dense_ld, s);
}

}  // namespace nv
