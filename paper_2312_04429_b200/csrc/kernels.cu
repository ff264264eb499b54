// kernels.cu -- CUDA-core kernels of the NIRVANA cache lookup for sm_100a:
//   k_normalise      query ingest / insert normalisation
//   k_score_stream   HBM-streaming small-batch cosine scan + running top-k (a2, a3)
//   k_finalize       cross-split merge, Fig. 11 K map, hole rule, latent gather,
//                    LCBFU access counters (a3, a5, a6, a7, a8)
//   k_insert_commit / k_copy_latents   LCBFU insertion (a10)
//   k_evict_*        LCBFU eviction: radix select of the n smallest f*K keys, presence
//                    clearing, dirty-entry removal (a9)
#include "common.cuh"
#include "kernels.h"
#include "evict.cuh"

namespace nv {

// ---------------------------------------------------------------------------------------
// Normalisation (reading R2).  One warp per row (8 rows per 256-thread CTA); dim <= 1024.
// Lane l holds elements l + 32k (k < 32) of the row zero-padded to P = next_pow2(dim).
// The sum of squares follows the oracle's halving tree exactly -- stride s = P/2 ... 1,
// a[i] = a[i] + a[i+s]: strides >= 32 pair slots inside a lane, strides < 32 pair lanes
// (shfl_down) -- so the sum, the correctly rounded fp64 sqrt and division and the direct
// fp64->bf16 RNE conversion (cvt.rn.bf16.f64) give bit-identical stored rows.
// ---------------------------------------------------------------------------------------
// NS = dim / 32 slots per lane (slot k of lane l = element l + 32k); the zero padding up to
// P = next_pow2(dim) is implicit: an addition of a padded +0.0 to a non-negative partial sum
// is an identity, so it is skipped at compile time without changing a single bit.
template <int NS>
__device__ __forceinline__ double warp_tree_sum(double (&v)[NS]) {
    // element stride 32h pairs slot k with slot k + h of the same lane (i < s <=> k < h);
    // slots >= NS are padding zeros and stay zero, strides >= P pair nothing
#pragma unroll
    for (int h = 16; h >= 1; h >>= 1) {
#pragma unroll
        for (int k = 0; k < 16; ++k)
            if (k < h && k + h < NS) v[k] = __dadd_rn(v[k], v[k + h]);
    }
    double r = v[0];
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1) {
        const double o = __shfl_down_sync(0xFFFFFFFFu, r, s);
        r = __dadd_rn(r, o);
    }
    return __shfl_sync(0xFFFFFFFFu, r, 0);
}

template <typename Tin>
__device__ __forceinline__ float load_in(const Tin* p);
template <>
__device__ __forceinline__ float load_in<float>(const float* p) { return __ldg(p); }
template <>
__device__ __forceinline__ float load_in<__nv_bfloat16>(const __nv_bfloat16* p) {
    return __bfloat162float(*p);
}

// Stores of one normalised row: ND = 1 (k_normalise) or up to kMaxWorld destinations
// (k_normalise_push: the same row into every rank's arena over NVLink).
template <int ND>
struct RowDst {
    __nv_bfloat16* y[ND];
    float* inv[ND];
    int32_t* status[ND];
    int n;
};

template <int ND>
__device__ __forceinline__ void put_bf16(const RowDst<ND>& o, int64_t idx, __nv_bfloat16 v) {
    if constexpr (ND == 1) o.y[0][idx] = v;
    else
        for (int d = 0; d < o.n; ++d) o.y[d][idx] = v;
}
template <int ND>
__device__ __forceinline__ void put_meta(const RowDst<ND>& o, int64_t row, float inv, int32_t st) {
    if constexpr (ND == 1) { o.inv[0][row] = inv; o.status[0][row] = st; }
    else
        for (int d = 0; d < o.n; ++d) { o.inv[d][row] = inv; o.status[d][row] = st; }
}

// Phase 2 by correctly rounded division, for a row where some y = x * rcp(nu) landed near a
// bf16 rounding midpoint (rare).  Kept out of line so the compiler cannot if-convert the
// 24 divisions into the fast path (it did: 26 MUFU.RCP64H + 188 DFMA per row, ncu s3).
template <typename Tin, int NS, int ND>
__device__ __noinline__ void normalise_row_exact(const Tin* __restrict__ xr, int lane, const RowDst<ND>& o,
                                                 int64_t orow, double nu) {
    constexpr int dim = NS * 32;
    const int64_t ybase = orow * (int64_t)dim;
    double v[NS];
#pragma unroll
    for (int k = 0; k < NS; ++k) {
        const double x = (double)load_in<Tin>(xr + lane + 32 * k);
        const __nv_bfloat16 b = __double2bfloat16(__ddiv_rn(x, nu));
        put_bf16(o, ybase + lane + 32 * k, b);
        const double yd = (double)__bfloat162float(b);
        v[k] = __dmul_rn(yd, yd);
    }
    const double s2 = warp_tree_sum<NS>(v);
    if (lane == 0) {
        if (s2 == 0.0) put_meta(o, orow, __int_as_float(0x7FC00000), CACHE_ROW_ZERO_NORM);
        else put_meta(o, orow, __double2float_rn(__ddiv_rn(1.0, __dsqrt_rn(s2))), CACHE_ROW_OK);
    }
}

// One warp normalises input row xr into output row `orow` of every destination.
template <typename Tin, int NS, int ND>
__device__ __forceinline__ void normalise_row(const Tin* __restrict__ xr, int lane, const RowDst<ND>& o,
                                              int64_t orow) {
    constexpr int dim = NS * 32;
    const int64_t ybase = orow * (int64_t)dim;
    // the inputs are not kept across the two phases (re-read from L1 in phase 2): the 24 fp64
    // squares + 24 fp32 inputs held 92 registers per thread and limited the kernel to 25%
    // occupancy (latency-bound, ncu r1ai)
    double v[NS];
    int bad = 0;
#pragma unroll
    for (int k = 0; k < NS; ++k) {
        const float xk = load_in<Tin>(xr + lane + 32 * k);
        const double xv = (double)xk;
        bad |= !isfinite(xk);
        v[k] = __dmul_rn(xv, xv);
    }
    bad = __any_sync(0xFFFFFFFFu, bad);
    int st = CACHE_ROW_NONFINITE;
    double s = 0.0;
    if (!bad) {
        s = warp_tree_sum<NS>(v);
        st = s == 0.0 ? CACHE_ROW_ZERO_NORM : (!isfinite(s) ? CACHE_ROW_NONFINITE : CACHE_ROW_OK);
    }
    if (st != CACHE_ROW_OK) {
        for (int i = lane; i < dim; i += 32) put_bf16(o, ybase + i, __float2bfloat16_rn(0.0f));
        if (lane == 0) put_meta(o, orow, __int_as_float(0x7FC00000), st);
        return;
    }
    const double nu = __dsqrt_rn(s);
    // bf16_RNE(x / nu) without a division per element: y = x * rcp(nu) is within ~2 fp64 ulps
    // of x / nu, so both round to the same bf16 unless y lies within a few ulps of a bf16
    // rounding midpoint (the 45 fp64 mantissa bits below the bf16 LSB == 2^44) or in the bf16
    // subnormal range -- then the whole row is redone with the exact correctly rounded
    // division (normalise_row_exact, which overwrites every stored value).  Bit-identical
    // to bf16_RNE(__ddiv_rn(x, nu)) by construction.
    //
    // Off those cases y is a normal bf16-range value (|y| <= ~1) that is not a rounding tie,
    // so RNE to 8 significant bits is "add half an LSB, truncate" on the bit pattern (a carry
    // into the exponent is the correct rounding up), and the bf16 is read off the rounded
    // double -- integer ops instead of cvt.rn.bf16.f64 plus two conversions back to fp64
    // (the XU conversion pipe was the busiest unit, ncu s3).  Exact zeros (x = +-0) round to
    // themselves.
    const double rnu = __drcp_rn(nu);
    int near = 0;
#pragma unroll
    for (int k = 0; k < NS; ++k) {
        const double x = (double)load_in<Tin>(xr + lane + 32 * k);
        const double y = __dmul_rn(x, rnu);
        // all on 32-bit halves (the 64-bit forms cost ~2x the integer instructions, and the
        // kernel is issue-bound: ncu s24, 55% issue slots busy)
        const uint32_t lo = (uint32_t)__double2loint(y), hi = (uint32_t)__double2hiint(y);
        // near a midpoint: |(u mod 2^45) - 2^44| <= 16  <=>  (u + 2^44 + 16) mod 2^45 <= 32
        uint32_t tlo, thi;
        asm("add.cc.u32 %0, %2, 16;\n\taddc.u32 %1, %3, 4096;" : "=r"(tlo), "=r"(thi) : "r"(lo), "r"(hi));
        const uint32_t ahi = hi & 0x7FFFFFFFu;
        near |= (((thi & 0x1FFFu) == 0u) & (tlo <= 32u)) | ((ahi < 0x38700000u) & ((ahi | lo) != 0u));
        // RNE to bf16 precision: + 2^44 (bit 12 of the high word), clear bits 0..44 (the low
        // word entirely); the bf16 is sign | (e11 - 896) << 7 | top 7 mantissa bits
        const uint32_t rhi = (hi + 0x1000u) & ~0x1FFFu;
        const uint32_t bits = ((rhi >> 16) & 0x8000u) | ((rhi & 0x7FF00000u) ? ((rhi >> 13) & 0x3FFFFu) - 0x1C000u : 0u);
        put_bf16(o, ybase + lane + 32 * k, __ushort_as_bfloat16((unsigned short)bits));
        const double yd = __hiloint2double((int)rhi, 0);   // == the stored bf16, exactly
        v[k] = __dmul_rn(yd, yd);
    }
    if (__any_sync(0xFFFFFFFFu, near)) {   // warp-uniform, rare
        __syncwarp();
        normalise_row_exact<Tin, NS, ND>(xr, lane, o, orow, nu);
        return;
    }
    const double s2 = warp_tree_sum<NS>(v);
    if (lane == 0) {
        if (s2 == 0.0) put_meta(o, orow, __int_as_float(0x7FC00000), CACHE_ROW_ZERO_NORM);
        else put_meta(o, orow, __double2float_rn(__ddiv_rn(1.0, __dsqrt_rn(s2))), CACHE_ROW_OK);
    }
}

template <typename Tin, int NS>
__global__ void __launch_bounds__(256, 4) k_normalise(const Tin* __restrict__ x, int64_t n,
                                                   __nv_bfloat16* __restrict__ y, float* __restrict__ inv,
                                                   int32_t* __restrict__ status, uint32_t* __restrict__ gk) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");   // let the scan's prologue start
    const int lane = threadIdx.x & 31;
    const int64_t r = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    if (r >= n) return;   // warp-uniform
    if (gk != nullptr && lane == 0) gk[r] = 0u;
    RowDst<1> o;
    o.y[0] = y;
    o.inv[0] = inv;
    o.status[0] = status;
    o.n = 1;
    normalise_row<Tin, NS, 1>(x + r * (int64_t)(NS * 32), lane, o, r);
}

// Publish: every thread fences its stores at system scope, the CTA counts itself done, and
// the last CTA of the grid stores the epoch into every consumer's flag word (release.sys).
// A fence + relaxed RMW chain + fence orders every CTA's data before the flag.
__device__ __forceinline__ bool push_aborted(const PushSignal& sg) {
    return sg.abort && *(volatile const uint32_t*)sg.abort;
}

__device__ __forceinline__ void push_signal(const PushSignal& sg) {
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned prev = atomicAdd(sg.done, 1u);
        if (prev == gridDim.x - 1) {
            atomicExch(sg.done, 0u);   // ready for the next launch (stream-ordered)
            __threadfence_system();
            for (int d = 0; d < sg.world; ++d)
                asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(sg.flag[d]), "r"(sg.epoch) : "memory");
        }
    }
}

// Query ingest fused with the all-gather: rank r normalises its own n rows and stores them
// (bf16 row, inv-norm, status) into global rows [row0, row0 + n) of EVERY rank's arena.
template <typename Tin, int NS>
__global__ void __launch_bounds__(256) k_normalise_push(const Tin* __restrict__ x, int64_t n, PushRows out,
                                                        int64_t row0, PushSignal sig) {
    if (push_aborted(sig)) return;   // a peer failed: no more stores into peer memory
    const int lane = threadIdx.x & 31;
    const int64_t r = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    if (r < n) {
        RowDst<kMaxWorld> o;
        for (int d = 0; d < kMaxWorld; ++d) { o.y[d] = out.y[d]; o.inv[d] = out.inv[d]; o.status[d] = out.status[d]; }
        o.n = out.n;
        normalise_row<Tin, NS, kMaxWorld>(x + r * (int64_t)(NS * 32), lane, o, row0 + r);
    }
    push_signal(sig);
}

__global__ void k_wait_flags(const uint32_t* __restrict__ flags, int world, uint32_t epoch,
                             unsigned long long timeout_ns, uint32_t* abort, uint32_t* err_host) {
    const int t = threadIdx.x;
    if (t >= world) return;
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
        uint32_t v;
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flags + t) : "memory");
        if ((int32_t)(v - epoch) >= 0) break;
        if (*(volatile uint32_t*)abort) break;   // an earlier wait already failed
        unsigned long long now;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
        if (now - t0 > timeout_ns) {   // rank t never published: flag it, do not hang or trap
            atomicOr(abort, 1u << t);
            *(volatile uint32_t*)err_host = 1u;
            __threadfence_system();
            break;
        }
        __nanosleep(1000);
    }
}

void launch_wait_flags(const uint32_t* flags, int world, uint32_t epoch, unsigned long long timeout_ns,
                       uint32_t* abort, uint32_t* err_host, cudaStream_t s) {
    k_wait_flags<<<1, 32, 0, s>>>(flags, world, epoch, timeout_ns, abort, err_host);
}

void launch_normalise_push(const void* x, int dtype, int64_t n, int dim, const PushRows& out, int64_t row0,
                           const PushSignal& sig, cudaStream_t s) {
    const unsigned grid = (unsigned)std::max<int64_t>(1, (n + 7) / 8);   // >= 1 CTA: always publish
#define NV_NORMP_NS(NSV)                                                                              \
    case NSV:                                                                                         \
        if (dtype == CACHE_DTYPE_BF16)                                                                \
            k_normalise_push<__nv_bfloat16, NSV><<<grid, 256, 0, s>>>((const __nv_bfloat16*)x, n, out, row0, sig); \
        else                                                                                          \
            k_normalise_push<float, NSV><<<grid, 256, 0, s>>>((const float*)x, n, out, row0, sig);   \
        break;
    switch (dim / 32) {
        NV_NORMP_NS(2) NV_NORMP_NS(4) NV_NORMP_NS(6) NV_NORMP_NS(8) NV_NORMP_NS(10) NV_NORMP_NS(12)
        NV_NORMP_NS(14) NV_NORMP_NS(16) NV_NORMP_NS(18) NV_NORMP_NS(20) NV_NORMP_NS(22) NV_NORMP_NS(24)
        NV_NORMP_NS(26) NV_NORMP_NS(28) NV_NORMP_NS(30) NV_NORMP_NS(32)
        default: break;
    }
#undef NV_NORMP_NS
}

void launch_normalise(const void* x, int dtype, int64_t n, int dim, __nv_bfloat16* y, float* inv,
                      int32_t* status, cudaStream_t s, uint32_t* gk) {
    if (n <= 0) return;
    const unsigned grid = (unsigned)((n + 7) / 8);
#define NV_NORM_NS(NSV)                                                                                   \
    case NSV:                                                                                             \
        if (dtype == CACHE_DTYPE_BF16)                                                                    \
            k_normalise<__nv_bfloat16, NSV><<<grid, 256, 0, s>>>((const __nv_bfloat16*)x, n, y, inv, status, gk); \
        else                                                                                              \
            k_normalise<float, NSV><<<grid, 256, 0, s>>>((const float*)x, n, y, inv, status, gk);        \
        break;
    switch (dim / 32) {   // dim is a multiple of 64, <= 1024
        NV_NORM_NS(2) NV_NORM_NS(4) NV_NORM_NS(6) NV_NORM_NS(8) NV_NORM_NS(10) NV_NORM_NS(12)
        NV_NORM_NS(14) NV_NORM_NS(16) NV_NORM_NS(18) NV_NORM_NS(20) NV_NORM_NS(22) NV_NORM_NS(24)
        NV_NORM_NS(26) NV_NORM_NS(28) NV_NORM_NS(30) NV_NORM_NS(32)
        default: break;
    }
#undef NV_NORM_NS
}

// ---------------------------------------------------------------------------------------
// Streaming scan on CUDA cores (small batches, HBM bound).  Each warp owns whole entry
// rows: lane l loads 16-byte chunks 32c+l of a 2*dim-byte row (coalesced 512 B per warp
// instruction), multiplies them with the BQ queries held in registers (fp32 FMA on the
// exactly widened bf16 values), reduces across the warp with shuffles, scales by the
// entry's inv-norm and offers the result to a register top-k owned by lane b (query b).
// CTA-level merge of the 8 warp lists -> one partial record list per (CTA, query).
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ int4 ld_stream(const int4* p) {
    int4 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

template <int BQ, int KMAX, int NCH>
__global__ void __launch_bounds__(256, 2)
k_score_stream(const __nv_bfloat16* __restrict__ emb, const float* __restrict__ inv_e,
               const uint32_t* __restrict__ ids, int64_t n_slots, int dim,
               const __nv_bfloat16* __restrict__ qbuf, int64_t b_total, Rec* __restrict__ ws) {
    __shared__ Rec sm[8][BQ][KMAX];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int q0 = blockIdx.y * BQ;
    const int nvec = dim / 8;   // 16-byte chunks per row
    // queries -> registers (fp32), positions (32c + lane)*8 + [0,8)
    float qf[BQ][NCH * 8];
#pragma unroll
    for (int b = 0; b < BQ; ++b) {
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
            const int v = 32 * c + lane;
            int4 w = make_int4(0, 0, 0, 0);
            if (v < nvec && q0 + b < b_total)
                w = *reinterpret_cast<const int4*>(qbuf + (int64_t)(q0 + b) * dim + v * 8);
            const uint32_t ww[4] = {(uint32_t)w.x, (uint32_t)w.y, (uint32_t)w.z, (uint32_t)w.w};
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                qf[b][c * 8 + 2 * h] = __uint_as_float(ww[h] << 16);
                qf[b][c * 8 + 2 * h + 1] = __uint_as_float(ww[h] & 0xFFFF0000u);
            }
        }
    }
    TopK<KMAX> tk;
    tk.init();
    const int64_t per = (n_slots + gridDim.x - 1) / gridDim.x;
    const int64_t r0 = (int64_t)blockIdx.x * per;
    const int64_t r1 = min(n_slots, r0 + per);
    for (int64_t row = r0 + warp; row < r1; row += 8) {
        const int4* rp = reinterpret_cast<const int4*>(emb + row * dim);
        int4 e[NCH];
#pragma unroll
        for (int c = 0; c < NCH; ++c)
            e[c] = (32 * c + lane < nvec) ? ld_stream(rp + 32 * c + lane) : make_int4(0, 0, 0, 0);
        const float ie = __ldg(inv_e + row);
        float acc[BQ];
#pragma unroll
        for (int b = 0; b < BQ; ++b) acc[b] = 0.0f;
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
            const uint32_t ww[4] = {(uint32_t)e[c].x, (uint32_t)e[c].y, (uint32_t)e[c].z, (uint32_t)e[c].w};
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                const float lo = __uint_as_float(ww[h] << 16);
                const float hi = __uint_as_float(ww[h] & 0xFFFF0000u);
#pragma unroll
                for (int b = 0; b < BQ; ++b) {
                    acc[b] = fmaf(lo, qf[b][c * 8 + 2 * h], acc[b]);
                    acc[b] = fmaf(hi, qf[b][c * 8 + 2 * h + 1], acc[b]);
                }
            }
        }
#pragma unroll
        for (int b = 0; b < BQ; ++b) {
#pragma unroll
            for (int m = 16; m >= 1; m >>= 1) acc[b] += __shfl_xor_sync(0xFFFFFFFFu, acc[b], m);
        }
        float mine = 0.0f;
#pragma unroll
        for (int b = 0; b < BQ; ++b)
            if (lane == b) mine = acc[b] * ie;
        if (lane < BQ && q0 + lane < b_total) tk.offer(mine, (uint32_t)row, ids);
    }
    if (lane < BQ) {
#pragma unroll
        for (int i = 0; i < KMAX; ++i) { sm[warp][lane][i].key = tk.k[i]; sm[warp][lane][i].slot = tk.s[i]; }
    }
    __syncthreads();
    if (threadIdx.x < BQ && q0 + (int)threadIdx.x < b_total) {
        const int b = threadIdx.x;
        TopK<KMAX> m;
        m.init();
        for (int w = 0; w < 8; ++w)
#pragma unroll
            for (int i = 0; i < KMAX; ++i)
                if (sm[w][b][i].key) m.offer_key(sm[w][b][i].key, sm[w][b][i].slot);
        Rec* out = ws + ((int64_t)blockIdx.x * b_total + q0 + b) * KMAX;
#pragma unroll
        for (int i = 0; i < KMAX; ++i) { Rec r; r.key = m.k[i]; r.slot = m.s[i]; r.pad = 0; out[i] = r; }
    }
}

template <int BQ, int KMAX>
static void launch_stream_bq(int nch, dim3 g, const __nv_bfloat16* emb, const float* inv_e,
                             const uint32_t* ids, int64_t n_slots, int dim,
                             const __nv_bfloat16* qbuf, int64_t b, Rec* ws, cudaStream_t s) {
    switch (nch) {
        case 1: k_score_stream<BQ, KMAX, 1><<<g, 256, 0, s>>>(emb, inv_e, ids, n_slots, dim, qbuf, b, ws); break;
        case 2: k_score_stream<BQ, KMAX, 2><<<g, 256, 0, s>>>(emb, inv_e, ids, n_slots, dim, qbuf, b, ws); break;
        case 3: k_score_stream<BQ, KMAX, 3><<<g, 256, 0, s>>>(emb, inv_e, ids, n_slots, dim, qbuf, b, ws); break;
        default: k_score_stream<BQ, KMAX, 4><<<g, 256, 0, s>>>(emb, inv_e, ids, n_slots, dim, qbuf, b, ws); break;
    }
}

int stream_parts(int64_t n_slots, int64_t b) {
    const int bq = b >= 4 ? 4 : (b >= 2 ? 2 : 1);
    const int64_t groups = (b + bq - 1) / bq;
    int64_t parts = (148 * 4 + groups - 1) / groups;
    parts = std::max<int64_t>(1, std::min<int64_t>(parts, (n_slots + 511) / 512));
    return (int)parts;
}

void launch_score_stream(int kmax, const __nv_bfloat16* emb, const float* inv_e, const uint32_t* ids,
                         int64_t n_slots, int dim, const __nv_bfloat16* qbuf, int64_t b, Rec* ws,
                         int parts, cudaStream_t s) {
    const int bq = b >= 4 ? 4 : (b >= 2 ? 2 : 1);
    const int nch = (dim / 8 + 31) / 32;
    dim3 g((unsigned)parts, (unsigned)((b + bq - 1) / bq));
#define NV_STREAM_K(BQV)                                                                              \
    do {                                                                                              \
        if (kmax == 1) launch_stream_bq<BQV, 1>(nch, g, emb, inv_e, ids, n_slots, dim, qbuf, b, ws, s); \
        else if (kmax == 4) launch_stream_bq<BQV, 4>(nch, g, emb, inv_e, ids, n_slots, dim, qbuf, b, ws, s); \
        else launch_stream_bq<BQV, 16>(nch, g, emb, inv_e, ids, n_slots, dim, qbuf, b, ws, s);      \
    } while (0)
    if (bq == 4) NV_STREAM_K(4);
    else if (bq == 2) NV_STREAM_K(2);
    else NV_STREAM_K(1);
#undef NV_STREAM_K
}

// ---------------------------------------------------------------------------------------
// Finalize + gather: Q queries per 256-thread CTA (see FinCfg).  Warp w < Q merges query b0+w's `parts`
// partial lists under the total order (R3) -> top-k; its lane 0 applies the Fig. 11 map
// (largest j with s > thr[j], strict, compared in fp64 on the clamped fp32
// score), the knob (R20) and the hole rule (m = present & ((2 << j*) - 1),
// j = 31 - clz(m)) and counts the access.  Then the whole CTA streams the (up to Q) selected
// 32 KiB states into latent_out with 8 16-byte loads in flight per thread, so the
// merges of one CTA overlap the copies of the others.
// ---------------------------------------------------------------------------------------
// Queries per CTA: the gather is latency-bound on the bytes each SM has in flight (8 x 16 B
// loads per thread), so top-1 uses 4 queries per CTA capped at 32 registers (8 CTAs = 2,048
// threads per SM, all 1,024 CTAs of a 4,096-query batch resident at once); top-k > 1 keeps 8
// (its register top-k needs more registers).
// Small batches (b <= 512, e.g. C3's 1-32 queries) take one query per CTA: the whole CTA copies
// that query's state in one round of loads instead of four back-to-back rounds.
template <int KMAX>
struct FinCfg {
    static constexpr int Q = KMAX == 1 ? 4 : 8;
    static constexpr int MINB = KMAX == 1 ? 8 : 1;
};
constexpr int64_t kFinSmallB = 512;
template <int KMAX, int QPB = FinCfg<KMAX>::Q>
__global__ void __launch_bounds__(256, FinCfg<KMAX>::MINB)
k_finalize(const Rec* __restrict__ ws, int parts, int64_t B, int topk, const float* __restrict__ inv_q,
           const int32_t* __restrict__ qstatus, const uint32_t* __restrict__ ids,
           const uint32_t* __restrict__ present, const int32_t* __restrict__ lslot,
           uint32_t* __restrict__ fcnt, uint32_t* __restrict__ lastacc, uint32_t clock,
           const uint8_t* __restrict__ pool, int64_t latent_bytes,
           KMap km, uint64_t* __restrict__ out_ids, float* __restrict__ out_scores,
           int32_t* __restrict__ out_k, uint8_t* __restrict__ latent_out, void** __restrict__ out_ptr,
           int32_t* __restrict__ out_status) {
    constexpr int kFinQ = QPB;
    __shared__ unsigned long long s_keys[kFinQ][KMAX];
    __shared__ uint32_t s_slots[kFinQ][KMAX];
    __shared__ long long s_src[kFinQ];
    // launched with programmatic serialization behind the scan: wait for its records
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t b0 = (int64_t)blockIdx.x * kFinQ;
    const int64_t b = b0 + warp;
    const bool mine = warp < kFinQ && b < B;   // warp w merges query b0 + w (warps >= kFinQ only copy)
    if (lane == 0 && warp < kFinQ) s_src[warp] = -1;
    unsigned long long* s_key = s_keys[warp < kFinQ ? warp : 0];
    uint32_t* s_slot = s_slots[warp < kFinQ ? warp : 0];
    const int st = mine ? qstatus[b] : CACHE_ROW_ZERO_NORM;
    if (mine) {
        TopK<KMAX> tk;
        tk.init();
        if (st == CACHE_ROW_OK) {
            for (int p = lane; p < parts; p += 32) {
                const Rec* r = ws + ((int64_t)p * B + b) * KMAX;
                for (int i = 0; i < topk; ++i) {
                    const Rec rr = r[i];
                    if (rr.key == 0ull) break;
                    tk.offer_key(rr.key, rr.slot);
                }
            }
        }
        for (int i = 0; i < topk; ++i) {
            const unsigned long long m = warp_max_u64(tk.k[0]);
            if (m != 0ull && tk.k[0] == m) {
                s_key[i] = m;
                s_slot[i] = tk.s[0];
                tk.pop();
            }
            if (m == 0ull && lane == 0) s_key[i] = 0ull;
            __syncwarp();
        }
        if (lane == 0) {
            const float iq = st == CACHE_ROW_OK ? inv_q[b] : 0.0f;
            for (int i = 0; i < topk; ++i) {
                const unsigned long long key = s_key[i];
                out_ids[b * topk + i] = key ? (uint64_t)key_id(key) : CACHE_NO_ID;
                out_scores[b * topk + i] = key ? fminf(fmaxf(key_to_f32(key) * iq, -1.0f), 1.0f) : -INFINITY;
            }
            int K = 0;
            long long src = -1;
            if (s_key[0] != 0ull) {
                const float c = fminf(fmaxf(key_to_f32(s_key[0]) * iq, -1.0f), 1.0f);
                int jstar = -1;
                for (int j = 0; j < km.num_k; ++j)
                    if ((double)c > km.thr[j]) jstar = j;
                if (jstar >= 0) {
                    jstar = min(jstar + km.k_bias, km.num_k - 1);
                    const uint32_t slot = s_slot[0];
                    const uint32_t m = present[slot] & ((2u << jstar) - 1u);
                    if (m) {
                        const int j = 31 - __clz(m);
                        K = km.kv[j];
                        src = lslot[(int64_t)slot * km.num_k + j];
                        if (fcnt) {   // null: a read-only lookup (cache_query_peek) counts no access
                            atomicAdd(fcnt + (int64_t)slot * km.num_k + j, 1u);
                            lastacc[(int64_t)slot * km.num_k + j] = clock;   // LRU clock (same value for all hits)
                        }
                    }
                }
            }
            out_k[b] = K;
            if (out_status) out_status[b] = st;
            if (out_ptr) out_ptr[b] = (K > 0 && latent_out) ? (void*)(latent_out + b * latent_bytes) : nullptr;
            s_src[warp] = src;
        }
    }
    __syncthreads();
    if (!latent_out || !pool || latent_bytes <= 0) return;
    const int64_t nv = latent_bytes / 16;
    for (int w = 0; w < kFinQ; ++w) {
        const long long src = s_src[w];
        if (src < 0) continue;   // CTA-uniform
        const int4* sp = reinterpret_cast<const int4*>(pool + src * latent_bytes);
        int4* dp = reinterpret_cast<int4*>(latent_out + (b0 + w) * latent_bytes);
        int64_t i = threadIdx.x;
        for (; i + 7 * 256 < nv; i += 8 * 256) {
            int4 a[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) a[u] = ld_stream(sp + i + u * 256);
#pragma unroll
            for (int u = 0; u < 8; ++u) __stcs(dp + i + u * 256, a[u]);
        }
        for (; i < nv; i += 256) __stcs(dp + i, ld_stream(sp + i));
    }
}

void launch_finalize(int kmax, const Rec* ws, int parts, int64_t B, int topk, const float* inv_q,
                     const int32_t* qstatus, const uint32_t* ids, const uint32_t* present,
                     const int32_t* lslot, uint32_t* fcnt, uint32_t* lastacc, uint32_t clock,
                     const uint8_t* pool, int64_t latent_bytes,
                     const KMap& km, uint64_t* out_ids, float* out_scores, int32_t* out_k,
                     uint8_t* latent_out, void** out_ptr, int32_t* out_status, cudaStream_t s, bool pdl) {
    if (B <= 0) return;
    const bool small = B <= kFinSmallB;
    const int q = small ? 1 : (kmax == 1 ? FinCfg<1>::Q : FinCfg<16>::Q);
    const unsigned grid = (unsigned)((B + q - 1) / q);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;   // no PDL edge when the launch follows an event wait on a side stream
#define NV_FIN(KM)                                                                                      \
    cudaLaunchKernelEx(&cfg, small ? k_finalize<KM, 1> : k_finalize<KM>, ws, parts, B, topk, inv_q, qstatus, \
                       ids, present, lslot, fcnt, lastacc, clock, pool, latent_bytes, km, out_ids,          \
                       out_scores, out_k, latent_out, out_ptr, out_status)
    if (kmax == 1) NV_FIN(1);
    else if (kmax == 4) NV_FIN(4);
    else NV_FIN(16);
#undef NV_FIN
}

// ---------------------------------------------------------------------------------------
// Cache-selector profiling (Alg. 2): the similarity of each profiling prompt to its
// nearest cached prompt (the top-1 record of the scan, scored exactly as cache_query_batch
// reports it) against the quality the model reached at each K.  Reading R25: the threshold of
// K is the largest similarity at which some profiled image failed (quality <= alpha), so every
// profiled pair with s > threshold passed -- the runtime rule of Fig. 11 is strict '>'.
// ---------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256)
k_profile_reduce(const cache_shard_rec* __restrict__ recs, const float* __restrict__ inv_q,
                 const int32_t* __restrict__ qstatus, int64_t b, const float* __restrict__ quality, int num_k,
                 float alpha, uint32_t* __restrict__ fail, uint32_t* __restrict__ smin) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < b; i += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long key = recs[i].key;
        if (key == 0ull || qstatus[i] != CACHE_ROW_OK) continue;
        const float sc = fminf(fmaxf(key_to_f32(key) * inv_q[i], -1.0f), 1.0f);
        const uint32_t o = orderable_f32(sc);
        atomicMin(smin, o);
        for (int j = 0; j < num_k; ++j)
            if (quality[(int64_t)j * b + i] <= alpha) atomicMax(&fail[j], o);
    }
}

void launch_profile_reduce(const cache_shard_rec* recs, const float* inv_q, const int32_t* qstatus, int64_t b,
                           const float* quality, int num_k, float alpha, uint32_t* fail, uint32_t* smin,
                           cudaStream_t s) {
    if (b <= 0) return;
    const unsigned grid = (unsigned)std::min<int64_t>(148 * 4, (b + 255) / 256);
    k_profile_reduce<<<grid, 256, 0, s>>>(recs, inv_q, qstatus, b, quality, num_k, alpha, fail, smin);
}

// ---------------------------------------------------------------------------------------
// Insert: commit normalised rows into their slots and copy latent payloads.
// ---------------------------------------------------------------------------------------
__global__ void __launch_bounds__(128)
k_insert_commit(const __nv_bfloat16* __restrict__ ystage, const float* __restrict__ invstage,
                const InsertPlan* __restrict__ plan, int64_t n_valid, int dim, int num_k,
                __nv_bfloat16* __restrict__ emb, float* __restrict__ inv_e, uint32_t* __restrict__ ids,
                uint32_t* __restrict__ present, int32_t* __restrict__ lslot, uint32_t* __restrict__ fcnt,
                uint32_t* __restrict__ lastacc, uint32_t clock) {
    const int64_t i = blockIdx.x;
    if (i >= n_valid) return;
    const InsertPlan p = plan[i];
    const int4* src = reinterpret_cast<const int4*>(ystage + p.src_row * (int64_t)dim);
    int4* dst = reinterpret_cast<int4*>(emb + p.slot * (int64_t)dim);
    for (int v = threadIdx.x; v < dim / 8; v += 128) dst[v] = src[v];
    if (threadIdx.x < num_k) {
        lslot[p.slot * num_k + threadIdx.x] = p.lslot[threadIdx.x];
        fcnt[p.slot * num_k + threadIdx.x] = 0u;
        lastacc[p.slot * num_k + threadIdx.x] = clock;   // LRU: a fresh item counts as just used
    }
    if (threadIdx.x == 0) {
        inv_e[p.slot] = invstage[p.src_row];
        ids[p.slot] = p.id;
        present[p.slot] = p.mask;
    }
}

__global__ void __launch_bounds__(128)
k_copy_latents(const uint8_t* __restrict__ src, const CopyPlan* __restrict__ plan, int64_t n,
               int64_t latent_bytes, uint8_t* __restrict__ pool) {
    const int64_t i = blockIdx.x;
    if (i >= n) return;
    const CopyPlan p = plan[i];
    const int4* sp = reinterpret_cast<const int4*>(src + p.src_item * latent_bytes);
    int4* dp = reinterpret_cast<int4*>(pool + p.dst_slot * latent_bytes);
    for (int64_t v = threadIdx.x; v < latent_bytes / 16; v += 128) dp[v] = sp[v];
}

void launch_insert_commit(const __nv_bfloat16* ystage, const float* invstage, const InsertPlan* plan,
                          int64_t n_valid, int dim, int num_k, __nv_bfloat16* emb, float* inv_e,
                          uint32_t* ids, uint32_t* present, int32_t* lslot, uint32_t* fcnt, uint32_t* lastacc,
                          uint32_t clock, cudaStream_t s) {
    if (n_valid > 0)
        k_insert_commit<<<(unsigned)n_valid, 128, 0, s>>>(ystage, invstage, plan, n_valid, dim, num_k,
                                                          emb, inv_e, ids, present, lslot, fcnt, lastacc, clock);
}

void launch_copy_latents(const uint8_t* src, const CopyPlan* plan, int64_t n, int64_t latent_bytes,
                         uint8_t* pool, cudaStream_t s) {
    if (n > 0) k_copy_latents<<<(unsigned)n, 128, 0, s>>>(src, plan, n, latent_bytes, pool);
}

// ---------------------------------------------------------------------------------------
// Eviction.  Item key (reading R11): min(f*K, 2^29-1) << 35 | id << 3 | j,
// unique per item, ascending = evicted first.  Exact selection of the n smallest keys by an
// 8-pass MSB-first radix select (8-bit digits): histogram of keys matching the prefix ->
// pick the digit holding the remaining-th key.  Then every key <= the selected key is
// evicted: presence bit cleared, latent slot freed; entries left with no K are dirty and
// are invalidated (inv_norm = NaN) in the same kernel.
// ---------------------------------------------------------------------------------------
// item_score / item_key / entry_key / DigitRun: evict.cuh (shared with evict.cu).

template <int POLICY, int GRAN>
__global__ void __launch_bounds__(256)
k_evict_hist(const uint32_t* __restrict__ present, const uint32_t* __restrict__ fcnt,
             const uint32_t* __restrict__ lastacc, const uint32_t* __restrict__ ids, int64_t n_slots, KMap km,
             const EvictState* __restrict__ st, int shift, unsigned int* __restrict__ hist, PushHist ph,
             PushSignal sig) {
    if (ph.world && push_aborted(sig)) return;
    __shared__ unsigned int sh[256];
    sh[threadIdx.x] = 0;
    __syncthreads();
    const int nk = km.num_k;
    int kv[CACHE_MAX_K];
#pragma unroll
    for (int j = 0; j < CACHE_MAX_K; ++j) kv[j] = km.kv[j];
    const unsigned long long prefix = st->prefix, mask = st->mask;
    DigitRun run;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n_slots;
         e += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t m = present[e];
        if (!m) continue;
        const uint32_t id = ids[e];
        if constexpr (GRAN == CACHE_EVICT_ENTRY) {
            const unsigned long long key = entry_key<POLICY>(fcnt, lastacc, e, m, id, nk, kv);
            if ((key & mask) == prefix) run.add(sh, (unsigned)(key >> shift) & 255u);
        } else {
#pragma unroll
            for (int j = 0; j < CACHE_MAX_K; ++j) {
                if (j >= nk || !((m >> j) & 1u)) continue;
                const unsigned long long key =
                    item_key(item_score<POLICY>(fcnt, lastacc, e * nk + j, kv[j]), id, j);
                if ((key & mask) == prefix) run.add(sh, (unsigned)(key >> shift) & 255u);
            }
        }
    }
    run.flush(sh);
    __syncthreads();
    if (ph.world == 0) {
        if (sh[threadIdx.x]) atomicAdd(&hist[threadIdx.x], sh[threadIdx.x]);
    } else {   // fused all-reduce: add into every rank's accumulator, then publish the pass
        if (sh[threadIdx.x])
            for (int r = 0; r < ph.world; ++r) atomicAdd(ph.dst[r] + threadIdx.x, sh[threadIdx.x]);
        push_signal(sig);
    }
}

__global__ void k_evict_pick(unsigned int* __restrict__ hist, EvictState* __restrict__ st, int shift) {
    if (threadIdx.x == 0) {
        unsigned long long cum = 0;
        const unsigned long long rem = st->remaining;
        for (int d = 0; d < 256; ++d) {
            if (cum + hist[d] >= rem) {
                st->prefix |= (unsigned long long)d << shift;
                st->remaining = rem - cum;
                break;
            }
            cum += hist[d];
        }
        st->mask |= 255ull << shift;
    }
    __syncthreads();
    for (int d = threadIdx.x; d < 256; d += blockDim.x) hist[d] = 0;
}

// warp_claim: evict.cuh.

template <int POLICY, int GRAN>
__global__ void __launch_bounds__(256)
k_evict_apply(uint32_t* __restrict__ present, uint32_t* __restrict__ fcnt, const uint32_t* __restrict__ lastacc,
              const uint32_t* __restrict__ ids, const int32_t* __restrict__ lslot, float* __restrict__ inv_e,
              int64_t n_slots, KMap km,
              const EvictState* __restrict__ st, unsigned long long* __restrict__ ev_key,
              unsigned long long* __restrict__ ev_pool, int64_t* __restrict__ ev_eslot,
              unsigned long long* __restrict__ counters, unsigned long long* __restrict__ dirty_slot,
              unsigned long long* __restrict__ dirty_id, unsigned long long ev_cap, unsigned long long dirty_cap,
              const uint32_t* __restrict__ abort) {
    if (abort && *(volatile const uint32_t*)abort) return;   // the distributed selection did not finish
    const unsigned long long T = st->prefix;
    const int lane = threadIdx.x & 31;
    const int nk = km.num_k;
    int kv[CACHE_MAX_K];
#pragma unroll
    for (int j = 0; j < CACHE_MAX_K; ++j) kv[j] = km.kv[j];
    for (int64_t e0 = blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31); e0 < n_slots;
         e0 += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = e0 + lane;
        const uint32_t m = e < n_slots ? present[e] : 0u;
        const uint32_t id = m ? ids[e] : 0u;
        if constexpr (GRAN == CACHE_EVICT_ENTRY) {
            // whole entry: all stored states freed (their pool slots listed in ev_pool, counted
            // in counters[2]), entry invalidated; one record per evicted entry in both lists
            const unsigned long long key = m ? entry_key<POLICY>(fcnt, lastacc, e, m, id, nk, kv) : 0ull;
            const bool take = m && key <= T;
            const unsigned long long at = warp_claim(&counters[0], take, lane);
#pragma unroll
            for (int j = 0; j < CACHE_MAX_K; ++j) {
                if (j >= nk) break;   // warp-uniform
                const bool freed = take && ((m >> j) & 1u);
                const unsigned long long pat = warp_claim(&counters[2], freed, lane);
                if (freed && pat < ev_cap * (unsigned long long)nk)
                    ev_pool[pat] = (unsigned long long)(uint32_t)lslot[e * nk + j];
            }
            if (take) {
                for (int j = 0; j < nk; ++j) fcnt[e * nk + j] = 0u;
                present[e] = 0u;
                inv_e[e] = __int_as_float(0x7FC00000);
                if (at < ev_cap && at < dirty_cap) {   // overflow = caller error, reported by the host
                    ev_key[at] = key;
                    dirty_slot[at] = (unsigned long long)e;
                    dirty_id[at] = id;
                }
            }
            (void)warp_claim(&counters[1], take, lane);   // dirty count = evicted count in entry mode
        } else {
            uint32_t keep = m;
#pragma unroll
            for (int j = 0; j < CACHE_MAX_K; ++j) {
                if (j >= nk) break;   // warp-uniform
                const bool has = (m >> j) & 1u;
                const unsigned long long key =
                    has ? item_key(item_score<POLICY>(fcnt, lastacc, e * nk + j, kv[j]), id, j) : 0ull;
                const bool take = has && key <= T;
                const unsigned long long at = warp_claim(&counters[0], take, lane);
                if (take) {
                    keep &= ~(1u << j);
                    if (at < ev_cap) {
                        ev_key[at] = key;
                        ev_pool[at] = (unsigned long long)(uint32_t)lslot[e * nk + j];
                        ev_eslot[at] = e;
                    }
                    fcnt[e * nk + j] = 0u;
                }
            }
            const bool dirty = m && keep == 0u;
            if (keep != m) {
                present[e] = keep;
                if (dirty) inv_e[e] = __int_as_float(0x7FC00000);
            }
            const unsigned long long at = warp_claim(&counters[1], dirty, lane);
            if (dirty && at < dirty_cap) {
                dirty_slot[at] = (unsigned long long)e;
                dirty_id[at] = id;
            }
        }
    }
}

// Grid = one wave of resident CTAs (the sweeps are grid-stride loops).
template <typename K>
static int one_wave(K kern) {
    int bps = 0, dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern, 256, 0) != cudaSuccess || bps < 1) bps = 4;
    return bps * sms;
}

// NV_EVICT_DISPATCH: evict.cuh.

void launch_evict_hist(const uint32_t* present, const uint32_t* fcnt, const uint32_t* lastacc, const uint32_t* ids,
                       int64_t n_slots, const KMap& km, const EvictState* st, int pass, unsigned int* hist,
                       cudaStream_t s) {
#define NV_HIST(P, G)                                                                                  \
    do {                                                                                               \
        static const int wave = one_wave(k_evict_hist<P, G>);                                          \
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(wave, (n_slots + 255) / 256));   \
        k_evict_hist<P, G><<<grid, 256, 0, s>>>(present, fcnt, lastacc, ids, n_slots, km, st, 56 - 8 * pass, hist, \
                                                PushHist{}, PushSignal{});                             \
    } while (0)
    NV_EVICT_DISPATCH(NV_HIST);
#undef NV_HIST
}

void launch_evict_hist_push(const uint32_t* present, const uint32_t* fcnt, const uint32_t* lastacc,
                            const uint32_t* ids, int64_t n_slots, const KMap& km, const EvictState* st, int pass,
                            const PushHist& ph, const PushSignal& sig, cudaStream_t s) {
#define NV_HISTP(P, G)                                                                                 \
    do {                                                                                               \
        static const int wave = one_wave(k_evict_hist<P, G>);                                          \
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(wave, (n_slots + 255) / 256));   \
        k_evict_hist<P, G><<<grid, 256, 0, s>>>(present, fcnt, lastacc, ids, n_slots, km, st, 56 - 8 * pass,  \
                                                nullptr, ph, sig);                                     \
    } while (0)
    NV_EVICT_DISPATCH(NV_HISTP);
#undef NV_HISTP
}

// Distributed fused eviction: this rank's 4,096-bin level histogram added into every rank's
// arena accumulator (P2P atomics over NVLink), then the grid publishes the level's epoch flag.
__global__ void __launch_bounds__(256) k_push_hist_bins(const uint32_t* __restrict__ local, int nbins, PushHist ph,
                                                        PushSignal sig) {
    if (push_aborted(sig)) return;
    for (int i = blockIdx.x * 256 + threadIdx.x; i < nbins; i += gridDim.x * 256) {
        const uint32_t v = local[i];
        if (v)
            for (int r = 0; r < ph.world; ++r) atomicAdd(ph.dst[r] + i, v);
    }
    push_signal(sig);
}

void launch_push_hist_bins(const uint32_t* local, int nbins, const PushHist& ph, const PushSignal& sig, cudaStream_t s) {
    k_push_hist_bins<<<(nbins + 255) / 256, 256, 0, s>>>(local, nbins, ph, sig);
}

void launch_evict_pick(unsigned int* hist, EvictState* st, int pass, cudaStream_t s) {
    k_evict_pick<<<1, 256, 0, s>>>(hist, st, 56 - 8 * pass);
}

// ---------------------------------------------------------------------------------------
// Sharded lookup.
// k_local_merge: one warp per query merges the scorer's partial lists of this shard into
// one top-k list of 16-byte shard records (key, slot, presence mask, owner rank).
// k_merge_sharded: one CTA per local query merges the world lists, applies Fig. 11 + the
// hole rule with the record's presence mask, then reads the winner's latent-slot table
// entry and the 32 KiB state directly from the OWNER's memory (peer pointers over NVLink,
// or local pointers for the own rank) and counts the access with an atomic on the owner's
// counter -- the fetch is fused into the merge kernel, no second collective.
// ---------------------------------------------------------------------------------------
// kPush = false: records -> out[b][topk] (all-gathered by the caller).  kPush = true: the
// records of global row b go straight into its owner's inbox (rank b / nb, row b % nb, sender
// slot `owner`) over NVLink, then the grid publishes the epoch (record push fused with the
// local merge: no collective).
template <int KMAX, bool kPush>
__global__ void __launch_bounds__(256)
k_local_merge(const Rec* __restrict__ ws, int parts, int64_t B, int topk, const int32_t* __restrict__ qstatus,
              const uint32_t* __restrict__ present, int owner, cache_shard_rec* __restrict__ out, PushRecs dst,
              PushSignal sig) {
    if (kPush && push_aborted(sig)) return;
    const int lane = threadIdx.x & 31;
    const int64_t b = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    if (b < B) {
        cache_shard_rec* o_row = kPush ? dst.inbox[b / dst.nb] + ((int64_t)dst.me * dst.nb + b % dst.nb) * topk
                                       : out + b * topk;
        TopK<KMAX> tk;
        tk.init();
        if (qstatus[b] == CACHE_ROW_OK) {
            for (int p = lane; p < parts; p += 32) {
                const Rec* r = ws + ((int64_t)p * B + b) * KMAX;
                for (int i = 0; i < topk; ++i) {
                    const Rec rr = r[i];
                    if (rr.key == 0ull) break;
                    tk.offer_key(rr.key, rr.slot);
                }
            }
        }
        for (int i = 0; i < topk; ++i) {
            const unsigned long long m = warp_max_u64(tk.k[0]);
            if (m != 0ull && tk.k[0] == m) {
                cache_shard_rec o;
                o.key = m;
                o.slot = tk.s[0];
                o.present_mask = (uint8_t)(present[tk.s[0]] & 0xFFu);
                o.owner = (uint8_t)owner;
                o.reserved = 0;
                o_row[i] = o;
                tk.pop();
            }
            if (m == 0ull && lane == 0) {
                cache_shard_rec o{};
                o_row[i] = o;
            }
        }
    }
    if (kPush) push_signal(sig);
}

void launch_local_merge(int kmax, const Rec* ws, int parts, int64_t B, int topk, const int32_t* qstatus,
                        const uint32_t* present, int owner, cache_shard_rec* out, cudaStream_t s) {
    if (B <= 0) return;
    const unsigned grid = (unsigned)((B + 7) / 8);
    const PushRecs d{};
    const PushSignal g{};
    if (kmax == 1) k_local_merge<1, false><<<grid, 256, 0, s>>>(ws, parts, B, topk, qstatus, present, owner, out, d, g);
    else if (kmax == 4) k_local_merge<4, false><<<grid, 256, 0, s>>>(ws, parts, B, topk, qstatus, present, owner, out, d, g);
    else k_local_merge<16, false><<<grid, 256, 0, s>>>(ws, parts, B, topk, qstatus, present, owner, out, d, g);
}

void launch_local_merge_push(int kmax, const Rec* ws, int parts, int64_t B, int topk, const int32_t* qstatus,
                             const uint32_t* present, int owner, const PushRecs& dst, const PushSignal& sig,
                             cudaStream_t s) {
    const unsigned grid = (unsigned)std::max<int64_t>(1, (B + 7) / 8);   // >= 1 CTA: always publish
    if (kmax == 1) k_local_merge<1, true><<<grid, 256, 0, s>>>(ws, parts, B, topk, qstatus, present, owner, nullptr, dst, sig);
    else if (kmax == 4) k_local_merge<4, true><<<grid, 256, 0, s>>>(ws, parts, B, topk, qstatus, present, owner, nullptr, dst, sig);
    else k_local_merge<16, true><<<grid, 256, 0, s>>>(ws, parts, B, topk, qstatus, present, owner, nullptr, dst, sig);
}

template <int KMAX>
__global__ void __launch_bounds__(128)
k_merge_sharded(const cache_shard_rec* __restrict__ recs, int64_t rec_stride, int64_t rec_row0, int world,
                int64_t row0, int topk,
                const float* __restrict__ inv_q, const int32_t* __restrict__ qstatus, PeerPtrs peers,
                uint32_t clock, int64_t latent_bytes, KMap km, uint64_t* __restrict__ out_ids,
                float* __restrict__ out_scores,
                int32_t* __restrict__ out_k, uint8_t* __restrict__ latent_out, void** __restrict__ out_ptr,
                int32_t* __restrict__ out_status) {
    if (peers.abort && *(volatile const uint32_t*)peers.abort) return;   // a peer failed: no P2P reads
    __shared__ unsigned long long s_key[KMAX];
    __shared__ uint32_t s_slot[KMAX];
    __shared__ long long s_src;
    __shared__ int s_owner;
    const int64_t i = blockIdx.x;          // local output row
    const int64_t g = row0 + i;            // global query row
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int st = qstatus[g];
    if (warp == 0) {
        // candidate = (key, slot, owner << 8 | mask) -- keys are unique across shards (ids are)
        unsigned long long ck[KMAX];
        uint32_t cs[KMAX], cm[KMAX];
#pragma unroll
        for (int t = 0; t < KMAX; ++t) { ck[t] = 0ull; cs[t] = 0u; cm[t] = 0u; }
        if (st == CACHE_ROW_OK) {
            for (int idx = lane; idx < world * topk; idx += 32) {
                const int r = idx / topk, t = idx - r * topk;
                const cache_shard_rec rec = recs[((int64_t)r * rec_stride + rec_row0 + i) * topk + t];
                if (rec.key == 0ull || rec.key <= ck[KMAX - 1]) continue;
                const uint32_t meta = ((uint32_t)rec.owner << 8) | rec.present_mask;
#pragma unroll
                for (int u = KMAX - 1; u > 0; --u) {
                    if (rec.key > ck[u - 1]) { ck[u] = ck[u - 1]; cs[u] = cs[u - 1]; cm[u] = cm[u - 1]; }
                    else if (rec.key > ck[u]) { ck[u] = rec.key; cs[u] = rec.slot; cm[u] = meta; }
                }
                if (rec.key > ck[0]) { ck[0] = rec.key; cs[0] = rec.slot; cm[0] = meta; }
            }
        }
        __shared__ uint32_t s_meta0;
        for (int t = 0; t < topk; ++t) {
            const unsigned long long m = warp_max_u64(ck[0]);
            if (m != 0ull && ck[0] == m) {
                s_key[t] = m;
                s_slot[t] = cs[0];
                if (t == 0) s_meta0 = cm[0];
#pragma unroll
                for (int u = 0; u < KMAX - 1; ++u) { ck[u] = ck[u + 1]; cs[u] = cs[u + 1]; cm[u] = cm[u + 1]; }
                ck[KMAX - 1] = 0ull;
            }
            if (m == 0ull && lane == 0) s_key[t] = 0ull;
            __syncwarp();
        }
        if (lane == 0) {
            const float iq = st == CACHE_ROW_OK ? inv_q[g] : 0.0f;
            for (int t = 0; t < topk; ++t) {
                const unsigned long long key = s_key[t];
                out_ids[i * topk + t] = key ? (uint64_t)key_id(key) : CACHE_NO_ID;
                out_scores[i * topk + t] = key ? fminf(fmaxf(key_to_f32(key) * iq, -1.0f), 1.0f) : -INFINITY;
            }
            int K = 0, owner = 0;
            long long src = -1;
            if (s_key[0] != 0ull) {
                const float c = fminf(fmaxf(key_to_f32(s_key[0]) * iq, -1.0f), 1.0f);
                int jstar = -1;
                for (int j = 0; j < km.num_k; ++j)
                    if ((double)c > km.thr[j]) jstar = j;
                if (jstar >= 0) {
                    jstar = min(jstar + km.k_bias, km.num_k - 1);
                    owner = (int)(s_meta0 >> 8);
                    const uint32_t m = (s_meta0 & 0xFFu) & ((2u << jstar) - 1u);
                    if (m) {
                        const int j = 31 - __clz(m);
                        K = km.kv[j];
                        const int64_t e = (int64_t)s_slot[0] * km.num_k + j;
                        src = peers.lslot[owner][e];                  // P2P read of the owner's table
                        atomicAdd(peers.fcnt[owner] + e, 1u);         // P2P atomic on the owner's f
                        peers.lastacc[owner][e] = clock;              // P2P store of the LRU clock
                    }
                }
            }
            out_k[i] = K;
            if (out_status) out_status[i] = st;
            if (out_ptr) out_ptr[i] = (K > 0 && latent_out) ? (void*)(latent_out + i * latent_bytes) : nullptr;
            s_src = src;
            s_owner = owner;
        }
    }
    __syncthreads();
    const long long src = s_src;
    if (src >= 0 && latent_out && latent_bytes > 0) {
        const int4* sp = reinterpret_cast<const int4*>(peers.pool[s_owner] + src * latent_bytes);
        int4* dp = reinterpret_cast<int4*>(latent_out + i * latent_bytes);
        const int64_t nv = latent_bytes / 16;
        int64_t v = threadIdx.x;
        for (; v + 3 * 128 < nv; v += 4 * 128) {
            const int4 a0 = sp[v], a1 = sp[v + 128], a2 = sp[v + 256], a3 = sp[v + 384];
            __stcs(dp + v, a0);
            __stcs(dp + v + 128, a1);
            __stcs(dp + v + 256, a2);
            __stcs(dp + v + 384, a3);
        }
        for (; v < nv; v += 128) __stcs(dp + v, sp[v]);
    }
}

void launch_merge_sharded(int kmax, const cache_shard_rec* recs, int64_t rec_stride, int64_t rec_row0, int world,
                          int64_t row0, int64_t nb, int topk, const float* inv_q, const int32_t* qstatus,
                          const PeerPtrs& peers, uint32_t clock, int64_t latent_bytes, const KMap& km,
                          uint64_t* out_ids, float* out_scores, int32_t* out_k, uint8_t* latent_out, void** out_ptr,
                          int32_t* out_status, cudaStream_t s) {
    if (nb <= 0) return;
#define NV_MS(KM)                                                                                              \
    k_merge_sharded<KM><<<(unsigned)nb, 128, 0, s>>>(recs, rec_stride, rec_row0, world, row0, topk, inv_q,     \
                                                     qstatus, peers, clock, latent_bytes, km, out_ids,         \
                                                     out_scores, out_k, latent_out, out_ptr, out_status)
    if (kmax == 1) NV_MS(1);
    else if (kmax == 4) NV_MS(4);
    else NV_MS(16);
#undef NV_MS
}

void launch_evict_apply(uint32_t* present, uint32_t* fcnt, const uint32_t* lastacc, const uint32_t* ids,
                        const int32_t* lslot, float* inv_e, int64_t n_slots, const KMap& km, const EvictState* st,
                        unsigned long long* ev_key, unsigned long long* ev_pool, int64_t* ev_eslot,
                        unsigned long long* counters, unsigned long long* dirty_slot, unsigned long long* dirty_id,
                        int64_t ev_cap, int64_t dirty_cap, cudaStream_t s, const uint32_t* abort) {
#define NV_APPLY(P, G)                                                                                 \
    do {                                                                                               \
        static const int wave = one_wave(k_evict_apply<P, G>);                                         \
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(wave, (n_slots + 255) / 256));   \
        k_evict_apply<P, G><<<grid, 256, 0, s>>>(present, fcnt, lastacc, ids, lslot, inv_e, n_slots, km, st,  \
                                                 ev_key, ev_pool, ev_eslot, counters, dirty_slot, dirty_id, \
                                                 (unsigned long long)ev_cap, (unsigned long long)dirty_cap, abort); \
    } while (0)
    NV_EVICT_DISPATCH(NV_APPLY);
#undef NV_APPLY
}

}  // namespace nv
