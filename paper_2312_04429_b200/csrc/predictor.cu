// predictor.cu -- match predictor: a linear one-class SVM
// f(x) = <w, x> - rho over the unit-scaled cached embeddings, trained on the GPU (reading
// R22): per epoch
//   k_pred_margins   m_e = <w, x~_e> * inv_e for every live slot (a GEMV over the bf16 rows;
//                    one warp per row, 128-bit loads) -> orderable u32 keys
//   k_sel_hist/pick  exact k-th smallest key, k = ceil(nu n) (4 radix passes of 8 bits)
//                    -> rho = that margin (the exact minimiser of J in rho)
//   k_pred_viol      deterministic per-block sums of x~_e * inv_e over the violators
//                    (m_e < rho), fixed row ranges and order
//   k_pred_update    w <- w - eta (nu w - g / n) / nu        (one thread per column)
// and evaluated per query by k_predict (one warp per query: <w, q~> * inv_q - rho >= 0).
#include "kernels.h"

namespace nv {

__device__ __forceinline__ float bf16lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }

// <w, row> over dim bf16 values; w in shared memory; warp-cooperative, result in every lane
__device__ __forceinline__ float warp_dot_bf16(const __nv_bfloat16* __restrict__ row, const float* __restrict__ ws,
                                               int dim, int lane) {
    float acc = 0.0f;
    const int4* rp = reinterpret_cast<const int4*>(row);
    for (int v = lane; v < dim / 8; v += 32) {
        const int4 q = __ldg(rp + v);
        const uint32_t u[4] = {(uint32_t)q.x, (uint32_t)q.y, (uint32_t)q.z, (uint32_t)q.w};
#pragma unroll
        for (int h = 0; h < 4; ++h) {
            acc = fmaf(bf16lo(u[h]), ws[v * 8 + 2 * h], acc);
            acc = fmaf(bf16hi(u[h]), ws[v * 8 + 2 * h + 1], acc);
        }
    }
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, m);
    return acc;
}

__global__ void __launch_bounds__(256)
k_pred_margins(const __nv_bfloat16* __restrict__ emb, const float* __restrict__ inv_e, int64_t n_slots, int dim,
               const float* __restrict__ w, uint32_t* __restrict__ keys) {
    extern __shared__ float ws[];
    for (int i = threadIdx.x; i < dim; i += blockDim.x) ws[i] = w[i];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * 8;
    for (int64_t e = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5); e < n_slots; e += nw) {
        const float ie = inv_e[e];
        if (isnan(ie)) {   // empty slot: never selected, never a violator
            if (lane == 0) keys[e] = 0xFFFFFFFFu;
            continue;
        }
        const float m = warp_dot_bf16(emb + e * dim, ws, dim, lane) * ie;
        if (lane == 0) keys[e] = orderable_f32(m);   // ascending key = ascending margin
    }
}

__global__ void __launch_bounds__(256)
k_sel_hist(const uint32_t* __restrict__ keys, int64_t n, const EvictState* __restrict__ st, int shift,
           unsigned int* __restrict__ hist) {
    __shared__ unsigned int sh[256];
    sh[threadIdx.x] = 0;
    __syncthreads();
    const uint32_t prefix = (uint32_t)st->prefix, mask = (uint32_t)st->mask;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t k = keys[i];
        if ((k & mask) == prefix) atomicAdd(&sh[(k >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (sh[threadIdx.x]) atomicAdd(&hist[threadIdx.x], sh[threadIdx.x]);
}

__global__ void k_sel_pick(unsigned int* __restrict__ hist, EvictState* __restrict__ st, int shift) {
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

// per-block partial sums of the violator rows (key < kth key); block b owns rows [b*per, ...)
__global__ void __launch_bounds__(256)
k_pred_viol(const __nv_bfloat16* __restrict__ emb, const float* __restrict__ inv_e, const uint32_t* __restrict__ keys,
            int64_t n_slots, int dim, const EvictState* __restrict__ st, int all_rows, float* __restrict__ gpart,
            unsigned int* __restrict__ cpart) {
    const uint32_t kkey = (uint32_t)st->prefix;
    const int64_t per = (n_slots + gridDim.x - 1) / gridDim.x;
    const int64_t r0 = (int64_t)blockIdx.x * per, r1 = min(n_slots, r0 + per);
    float acc[4] = {0.f, 0.f, 0.f, 0.f};   // columns t, t+256, t+512, t+768
    unsigned int cnt = 0;
    for (int64_t e = r0; e < r1; ++e) {
        const uint32_t k = keys[e];
        const bool take = all_rows ? (k != 0xFFFFFFFFu) : (k < kkey);
        if (!take) continue;   // block-uniform
        const float ie = inv_e[e];
        const __nv_bfloat16* row = emb + e * dim;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int col = threadIdx.x + 256 * u;
            if (col < dim) acc[u] += __bfloat162float(row[col]) * ie;
        }
        ++cnt;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int col = threadIdx.x + 256 * u;
        if (col < dim) gpart[(int64_t)blockIdx.x * dim + col] = acc[u];
    }
    if (threadIdx.x == 0) cpart[blockIdx.x] = cnt;
}

// mode 0: w = g / n_sel (initial mean direction); mode 1: subgradient step on nu J
__global__ void k_pred_update(const float* __restrict__ gpart, const unsigned int* __restrict__ cpart, int nblk,
                              int dim, float* __restrict__ w, double nu, double eta, int64_t n, int mode) {
    const int col = blockIdx.x * blockDim.x + threadIdx.x;
    if (col >= dim) return;
    double g = 0.0;
    unsigned long long c = 0;
    for (int b = 0; b < nblk; ++b) {   // fixed order: deterministic
        g += (double)gpart[(int64_t)b * dim + col];
        c += cpart[b];
    }
    if (mode == 0) {
        w[col] = c ? (float)(g / (double)c) : 0.0f;
    } else {
        const double wv = (double)w[col];
        w[col] = (float)(wv - eta * (nu * wv - g / (double)n) / nu);
    }
}

__global__ void k_pred_finish(const EvictState* __restrict__ st, float* __restrict__ rho) {
    *rho = key_to_f32((unsigned long long)(uint32_t)st->prefix << 32);
}

__global__ void __launch_bounds__(256)
k_predict(const __nv_bfloat16* __restrict__ qbuf, const float* __restrict__ inv_q, const int32_t* __restrict__ qstatus,
          int64_t b, int dim, const float* __restrict__ w, const float* __restrict__ rho, uint8_t* __restrict__ flags,
          float* __restrict__ margin) {
    extern __shared__ float ws[];
    for (int i = threadIdx.x; i < dim; i += blockDim.x) ws[i] = w[i];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t q = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    if (q >= b) return;
    const float f = qstatus[q] == CACHE_ROW_OK ? warp_dot_bf16(qbuf + q * dim, ws, dim, lane) * inv_q[q] - *rho
                                               : -INFINITY;
    if (lane == 0) {
        if (flags) flags[q] = f >= 0.0f ? 1 : 0;
        if (margin) margin[q] = f;
    }
}

// ---------------------------------------------------------------------------------------
void pred_margins(const __nv_bfloat16* emb, const float* inv_e, int64_t n_slots, int dim, const float* w,
                  uint32_t* keys, cudaStream_t s) {
    const int grid = (int)std::min<int64_t>(148 * 8, (n_slots + 7) / 8);
    k_pred_margins<<<grid, 256, dim * 4, s>>>(emb, inv_e, n_slots, dim, w, keys);
}
void pred_select(const uint32_t* keys, int64_t n, EvictState* st, unsigned int* hist, cudaStream_t s) {
    const int grid = (int)std::min<int64_t>(148 * 4, (n + 255) / 256 + 1);
    for (int pass = 0; pass < 4; ++pass) {
        const int shift = 24 - 8 * pass;
        k_sel_hist<<<grid, 256, 0, s>>>(keys, n, st, shift, hist);
        k_sel_pick<<<1, 256, 0, s>>>(hist, st, shift);
    }
}
void pred_viol(const __nv_bfloat16* emb, const float* inv_e, const uint32_t* keys, int64_t n_slots, int dim,
               const EvictState* st, int all_rows, float* gpart, unsigned int* cpart, int nblk, cudaStream_t s) {
    k_pred_viol<<<nblk, 256, 0, s>>>(emb, inv_e, keys, n_slots, dim, st, all_rows, gpart, cpart);
}
void pred_update(const float* gpart, const unsigned int* cpart, int nblk, int dim, float* w, double nu, double eta,
                 int64_t n, int mode, cudaStream_t s) {
    k_pred_update<<<(dim + 127) / 128, 128, 0, s>>>(gpart, cpart, nblk, dim, w, nu, eta, n, mode);
}
void pred_finish(const EvictState* st, float* rho, cudaStream_t s) { k_pred_finish<<<1, 1, 0, s>>>(st, rho); }
void pred_predict(const __nv_bfloat16* qbuf, const float* inv_q, const int32_t* qstatus, int64_t b, int dim,
                  const float* w, const float* rho, uint8_t* flags, float* margin, cudaStream_t s) {
    if (b > 0)
        k_predict<<<(unsigned)((b + 7) / 8), 256, dim * 4, s>>>(qbuf, inv_q, qstatus, b, dim, w, rho, flags, margin);
}

}  // namespace nv
