// rasp_kernels.cuh -- sm_100a kernels of the word-RASP batch engine.
//
// Hot path: Phi^K over a batch of independent machines <i, a, M, u, y>,
// bit-exact with raspvisor/hypervisor.py:72-164 (_advance/_worker).
//
// Execution model:
//   * one machine per lane; i, a, u0, y0 and the step bookkeeping live in
//     registers for a whole epoch of K steps;
//   * each warp owns a private shared-memory tile: M (n rows) and the input
//     tape u[1..ell] (ell+1 rows, one pad row), row-major with 32 lanes per
//     row, so lane L's cell k sits at tile[k*32 + L] -- bank = lane for every
//     data-dependent address, i.e. conflict-free random access;
//   * the output tape y is write-only during a run and goes straight to HBM;
//   * opcode dispatch is a predicated select over all candidates (no
//     divergent branch on the opcode); the fixed-point test uses the
//     equivalent short form of hv:115 for w >= 2;
//   * a warp leaves the epoch early when __any_sync says no lane is live;
//   * epochs are separated by stream compaction: survivors are appended to
//     the next live list (warp-aggregated atomics), halted machines retire.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace rasp {

constexpr unsigned kFull = 0xffffffffu;
constexpr int8_t kRunning = 0, kHalted = 1, kExhausted = 2;

struct Geo {
    uint64_t mask;    // 2^w - 1
    uint64_t fm;      // ceil(2^64 / n): Lemire fastmod magic (32-bit words, generic n)
    uint64_t jmask;   // mask & (n - 1)   (power-of-two n)
    uint32_t n;
    uint32_t nm1;     // n - 1            (power-of-two n)
    uint32_t ell;
    uint32_t s;
};

struct Side {
    void *iw, *ac, *M, *u, *y;
    int8_t *status;
    int64_t *steps;
    int64_t *tau_h;
};

struct EpochArgs {
    Geo g;
    Side in, out;
    const uint32_t *list_in;       // nullptr: identity list 0..count-1 (first epoch)
    uint32_t *list_out;
    const uint32_t *count_in_ptr;  // nullptr: use count_in
    uint32_t *count_out;
    uint32_t *tile_ctr;
    int64_t tau_max;
    uint32_t count_in;
    uint32_t K;                    // applying steps in this epoch
    uint32_t first;                // read the batch from `in`
    uint32_t fresh;                // status=0, steps=0, tau_h=-1 on input
    uint32_t inplace;              // in == out
    uint32_t tile_cells;           // n + ell + 1
};

// x mod n for a word x.
template <class CT, bool POW2>
__device__ __forceinline__ uint32_t modn(CT x, const Geo &g)
{
    if constexpr (POW2) {
        return static_cast<uint32_t>(x) & g.nm1;
    } else if constexpr (sizeof(CT) == 4) {
        const uint64_t low = g.fm * static_cast<uint64_t>(x);
        return static_cast<uint32_t>(__umul64hi(low, static_cast<uint64_t>(g.n)));
    } else {
        return static_cast<uint32_t>(x % static_cast<uint64_t>(g.n));
    }
}

// Per-lane row copy between a machine's HBM row (element type S, contiguous)
// and its shared-memory column (element type CT, stride 32).
template <class S, class CT>
__device__ __forceinline__ void load_row(const S *__restrict__ row, uint32_t ncells, CT *col)
{
    constexpr uint32_t PER = 16 / sizeof(S);
    uint32_t k = 0;
    if (((reinterpret_cast<uintptr_t>(row) & 15) == 0)) {
        const uint4 *v = reinterpret_cast<const uint4 *>(row);
        for (; k + PER <= ncells; k += PER) {
            const uint4 q = v[k / PER];
            S e[PER];
            memcpy(e, &q, 16);
#pragma unroll
            for (uint32_t p = 0; p < PER; ++p) col[(k + p) * 32] = static_cast<CT>(e[p]);
        }
    }
    for (; k < ncells; ++k) col[k * 32] = static_cast<CT>(row[k]);
}

template <class S, class CT>
__device__ __forceinline__ void store_row(S *__restrict__ row, uint32_t ncells, const CT *col)
{
    constexpr uint32_t PER = 16 / sizeof(S);
    uint32_t k = 0;
    if (((reinterpret_cast<uintptr_t>(row) & 15) == 0)) {
        uint4 *v = reinterpret_cast<uint4 *>(row);
        for (; k + PER <= ncells; k += PER) {
            S e[PER];
#pragma unroll
            for (uint32_t p = 0; p < PER; ++p) e[p] = static_cast<S>(col[(k + p) * 32]);
            uint4 q;
            memcpy(&q, e, 16);
            v[k / PER] = q;
        }
    }
    for (; k < ncells; ++k) row[k] = static_cast<S>(col[k * 32]);
}

template <class S>
__device__ __forceinline__ void copy_cells(S *__restrict__ dst, const S *__restrict__ src, uint64_t n)
{
    for (uint64_t k = 0; k < n; ++k) dst[k] = src[k];
}

// One machine held by one lane.  `sM`/`sU` point at the lane's column.
template <class S, class CT, bool POW2, bool GE2>
struct Lane {
    CT i, a;
    uint32_t u0, y0;
    uint32_t rem;      // remaining budget at epoch start (clamped)
    uint32_t tfin;     // step index of the verdict within this epoch
    bool active, halted, dirty;

    // Evaluate the step at local time t; classify or (if apply) commit it.
    // The five-candidate equality of hv:115 decides fixedness; for w >= 2
    // it reduces to: o not in 1..7, RD at capacity, or BNZ taken to itself.
    __device__ __forceinline__ void step(CT *sM, const CT *sU, S *yrow, const Geo &g,
                                         uint32_t t, bool apply)
    {
        const CT mask = static_cast<CT>(g.mask);
        const uint32_t ia = modn<CT, POW2>(i, g);
        uint32_t ib;
        if constexpr (POW2) ib = static_cast<uint32_t>((i + 1) & static_cast<CT>(g.jmask));
        else ib = modn<CT, POW2>((i + 1) & mask, g);
        const CT o = sM[ia * 32];
        const CT jw = sM[ib * 32];
        const uint32_t jn = modn<CT, POW2>(jw, g);
        const CT mj = sM[jn * 32];
        const CT ud = sU[u0 * 32];

        const bool is_rd = (o == 6);
        const bool rd_ok = is_rd & (u0 < g.ell);
        const bool pri_ok = (o == 7) & (y0 < g.s);
        const bool taken = (o == 5) & (a != 0);
        const bool is_sto = (o == 4);
        const CT i2 = (i + 2) & mask;
        CT na = a;
        na = (o == 3) ? static_cast<CT>((a * mj) & mask) : na;
        na = (o == 2) ? static_cast<CT>((a + mj) & mask) : na;
        na = (o == 1) ? jw : na;
        const CT nm = is_sto ? a : ud;
        const bool wr = is_sto | rd_ok;
        bool fixed;
        CT ni;
        if constexpr (GE2) {
            fixed = (static_cast<CT>(o - 1) > 6) | (is_rd & !rd_ok) | (taken & (jw == i));
            ni = taken ? jw : i2;
        } else {
            const bool adv = (static_cast<CT>(o - 1) < 4) | ((o == 5) & (a == 0)) | rd_ok | (o == 7);
            ni = taken ? jw : (adv ? i2 : i);
            const CT nmf = wr ? nm : mj;
            fixed = (ni == i) & (na == a) & (nmf == mj) & !rd_ok & !pri_ok;
        }
        if (active) {
            if (fixed) {
                halted = true;
                tfin = t;
                active = false;
            } else if (t == rem) {
                tfin = t;
                active = false;
            } else if (apply) {
                i = ni;
                a = na;
                if (wr) {
                    sM[jn * 32] = nm;
                    dirty = true;
                }
                u0 += rd_ok ? 1u : 0u;
                if (pri_ok) {
                    yrow[y0] = static_cast<S>(mj);
                    ++y0;
                }
            }
        }
    }
};

template <class S, class CT, bool POW2, bool GE2, bool SMEM>
__global__ void __launch_bounds__(128)
epoch_kernel(const EpochArgs A, CT *gtiles)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t wib = threadIdx.x >> 5;
    const Geo g = A.g;
    const uint32_t n = g.n;
    const uint64_t ucols = static_cast<uint64_t>(g.ell) + 1;
    const uint64_t ycols = static_cast<uint64_t>(g.s) + 1;

    CT *tile;
    if constexpr (SMEM) {
        tile = reinterpret_cast<CT *>(smem_raw) + static_cast<size_t>(wib) * A.tile_cells * 32;
    } else {
        tile = gtiles + (static_cast<size_t>(blockIdx.x) * (blockDim.x >> 5) + wib) *
                            static_cast<size_t>(A.tile_cells) * 32;
    }
    CT *sM = tile + lane;
    CT *sU = sM + static_cast<size_t>(n) * 32;

    const uint32_t count = A.count_in_ptr ? *A.count_in_ptr : A.count_in;
    const uint32_t ntiles = (count + 31) / 32;
    const Side &src = A.first ? A.in : A.out;
    const Side &dst = A.out;
    const bool copy_side = A.first && !A.inplace;

    for (;;) {
        uint32_t tix = 0;
        if (lane == 0) tix = atomicAdd(A.tile_ctr, 1u);
        tix = __shfl_sync(kFull, tix, 0);
        if (tix >= ntiles) break;
        const uint32_t j = tix * 32 + lane;
        const bool valid = j < count;
        const uint64_t id = valid ? (A.list_in ? A.list_in[j] : j) : 0;

        Lane<S, CT, POW2, GE2> L;
        L.i = 0; L.a = 0; L.u0 = 0; L.y0 = 0; L.tfin = 0;
        L.halted = false; L.dirty = false;
        bool running = valid;
        int64_t steps0 = 0;
        if (valid) {
            if (A.first) {
                if (!A.fresh) {
                    const int8_t st = A.in.status[id];
                    if (st != kRunning) running = false;
                    else steps0 = A.in.steps[id];
                    if (copy_side) {
                        dst.status[id] = st;
                        dst.steps[id] = A.in.steps[id];
                        dst.tau_h[id] = A.in.tau_h[id];
                    }
                }
            } else {
                steps0 = dst.steps[id];
            }
        }
        const S *srcM = static_cast<const S *>(src.M) + id * n;
        const S *srcU = static_cast<const S *>(src.u) + id * ucols;
        const S *srcY = static_cast<const S *>(src.y) + id * ycols;
        if (valid && copy_side && !running) {
            // untouched machine, out-of-place: carry it over verbatim
            static_cast<S *>(dst.iw)[id] = static_cast<const S *>(A.in.iw)[id];
            static_cast<S *>(dst.ac)[id] = static_cast<const S *>(A.in.ac)[id];
            copy_cells(static_cast<S *>(dst.M) + id * n, srcM, n);
            copy_cells(static_cast<S *>(dst.u) + id * ucols, srcU, ucols);
            copy_cells(static_cast<S *>(dst.y) + id * ycols, srcY, ycols);
        }
        if (running) {
            L.i = static_cast<CT>(static_cast<const S *>(src.iw)[id]);
            L.a = static_cast<CT>(static_cast<const S *>(src.ac)[id]);
            L.u0 = static_cast<uint32_t>(srcU[0]);
            L.y0 = static_cast<uint32_t>(srcY[0]);
            load_row<S, CT>(srcM, n, sM);
            load_row<S, CT>(srcU + 1, g.ell, sU);
            if (copy_side) {
                copy_cells(static_cast<S *>(dst.u) + id * ucols + 1, srcU + 1, g.ell);
                copy_cells(static_cast<S *>(dst.y) + id * ycols + 1, srcY + 1, g.s);
            }
        }
        const uint64_t rem64 = (steps0 >= A.tau_max) ? 0ull
                                                     : static_cast<uint64_t>(A.tau_max - steps0);
        L.rem = rem64 > 0xffffffffull ? 0xffffffffu : static_cast<uint32_t>(rem64);
        L.active = running;
        S *yrow = static_cast<S *>(dst.y) + id * ycols + 1;

        const uint32_t K = A.K;
        uint32_t t = 0;
        for (; t < K; ++t) {
            if (!__any_sync(kFull, L.active)) break;
            L.step(sM, sU, yrow, g, t, true);
        }
        if (t == K && __any_sync(kFull, L.active)) L.step(sM, sU, yrow, g, t, false);

        bool survivor = false;
        if (running) {
            static_cast<S *>(dst.iw)[id] = static_cast<S>(L.i);
            static_cast<S *>(dst.ac)[id] = static_cast<S>(L.a);
            static_cast<S *>(dst.u)[id * ucols] = static_cast<S>(L.u0);
            static_cast<S *>(dst.y)[id * ycols] = static_cast<S>(L.y0);
            if (L.dirty || copy_side) store_row<S, CT>(static_cast<S *>(dst.M) + id * n, n, sM);
            if (L.halted) {
                const int64_t tau = steps0 + L.tfin;
                dst.status[id] = kHalted;
                dst.steps[id] = tau;
                dst.tau_h[id] = tau;
            } else if (!L.active) {
                dst.status[id] = kExhausted;
                dst.steps[id] = steps0 + L.tfin;
                if (A.fresh && copy_side) dst.tau_h[id] = -1;
            } else {
                survivor = true;
                dst.steps[id] = steps0 + K;
                if (A.fresh && copy_side) {
                    dst.status[id] = kRunning;
                    dst.tau_h[id] = -1;
                }
            }
        }
        const unsigned sv = __ballot_sync(kFull, survivor);
        if (sv) {
            uint32_t base = 0;
            if (lane == 0) base = atomicAdd(A.count_out, static_cast<uint32_t>(__popc(sv)));
            base = __shfl_sync(kFull, base, 0);
            if (survivor) A.list_out[base + __popc(sv & ((1u << lane) - 1u))] = static_cast<uint32_t>(id);
        }
    }
}

// 102-bucket halting histogram (hypervisor.py:326-352).
__global__ void histogram_kernel(const int8_t *__restrict__ status, const int64_t *__restrict__ tau_h,
                                 uint64_t d, unsigned long long *__restrict__ out)
{
    __shared__ unsigned int h[102];
    for (int k = threadIdx.x; k < 102; k += blockDim.x) h[k] = 0;
    __syncthreads();
    for (uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; j < d;
         j += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const int8_t st = status[j];
        if (st == kHalted) {
            const int64_t t = tau_h[j];
            atomicAdd(&h[t < 100 ? static_cast<int>(t) : 100], 1u);
        } else if (st == kExhausted) {
            atomicAdd(&h[101], 1u);
        }
    }
    __syncthreads();
    for (int k = threadIdx.x; k < 102; k += blockDim.x)
        if (h[k]) atomicAdd(&out[k], static_cast<unsigned long long>(h[k]));
}

// Word-range and cursor-range validation (m:324-327, hv:285-290).
template <class S>
__global__ void validate_kernel(Side b, uint64_t d, uint32_t n, uint64_t ucols, uint64_t ycols,
                                uint64_t mask, uint64_t ell, uint64_t s,
                                unsigned long long *__restrict__ out)
{
    unsigned long long c[7] = {0, 0, 0, 0, 0, 0, 0};
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    const uint64_t t0 = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    const S *iw = static_cast<const S *>(b.iw), *ac = static_cast<const S *>(b.ac);
    const S *M = static_cast<const S *>(b.M), *u = static_cast<const S *>(b.u),
            *y = static_cast<const S *>(b.y);
    for (uint64_t j = t0; j < d; j += stride) {
        c[0] += static_cast<uint64_t>(iw[j]) > mask;
        c[1] += static_cast<uint64_t>(ac[j]) > mask;
        c[5] += static_cast<uint64_t>(u[j * ucols]) > ell;
        c[6] += static_cast<uint64_t>(y[j * ycols]) > s;
    }
    for (uint64_t j = t0; j < d * n; j += stride) c[2] += static_cast<uint64_t>(M[j]) > mask;
    for (uint64_t j = t0; j < d * ucols; j += stride) c[3] += static_cast<uint64_t>(u[j]) > mask;
    for (uint64_t j = t0; j < d * ycols; j += stride) c[4] += static_cast<uint64_t>(y[j]) > mask;
#pragma unroll
    for (int k = 0; k < 7; ++k) {
        unsigned long long v = c[k];
        for (int off = 16; off; off >>= 1) v += __shfl_down_sync(kFull, v, off);
        if ((threadIdx.x & 31) == 0 && v) atomicAdd(&out[k], v);
    }
}

}  // namespace rasp
