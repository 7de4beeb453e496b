// rasp_kernels.cuh -- sm_100a kernels of the word-RASP batch engine.
//
// Hot path: Phi^K over a batch of independent machines <i, a, M, u, y>,
// bit-exact with raspvisor/hypervisor.py:72-164 (_advance/_worker).
//
// Execution model:
//   * one machine per lane; i, a and the cursor addresses live in registers
//     for a whole epoch of K steps;
//   * each warp owns a private shared-memory tile with one row per machine
//     cell and 32 lanes per row: M (n rows), the input tape u[1..ell] (ell+1
//     rows, one pad row) and s output rows.  Cells are SC = u16/u32/u64
//     (the smallest of those holding w bits), lane-interleaved at SC
//     granularity: lane L's cell k is at row k, column L.  For SC >= 4 bytes
//     every data-dependent access is bank-conflict-free; u16 cells pack two
//     lanes per bank word (at most 2-way conflicts) to double the machines
//     resident per SM;
//   * the output tape y is write-only during a run: appended cells collect in
//     tile rows and are flushed to HBM at the end of the epoch;
//   * opcode dispatch is a predicated select over all candidates (no branch
//     on the opcode); the fixed-point test uses the equivalent short form of
//     hv:115 for w >= 2 and the full five-candidate equality
//     for w = 1;
//   * a warp leaves the epoch early when __any_sync says no lane is live;
//   * epochs are separated by stream compaction: survivors are appended to
//     the next live list (warp-aggregated atomics), finished machines retire.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace rasp {

constexpr unsigned kFull = 0xffffffffu;
constexpr int8_t kRunning = 0, kHalted = 1, kExhausted = 2;

// Word arithmetic regime: w == 1 (generic fixedness test), 2 <= w < bits(CT)
// (masked), w == bits(CT) (native wrap-around, no masks), and CELL: w equals
// the tile cell width but not bits(CT) (w = 16 on u16 cells) -- the
// accumulator then carries garbage above bit w between steps (every store
// truncates to the cell, every test masks), which saves the masks on ADD/MUL.
enum class Arith { W1, NARROW, FULL, CELL };

struct Geo {
    uint64_t mask;    // 2^w - 1
    uint64_t fm;      // ceil(2^64 / n) (unused by the kernels; kept for the layout)
    uint32_t n;
    uint32_t nm1;     // n - 1               (power-of-two n)
    uint32_t jm;      // (2^w - 1) & (n - 1) (power-of-two n)
    uint32_t ell;
    uint32_t s;
    uint32_t m32;     // floor(2^32 / n): quotient estimate for x mod n of 32-bit words
};

struct Side {
    void *iw, *ac, *M, *u, *y;
    int8_t *status;
    int64_t *steps;
    int64_t *tau_h;
};

constexpr int kMaxEpochs = 1024;

// --- checked build (-DRASP_CHECKED=1): the stand-in for compute-sanitizer --------
//
// Every shared-memory access of the kernels is checked against the block's
// dynamic shared window, every cell access of a step against the lane's own
// column of its warp's tile (the lane-column layout's ownership rule: a lane
// that touched another lane's cells would be a cross-thread hazard), and every
// per-machine global row index against the batch.  The first violation is
// recorded in g_check (code, two operands, thread); rasp_run of a checked
// build synchronises and fails with RASP_ECHECK when one was seen.
#ifndef RASP_CHECKED
#define RASP_CHECKED 0
#endif
enum CheckCode : unsigned long long {
    kChkSmemRange = 1,   // shared access outside the dynamic window
    kChkColumn = 2,      // step cell access outside the lane's own column
    kChkRow = 3,         // machine index beyond the batch
    kChkYTape = 4,       // direct-to-HBM output cursor beyond the tape
    kChkList = 5,        // compaction list slot beyond the batch
};
#if RASP_CHECKED
static __device__ unsigned long long g_check[4];   // one per module (translation unit)
extern __shared__ __align__(16) unsigned char rasp_dyn_smem[];
static __device__ __noinline__ void check_fail(unsigned long long code, unsigned long long a, unsigned long long b)
{
    if (atomicCAS(&g_check[0], 0ull, code) == 0ull) {
        g_check[1] = a;
        g_check[2] = b;
        g_check[3] = (static_cast<unsigned long long>(blockIdx.x) << 32) | threadIdx.x;
    }
}
__device__ __forceinline__ void check_smem(uint32_t a, uint32_t bytes)
{
    uint32_t dsz;
    asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dsz));
    const uint32_t lo = static_cast<uint32_t>(__cvta_generic_to_shared(rasp_dyn_smem));
    if (a < lo || a + bytes > lo + dsz) check_fail(kChkSmemRange, a, lo + dsz);
}
#define RASP_CHECK(cond, code, a, b) \
    do {                             \
        if (!(cond)) ::rasp::check_fail((code), (a), (b)); \
    } while (0)
#else
__device__ __forceinline__ void check_smem(uint32_t, uint32_t) {}
#define RASP_CHECK(cond, code, a, b) \
    do {                             \
    } while (0)
#endif

#ifndef RASP_UNROLL
#define RASP_UNROLL 8
#endif
#ifndef RASP_UNROLL_BIG
#define RASP_UNROLL_BIG 16
#endif
// Launch shape of the shared-memory epoch kernels: at most RASP_BLOCK_WARPS
// warps per block, RASP_MIN_BLOCKS blocks resident per SM (caps registers).
#ifndef RASP_BLOCK_WARPS
#define RASP_BLOCK_WARPS 4
#endif
// 5 blocks of 4 warps: 20 warps per SM with up to 102 registers.  Measured
// (C2 / C3): 10 blocks (40 warps, 48 registers) 0.549 / 7.46 ms, 8 -> 0.522 /
// 7.31, 6 -> 0.515 / 7.31, 5 -> 0.506 / 7.30, 4 -> 0.534 / 7.64; 10 blocks of
// 2 warps = 5 of 4.
#ifndef RASP_MIN_BLOCKS
#define RASP_MIN_BLOCKS 5
#endif
// Matrix-op row moves in flight per lane (16 B each) when loading a tile.
#ifndef RASP_MX_BATCH
#define RASP_MX_BATCH 4
#endif

// Device-side epoch schedule (workspace).  Epoch e reads its length K[e] and
// start offset covered[e]; the last block of epoch e writes K[e+1] from the
// survival ratio it observed, so the host can enqueue epochs without
// knowing the halting-time distribution.
struct Sched {
    int64_t covered[kMaxEpochs];     // steps every fresh survivor has taken before epoch e
    uint32_t K[kMaxEpochs];          // applying steps in epoch e (0: nothing left)
    uint32_t count[kMaxEpochs];      // survivors after epoch e
    uint32_t tile_ctr[kMaxEpochs];
    uint32_t blocks_done[kMaxEpochs];
};

struct EpochArgs {
    Geo g;
    Side in, out;
    Sched *sched;
    const uint32_t *list_in;       // nullptr: identity list 0..count-1 (first epoch)
    uint32_t *list_out;
    int64_t tau_max;
    uint32_t e;                    // epoch index
    uint32_t count_in;             // first epoch: batch size
    uint32_t K0;                   // first epoch length
    uint32_t kmax;                 // longest epoch
    uint32_t first;                // read the batch from `in`
    uint32_t fresh;                // status=0, steps=0, tau_h=-1 on input
    uint32_t inplace;              // in == out
    uint32_t tile_rows;            // n + ell + 1 (+ s output rows unless BIG)
    uint32_t stable_q8;            // survival ratio (x256) at which the rest runs as one epoch
    uint32_t pf_dist;              // L2 prefetch distance in rounds of resident warps (0: off)
    uint32_t jump;                 // longest "rest of the budget" epoch, in units of the previous one
    uint32_t growth;               // next epoch length while machines still halt, x the last one
    uint32_t stable_hi_q8;         // survival ratio (x256) at which the rest runs as one epoch regardless
    unsigned long long *hist;      // int64[102] halting histogram accumulated by the run, or nullptr
    uint32_t refill_min;           // refill_kernel: free lanes that trigger a refill
};

template <class CT, Arith AR>
__device__ __forceinline__ CT wrap(CT x, CT mask)
{
    if constexpr (AR == Arith::FULL) return x;
    else return x & mask;
}

// x mod n for a word x.
template <class CT, bool POW2>
__device__ __forceinline__ uint32_t modn(CT x, const Geo &g)
{
    if constexpr (POW2) {
        return static_cast<uint32_t>(x) & g.nm1;
    } else if constexpr (sizeof(CT) == 4) {
        // q = floor(x * floor(2^32/n) / 2^32) is floor(x/n) or one less, so
        // r = x - q*n lies in [0, 2n): one conditional subtract (as an unsigned
        // min) -- 4 instructions against 8 for a 64-bit Lemire reduction
        // (n < 2^31, enforced by check_params)
        const uint32_t xv = static_cast<uint32_t>(x);
        const uint32_t r = xv - __umulhi(xv, g.m32) * g.n;
        return min(r, r - g.n);
    } else {
        return static_cast<uint32_t>(x % static_cast<uint64_t>(g.n));
    }
}

// --- per-lane row movement between HBM (element S, contiguous) and the
//     lane's tile column (element SC, stride 32 cells) ------------------------

template <class S, class SC>
__device__ __forceinline__ void put16(SC *col, uint32_t k, const uint4 q)
{
    const uint32_t wv[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        if constexpr (sizeof(S) == 1) {
#pragma unroll
            for (int b = 0; b < 4; ++b) col[(k + 4 * e + b) * 32] = static_cast<SC>((wv[e] >> (8 * b)) & 0xffu);
        } else if constexpr (sizeof(S) == 2) {
            col[(k + 2 * e) * 32] = static_cast<SC>(wv[e] & 0xffffu);
            col[(k + 2 * e + 1) * 32] = static_cast<SC>(wv[e] >> 16);
        } else if constexpr (sizeof(S) == 4) {
            col[(k + e) * 32] = static_cast<SC>(wv[e]);
        } else {
            if (e & 1) continue;
            col[(k + e / 2) * 32] = static_cast<SC>(static_cast<uint64_t>(wv[e]) |
                                                    (static_cast<uint64_t>(wv[e + 1]) << 32));
        }
    }
}

template <class S, class SC>
__device__ __forceinline__ uint4 get16(const SC *col, uint32_t k)
{
    uint32_t wv[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        if constexpr (sizeof(S) == 1) {
            uint32_t x = 0;
#pragma unroll
            for (int b = 0; b < 4; ++b) x |= (static_cast<uint32_t>(col[(k + 4 * e + b) * 32]) & 0xffu) << (8 * b);
            wv[e] = x;
        } else if constexpr (sizeof(S) == 2) {
            wv[e] = (static_cast<uint32_t>(col[(k + 2 * e) * 32]) & 0xffffu) |
                    (static_cast<uint32_t>(col[(k + 2 * e + 1) * 32]) << 16);
        } else if constexpr (sizeof(S) == 4) {
            wv[e] = static_cast<uint32_t>(col[(k + e) * 32]);
        } else {
            const uint64_t v = static_cast<uint64_t>(col[(k + e / 2) * 32]);
            wv[e] = (e & 1) ? static_cast<uint32_t>(v >> 32) : static_cast<uint32_t>(v);
        }
    }
    return make_uint4(wv[0], wv[1], wv[2], wv[3]);
}

// Loads are issued in batches (8 x 16 B, or 8 scalars) before any of the
// dependent shared-memory stores, so a row costs ~one DRAM latency instead
// of one per chunk.
// checked builds: the extent [col, col + ncells rows) lies in the dynamic window
template <class SC>
__device__ __forceinline__ void check_col_extent(const SC *col, uint32_t ncells)
{
#if RASP_CHECKED
    if (ncells == 0 || !__isShared(col)) return;
    const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(col));
    check_smem(a, sizeof(SC));
    check_smem(a + (ncells - 1) * 32 * static_cast<uint32_t>(sizeof(SC)), sizeof(SC));
#endif
}

// Rows that do not start on a 16-byte boundary (machine m's row starts at
// m * n words: with n * sizeof(S) not a multiple of 16, every other row is
// misaligned -- the paper rows' n = 250) take a scalar head up to the
// boundary, loaded together with the first vector batch and stored after the
// vector part, so a row still costs ceil(cells / (16 B x B)) memory round
// trips instead of one per B scalars.
template <class S, class SC, uint32_t B = 8>
__device__ __forceinline__ void load_row(const S *__restrict__ row, uint32_t ncells, SC *col)
{
    check_col_extent(col, ncells);
    constexpr uint32_t PER = 16 / sizeof(S);
    uint32_t k = 0;
    const uintptr_t ra = reinterpret_cast<uintptr_t>(row);
    if (ra % sizeof(S) == 0) {
        const uint32_t head = min(static_cast<uint32_t>(((16 - (ra & 15)) & 15) / sizeof(S)), ncells);
        S h[PER > 1 ? PER - 1 : 1];
#pragma unroll
        for (uint32_t j = 0; j + 1 < PER; ++j)
            if (j < head) h[j] = row[j];
        k = head;
        const uint4 *v = reinterpret_cast<const uint4 *>(row + head);
        for (; k + B * PER <= ncells; k += B * PER) {
            uint4 q[B];
#pragma unroll
            for (uint32_t j = 0; j < B; ++j) q[j] = v[(k - head) / PER + j];
#pragma unroll
            for (uint32_t j = 0; j < B; ++j) put16<S, SC>(col, k + j * PER, q[j]);
        }
        for (; k + PER <= ncells; k += PER) put16<S, SC>(col, k, v[(k - head) / PER]);
#pragma unroll
        for (uint32_t j = 0; j + 1 < PER; ++j)
            if (j < head) col[j * 32] = static_cast<SC>(h[j]);
    }
    for (; k + B <= ncells; k += B) {
        S e[B];
#pragma unroll
        for (uint32_t j = 0; j < B; ++j) e[j] = row[k + j];
#pragma unroll
        for (uint32_t j = 0; j < B; ++j) col[(k + j) * 32] = static_cast<SC>(e[j]);
    }
    for (; k < ncells; ++k) col[k * 32] = static_cast<SC>(row[k]);
}

// A machine's M row and input tape u[1..ell] in two memory round trips when
// the tape is short (ell <= 32): the tape's scalar loads (and a misaligned
// row's scalar head) ride with the first batch of M's 16-byte loads.
// Otherwise load_row twice.
template <class S, class SC, uint32_t B = 32>
__device__ __forceinline__ void load_rows_mu(const S *__restrict__ rm, uint32_t n, SC *colm,
                                             const S *__restrict__ ru, uint32_t ell, SC *colu)
{
    constexpr uint32_t PER = 16 / sizeof(S);
    const uintptr_t ra = reinterpret_cast<uintptr_t>(rm);
    const uint32_t head = static_cast<uint32_t>(((16 - (ra & 15)) & 15) / sizeof(S));
    if (ell > 32 || ra % sizeof(S) != 0 || n < head + B * PER) {
        load_row<S, SC, B>(rm, n, colm);
        load_row<S, SC, B>(ru, ell, colu);
        return;
    }
    check_col_extent(colm, n);
    check_col_extent(colu, ell);
    const uint4 *v = reinterpret_cast<const uint4 *>(rm + head);
    {
        S h[PER > 1 ? PER - 1 : 1];
        uint4 qm[B];
        S qu[32];
#pragma unroll
        for (uint32_t j = 0; j + 1 < PER; ++j)
            if (j < head) h[j] = rm[j];
#pragma unroll
        for (uint32_t j = 0; j < B; ++j) qm[j] = v[j];
#pragma unroll
        for (uint32_t j = 0; j < 32; ++j)
            if (j < ell) qu[j] = ru[j];
#pragma unroll
        for (uint32_t j = 0; j < B; ++j) put16<S, SC>(colm, head + j * PER, qm[j]);
#pragma unroll
        for (uint32_t j = 0; j < 32; ++j)
            if (j < ell) colu[j * 32] = static_cast<SC>(qu[j]);
#pragma unroll
        for (uint32_t j = 0; j + 1 < PER; ++j)
            if (j < head) colm[j * 32] = static_cast<SC>(h[j]);
    }
    load_row<S, SC, B>(rm + head + B * PER, n - head - B * PER, colm + (head + B * PER) * 32);
}

// The same for 16-byte aligned M rows only (the refill kernel: the general
// form's registers measured +1.2% on C5, whose rows are aligned).
template <class S, class SC, uint32_t B = 32>
__device__ __forceinline__ void load_rows_mu_aligned(const S *__restrict__ rm, uint32_t n, SC *colm,
                                             const S *__restrict__ ru, uint32_t ell, SC *colu)
{
    constexpr uint32_t PER = 16 / sizeof(S);
    if (ell > 32 || (reinterpret_cast<uintptr_t>(rm) & 15) != 0 || n < B * PER) {
        load_row<S, SC, B>(rm, n, colm);
        load_row<S, SC, B>(ru, ell, colu);
        return;
    }
    check_col_extent(colm, n);
    check_col_extent(colu, ell);
    const uint4 *v = reinterpret_cast<const uint4 *>(rm);
    {
        uint4 qm[B];
        S qu[32];
#pragma unroll
        for (uint32_t j = 0; j < B; ++j) qm[j] = v[j];
#pragma unroll
        for (uint32_t j = 0; j < 32; ++j)
            if (j < ell) qu[j] = ru[j];
#pragma unroll
        for (uint32_t j = 0; j < B; ++j) put16<S, SC>(colm, j * PER, qm[j]);
#pragma unroll
        for (uint32_t j = 0; j < 32; ++j)
            if (j < ell) colu[j * 32] = static_cast<SC>(qu[j]);
    }
    load_row<S, SC, B>(rm + B * PER, n - B * PER, colm + B * PER * 32);
}

// Shared loads in batches of B x 16 B before their global stores (one
// shared-load latency per batch instead of one per 16 bytes).  Write-backs of
// big tiles use B = 16: refill kernel C5 -1.4%, epoch kernel paper6 -0.8%,
// paper +0.1% (B = 8 had measured +0.8% on the epoch kernel before rows
// with a misaligned head were vectorised).
template <class S, class SC, uint32_t B = 1>
__device__ __forceinline__ void store_row(S *__restrict__ row, uint32_t ncells, const SC *col)
{
    check_col_extent(col, ncells);
    constexpr uint32_t PER = 16 / sizeof(S);
    uint32_t k = 0;
    const uintptr_t ra = reinterpret_cast<uintptr_t>(row);
    if (ra % sizeof(S) == 0) {   // scalar head up to the 16-byte boundary, then vectors
        const uint32_t head = min(static_cast<uint32_t>(((16 - (ra & 15)) & 15) / sizeof(S)), ncells);
        for (; k < head; ++k) row[k] = static_cast<S>(col[k * 32]);
        uint4 *v = reinterpret_cast<uint4 *>(row + head);
        for (; k + B * PER <= ncells; k += B * PER) {
            uint4 q[B];
#pragma unroll
            for (uint32_t j = 0; j < B; ++j) q[j] = get16<S, SC>(col, k + j * PER);
#pragma unroll
            for (uint32_t j = 0; j < B; ++j) v[(k - head) / PER + j] = q[j];
        }
        for (; k + PER <= ncells; k += PER) v[(k - head) / PER] = get16<S, SC>(col, k);
    }
    for (; k < ncells; ++k) row[k] = static_cast<S>(col[k * 32]);
}

template <class S>
__device__ __forceinline__ void copy_cells(S *__restrict__ dst, const S *__restrict__ src, uint64_t n)
{
    for (uint64_t k = 0; k < n; ++k) dst[k] = src[k];
}


// --- warp-wide row movement with stmatrix/ldmatrix (shared-memory tiles) --------
//
// One `stmatrix.x4` writes 16 bytes of every lane's row (8 u16 or 4 u32
// cells) into the 32 lane columns, replacing 8 (4) scalar shared stores per
// lane; `ldmatrix.x4` is the inverse for the write-back.
//   u32 cells: plain m8n8 -- matrix r row rho is tile row (k0 + r), lanes
//     4rho..4rho+3, so lane L keeps its natural column L.
//   u16 cells: the .trans form -- matrix r row rho is tile row
//     (k0 + 2r + (rho & 1)) holding lanes b, b+4, ..., b+28 (b = rho >> 1), so
//     lane L's column is position (L & 3) * 8 + (L >> 2) (mx_col).
// Every lane of the warp must execute these (.sync.aligned).
template <class SC>
constexpr bool kMx = sizeof(SC) == 2 || sizeof(SC) == 4;

template <class SC>
__device__ __forceinline__ uint32_t mx_col(uint32_t lane)
{
    if constexpr (sizeof(SC) == 2) return ((lane & 3u) << 3) | (lane >> 2);
    else return lane;
}

template <class SC>
__device__ __forceinline__ uint32_t mx_addr(uint32_t tile0, uint32_t row0, uint32_t lane)
{
    if constexpr (sizeof(SC) == 2)
        return tile0 + (row0 + 2u * (lane >> 3) + (lane & 1u)) * 64u + ((lane >> 1) & 3u) * 16u;
    else
        return tile0 + (row0 + (lane >> 3)) * 128u + (lane & 7u) * 16u;
}

template <class SC>
__device__ __forceinline__ void stsm(uint32_t addr, const uint4 v)
{
    check_smem(addr, 16);
    if constexpr (sizeof(SC) == 2)
        asm volatile("stmatrix.sync.aligned.m8n8.x4.trans.shared.b16 [%0], {%1, %2, %3, %4};"
                     ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
    else
        asm volatile("stmatrix.sync.aligned.m8n8.x4.shared.b16 [%0], {%1, %2, %3, %4};"
                     ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

template <class SC>
__device__ __forceinline__ uint4 ldsm(uint32_t addr)
{
    check_smem(addr, 16);
    uint4 v;
    if constexpr (sizeof(SC) == 2)
        asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr) : "memory");
    else
        asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr) : "memory");
    return v;
}

// Bytes of HBM row one matrix op covers, and whether rows of `ncells` words
// starting at `base` can be moved with vector loads of that size.
template <class S, class SC>
constexpr uint32_t kMxBytes = (16 / sizeof(SC)) * sizeof(S);

template <class S, class SC>
__device__ __forceinline__ bool mx_vec_ok(const void *base, uint64_t ncells)
{
    constexpr uint32_t GB = kMxBytes<S, SC>;
    if constexpr (!(sizeof(S) == sizeof(SC) || (sizeof(S) == 1 && sizeof(SC) == 2))) return false;
    return (reinterpret_cast<uintptr_t>(base) % GB) == 0 && (ncells * sizeof(S)) % GB == 0;
}

// One lane's 16 bytes of cells [k, k + 16/sizeof(SC)) as SC words.
template <class S, class SC>
__device__ __forceinline__ uint4 mx_gather(const S *__restrict__ row, uint32_t k, bool vec)
{
    constexpr uint32_t C = 16 / sizeof(SC);
    if constexpr (sizeof(S) == sizeof(SC)) {
        if (vec) return *reinterpret_cast<const uint4 *>(row + k);
    } else if constexpr (sizeof(S) == 1 && sizeof(SC) == 2) {
        if (vec) {
            const uint2 w = *reinterpret_cast<const uint2 *>(row + k);
            return make_uint4(__byte_perm(w.x, 0, 0x4140), __byte_perm(w.x, 0, 0x4342),
                              __byte_perm(w.y, 0, 0x4140), __byte_perm(w.y, 0, 0x4342));
        }
    }
    uint32_t r[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        if constexpr (C == 8)
            r[q] = (static_cast<uint32_t>(row[k + 2 * q]) & 0xffffu) | (static_cast<uint32_t>(row[k + 2 * q + 1]) << 16);
        else
            r[q] = static_cast<uint32_t>(row[k + q]);
    }
    return make_uint4(r[0], r[1], r[2], r[3]);
}

template <class S, class SC>
__device__ __forceinline__ void mx_scatter(S *__restrict__ row, uint32_t k, const uint4 v, bool vec)
{
    constexpr uint32_t C = 16 / sizeof(SC);
    if constexpr (sizeof(S) == sizeof(SC)) {
        if (vec) {
            *reinterpret_cast<uint4 *>(row + k) = v;
            return;
        }
    } else if constexpr (sizeof(S) == 1 && sizeof(SC) == 2) {
        if (vec) {
            *reinterpret_cast<uint2 *>(row + k) = make_uint2(__byte_perm(v.x, v.y, 0x6420), __byte_perm(v.z, v.w, 0x6420));
            return;
        }
    }
    const uint32_t r[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        if constexpr (C == 8) {
            row[k + 2 * q] = static_cast<S>(r[q] & 0xffffu);
            row[k + 2 * q + 1] = static_cast<S>(r[q] >> 16);
        } else {
            row[k + q] = static_cast<S>(r[q]);
        }
    }
}

// Warp-wide: cells [0, ncells) of each valid lane's HBM row -> tile rows
// row0.. of its column (`col` = the lane's column at row0, for the tail).
template <class S, class SC, uint32_t B>
__device__ __forceinline__ void mx_load(const S *__restrict__ row, bool valid, bool vec, uint32_t ncells,
                                        uint32_t tile0, uint32_t row0, uint32_t lane, SC *col)
{
    constexpr uint32_t C = 16 / sizeof(SC);
    const uint32_t full = ncells / C * C;
    uint32_t k = 0;
    for (; k + B * C <= full; k += B * C) {
        uint4 v[B];
#pragma unroll
        for (uint32_t j = 0; j < B; ++j) v[j] = valid ? mx_gather<S, SC>(row, k + j * C, vec) : make_uint4(0, 0, 0, 0);
#pragma unroll
        for (uint32_t j = 0; j < B; ++j) stsm<SC>(mx_addr<SC>(tile0, row0 + k + j * C, lane), v[j]);
    }
    for (; k < full; k += C) {
        const uint4 v = valid ? mx_gather<S, SC>(row, k, vec) : make_uint4(0, 0, 0, 0);
        stsm<SC>(mx_addr<SC>(tile0, row0 + k, lane), v);
    }
    if (valid)
        for (; k < ncells; ++k) col[k * 32] = static_cast<SC>(row[k]);
}

template <class S, class SC, uint32_t B>
__device__ __forceinline__ void mx_store(S *__restrict__ row, bool valid, bool vec, uint32_t ncells,
                                         uint32_t tile0, uint32_t row0, uint32_t lane, const SC *col)
{
    constexpr uint32_t C = 16 / sizeof(SC);
    const uint32_t full = ncells / C * C;
    uint32_t k = 0;
    for (; k + B * C <= full; k += B * C) {
        uint4 v[B];
#pragma unroll
        for (uint32_t j = 0; j < B; ++j) v[j] = ldsm<SC>(mx_addr<SC>(tile0, row0 + k + j * C, lane));
        if (valid) {
#pragma unroll
            for (uint32_t j = 0; j < B; ++j) mx_scatter<S, SC>(row, k + j * C, v[j], vec);
        }
    }
    for (; k < full; k += C) {
        const uint4 v = ldsm<SC>(mx_addr<SC>(tile0, row0 + k, lane));
        if (valid) mx_scatter<S, SC>(row, k, v, vec);
    }
    if (valid)
        for (; k < ncells; ++k) row[k] = static_cast<S>(col[k * 32]);
}


// L2 prefetch of [p, p + bytes): one per-lane prefetch per 128-byte line.
// (The bulk form, cp.async.bulk.prefetch, takes a warp-uniform address: with
// every lane prefetching its own machine's row ptxas runs it as a 32-step
// waterfall loop per call -- ~8% of the first epoch's instructions on C2.)
__device__ __forceinline__ void prefetch_l2(const void *p, uint32_t bytes)
{
    const uintptr_t end = reinterpret_cast<uintptr_t>(p) + bytes;
    for (uintptr_t a = reinterpret_cast<uintptr_t>(p) & ~uintptr_t(127); a < end; a += 128)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
}


// Warp-cooperative copy of a contiguous byte range (16-byte vectors when both
// ends allow it).
__device__ __forceinline__ void warp_copy(void *dst, const void *src, uint64_t bytes, uint32_t lane)
{
    const uintptr_t a = reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src);
    uint64_t k0 = 0;
    if ((a & 15) == 0) {
        const uint64_t n16 = bytes >> 4;
        for (uint64_t k = lane; k < n16; k += 32)
            reinterpret_cast<uint4 *>(dst)[k] = reinterpret_cast<const uint4 *>(src)[k];
        k0 = n16 << 4;
    }
    for (uint64_t k = k0 + lane; k < bytes; k += 32)
        static_cast<unsigned char *>(dst)[k] = static_cast<const unsigned char *>(src)[k];
}

// --- one machine per lane -------------------------------------------------------
//
// Tile layout per warp: row r holds cell r of all 32 lanes (SC each).
//   rows [0, n)            M
//   rows [n, n+ell+1)      u[1..ell] + one pad row (u[u0+1] is read every step)
//   rows [n+ell+1, +s)     y[1..s] appended during this epoch (flushed at its end)
// Cursors are kept as addresses (ua = &u[u0+1], ya = &y[y0+1] of this lane) so
// the hot loop does no address arithmetic for them.

template <class CT>
struct LaneState {
    CT i, a;          // i may carry bits above w when RAWI (reduced at every use)
    uint32_t ua, ya;  // addresses of u[u0+1] and y[y0+1]
    uint32_t rem;     // remaining budget at epoch start (clamped)
    uint32_t tlast;   // last local time at which the lane was still live
    bool active;
};

// Step constants (1, 2, bytes per tile row).  Kept as a struct so callers
// can pass them; they are compile-time values (runtime copies were
// rematerialised by ptxas from the constant bank inside the loop).
struct Opq {
    uint32_t one, two, row;
};

// Cell access.  SMEM kernels address the warp tile with 32-bit shared-window
// addresses (one LDS/STS with a register address per access); the huge-n
// fallback uses byte offsets from the warp's HBM tile `base`.
template <class SC, class CT, bool SMEM>
__device__ __forceinline__ CT ld_cell(char *base, uint32_t a)
{
    if constexpr (SMEM) {
        check_smem(a, sizeof(SC));
        if constexpr (sizeof(SC) == 2) {
            uint32_t v;   // zero-extending 16-bit load straight into a 32-bit register
            asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v) : "r"(a));
            return static_cast<CT>(v);
        } else if constexpr (sizeof(SC) == 4) {
            uint32_t v;
            asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
            return static_cast<CT>(v);
        } else {
            unsigned long long v;
            asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(a));
            return static_cast<CT>(v);
        }
    } else {
        return static_cast<CT>(*reinterpret_cast<const volatile SC *>(base + a));
    }
}

template <class SC, class CT, bool SMEM>
__device__ __forceinline__ void st_cell(char *base, uint32_t a, CT v)
{
    if constexpr (SMEM) {
        check_smem(a, sizeof(SC));
        if constexpr (sizeof(SC) == 2) {
            asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "h"(static_cast<unsigned short>(v)) : "memory");
        } else if constexpr (sizeof(SC) == 4) {
            asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(static_cast<uint32_t>(v)) : "memory");
        } else {
            asm volatile("st.shared.u64 [%0], %1;" ::"r"(a), "l"(static_cast<unsigned long long>(v)) : "memory");
        }
    } else {
        *reinterpret_cast<volatile SC *>(base + a) = static_cast<SC>(v);
    }
}

// RAWI: power-of-two n and w >= 2 -- i is advanced without masking; every
// use reduces it ((i mod 2^w) mod n == i & (mask & (n-1)) for n a power of
// two; equality with a word compares the low w bits).
template <bool POW2, Arith AR>
constexpr bool kRawI = POW2 && AR != Arith::W1;

// One fetch/decode of the lane's current instruction: everything the step
// and the fixedness test need.
template <class CT>
struct Fetch {
    CT o, jw, mj, ud;
    uint32_t jo;   // address of M[jw mod n]
};

// Lane-column ownership (checked builds): cell address `a` must be in the
// column of the lane whose row-0 cell is at `lm`, within the tile's rows (M,
// the input tape and its pad row, and the output rows when staged).
template <class SC>
__device__ __forceinline__ void check_col(uint32_t a, uint32_t lm, const Geo &g, bool yrows)
{
#if RASP_CHECKED
    constexpr uint32_t ROW = 32 * sizeof(SC);
    const uint32_t rows = g.n + g.ell + 1 + (yrows ? g.s : 0);
    if (a < lm || (a - lm) % ROW != 0 || (a - lm) / ROW >= rows) check_fail(kChkColumn, a, lm);
#endif
}

// LAZY_UD: skip the input-tape read (the ungated steps read u[u0+1] only
// when the instruction is an RD that will store it)
template <class SC, class CT, bool POW2, Arith AR, bool SMEM, bool LAZY_UD = false, bool LAZY_MJ = false>
__device__ __forceinline__ Fetch<CT> fetch(const LaneState<CT> &L, char *base, uint32_t lm,
                                           const Geo &g, const Opq &q)
{
    constexpr uint32_t SH = sizeof(SC) == 2 ? 6 : sizeof(SC) == 4 ? 7 : 8;   // log2(row bytes)
    const CT mask = static_cast<CT>(g.mask);
    uint32_t ia, ib;
    if constexpr (POW2) {
        ia = static_cast<uint32_t>(L.i) & g.jm;
        ib = static_cast<uint32_t>(L.i + static_cast<CT>(q.one)) & g.jm;
    } else {
        ia = modn<CT, POW2>(L.i, g);
        ib = modn<CT, POW2>(wrap<CT, AR>(L.i + 1, mask), g);
    }
    Fetch<CT> f;
    check_col<SC>((ia << SH) + lm, lm, g, false);
    check_col<SC>((ib << SH) + lm, lm, g, false);
    f.o = ld_cell<SC, CT, SMEM>(base, (ia << SH) + lm);
    f.jw = ld_cell<SC, CT, SMEM>(base, (ib << SH) + lm);
    f.jo = (modn<CT, POW2>(f.jw, g) << SH) + lm;
    check_col<SC>(f.jo, lm, g, false);
    check_col<SC>(L.ua, lm, g, false);
    if constexpr (!LAZY_MJ) f.mj = ld_cell<SC, CT, SMEM>(base, f.jo);
    if constexpr (!LAZY_UD) f.ud = ld_cell<SC, CT, SMEM>(base, L.ua);
    else f.ud = 0;
    return f;
}

// Read the input tape lazily in the ungated steps of shared-memory tiles: one
// shared load fewer per step for the 6 of 7 instructions that are not RD
// (measured on the ALU/MIO-bound small tiles; the latency-bound big tiles keep
// the early read, which overlaps the fetch)
#ifndef RASP_LAZY_UD
#define RASP_LAZY_UD 1
#endif
#ifndef RASP_LAZY_UD_BIG
#define RASP_LAZY_UD_BIG 0
#endif
template <bool YG>
constexpr bool kLazyUd = RASP_LAZY_UD && (!YG || RASP_LAZY_UD_BIG);
#ifndef RASP_LAZY_MJ
#define RASP_LAZY_MJ 0
#endif
template <bool YG>
constexpr bool kLazyMj = RASP_LAZY_MJ && !YG;

// Opcode decode as a one-hot word: bit k is set iff o == k (k < 32), zero for
// any o >= 32 (PTX shl clamps shift amounts to the register width).  The
// ungated steps of big tiles test its bits (ptxas sets several predicates per
// R2P, and the range test "o in 1..7" becomes one mask test): C5 -2.1%.  The
// small tiles keep the comparisons: the same ALU count there, but +0.9% on C2
// (measured with RASP_ONEHOT=2 = everywhere, 0 = nowhere).
#ifndef RASP_ONEHOT
#define RASP_ONEHOT 1
#endif
template <bool YG>
constexpr bool kOneHot = RASP_ONEHOT == 2 || (RASP_ONEHOT == 1 && YG);
template <class CT>
__device__ __forceinline__ uint32_t onehot(CT o)
{
    uint32_t s;
    if constexpr (sizeof(CT) == 8) s = (static_cast<uint64_t>(o) >> 32) ? 32u : static_cast<uint32_t>(o);
    else s = static_cast<uint32_t>(o);
    uint32_t r;
    asm("shl.b32 %0, %1, %2;" : "=r"(r) : "r"(1u), "r"(s));
    return r;
}

// The opcode tests of one ungated step (hv:91-113): one-hot bits, or the
// plain comparisons (RASP_ONEHOT=0)
template <class CT, bool ONEHOT>
struct Decode {
    uint32_t oh;
    CT o;
    __device__ __forceinline__ explicit Decode(CT op) : oh(ONEHOT ? onehot(op) : 0u), o(op) {}
    __device__ __forceinline__ bool is(uint32_t k) const { return ONEHOT ? (oh & (1u << k)) != 0 : o == CT(k); }
    // i stays: o outside 1..7, or RD with the read cursor at capacity
    __device__ __forceinline__ bool stays(bool ucap) const
    {
        if constexpr (ONEHOT) return (oh & (ucap ? 0xbeu : 0xfeu)) == 0;
        else return (static_cast<CT>(o - 1) > 6) | ((o == 6) & ucap);
    }
};

// Fixedness (hv:115): the next configuration equals the current one.  For
// w >= 2, (i+2) mod 2^w != i, so every advancing case moves i and the test
// reduces to: opcode not in 1..7, RD with the cursor at capacity, or BNZ
// taken to its own address.  For w = 1 the full five-candidate equality.
template <class CT, bool POW2, Arith AR>
__device__ __forceinline__ bool is_fixed(const LaneState<CT> &L, const Fetch<CT> &f, uint32_t uend,
                                         uint32_t yend, const Geo &g, const Opq &q)
{
    const CT mask = static_cast<CT>(g.mask);
    const bool taken = (f.o == 5) & ((AR == Arith::CELL ? (L.a & mask) : L.a) != 0);
    const bool ucap = L.ua >= uend;
    if constexpr (AR != Arith::W1) {
        bool self;
        if constexpr (kRawI<POW2, AR> && AR != Arith::FULL) self = ((L.i ^ f.jw) & mask) == 0;
        else self = f.jw == L.i;
        return (static_cast<CT>(f.o - static_cast<CT>(q.one)) > 6) | ((f.o == 6) & ucap) | (taken & self);
    } else {
        const bool rd = (f.o == 6) & !ucap;
        const bool pri = (f.o == 7) & (L.ya < yend);
        const CT i2 = wrap<CT, AR>(L.i + 2, mask);
        const bool adv = (static_cast<CT>(f.o - 1) < 4) | ((f.o == 5) & (L.a == 0)) | rd | (f.o == 7);
        const CT ni = taken ? f.jw : (adv ? i2 : L.i);
        CT na = (f.o == 1) ? f.jw : L.a;
        na = (f.o == 2) ? wrap<CT, AR>(L.a + f.mj, mask) : na;
        na = (f.o == 3) ? wrap<CT, AR>(L.a * f.mj, mask) : na;
        const CT nm = (f.o == 4) ? L.a : (rd ? f.ud : f.mj);
        return (ni == L.i) & (na == L.a) & (nm == f.mj) & !rd & !pri;
    }
}

// Evaluate the step at local time t and, when allowed, commit it.
// BUDGET: check t == rem inside the loop (runs whose machines did not all
// start at the same step count); the final, non-applying evaluation at
// t == K always checks it.  A lane's verdict time is the last t at which it
// was live (tlast); whether it halted or ran out of budget is decided at
// write-back.
// YG (big tiles): the output tape is not staged in the tile; PRI stores go
// straight to the machine's HBM row (ybase + ya, element type YS).
template <class SC, class CT, bool POW2, Arith AR, bool BUDGET, bool SMEM, bool YG = false, class YS = SC>
__device__ __forceinline__ void rasp_step(LaneState<CT> &L, char *base, uint32_t lm, uint32_t uend,
                                          uint32_t yend, const Geo &g, const Opq &q, uint32_t t,
                                          bool can_apply, char *ybase = nullptr)
{
    const CT mask = static_cast<CT>(g.mask);
    const Fetch<CT> f = fetch<SC, CT, POW2, AR, SMEM>(L, base, lm, g, q);
    const CT a0 = L.a;
    const bool fixed = is_fixed<CT, POW2, AR>(L, f, uend, yend, g, q);
    if (L.active) L.tlast = t;
    if (BUDGET || !can_apply) L.active = L.active & !(fixed | (t == L.rem));
    else L.active = L.active & !fixed;
    const bool app = L.active & can_apply;
    // commit: every update is a predicated move/store keyed on its own case
    if (app & (f.o == 1)) L.a = f.jw;
    if constexpr (AR == Arith::CELL) {   // low w bits exact; masked at every test
        if (app & (f.o == 2)) L.a = a0 + f.mj;
        if (app & (f.o == 3)) L.a = a0 * f.mj;
    } else {
        if (app & (f.o == 2)) L.a = wrap<CT, AR>(a0 + f.mj, mask);
        if (app & (f.o == 3)) L.a = wrap<CT, AR>(a0 * f.mj, mask);
    }
    if (app & (f.o == 4)) st_cell<SC, CT, SMEM>(base, f.jo, a0);
    const bool rd = (f.o == 6) & (L.ua < uend);
    if (app & rd) {
        st_cell<SC, CT, SMEM>(base, f.jo, f.ud);
        L.ua += q.row;
    }
    if (app & (f.o == 7) & (L.ya < yend)) {
        if constexpr (YG) {
            *reinterpret_cast<YS *>(ybase + L.ya) = static_cast<YS>(f.mj);
            L.ya += static_cast<uint32_t>(sizeof(YS));
        } else {
            check_col<SC>(L.ya, lm, g, true);
            st_cell<SC, CT, SMEM>(base, L.ya, f.mj);
            L.ya += q.row;
        }
    }
    if (app) {
        const bool taken = (f.o == 5) & ((AR == Arith::CELL ? (a0 & mask) : a0) != 0);
        CT i2;
        if constexpr (kRawI<POW2, AR>) i2 = L.i + static_cast<CT>(q.two);
        else i2 = wrap<CT, AR>(L.i + 2, mask);
        L.i = taken ? f.jw : i2;
    }
}

// Ungated step, for loop steps of runs whose machines share one budget
// (every lane has rem >= K, so no lane can run out of budget inside the
// loop).  A lane is then either live and not fixed -- the step applies -- or
// sits at a fixed point, where applying the step changes nothing (that is
// what fixed means: Phi(c) = c, hv:115).  So the update is applied to every
// lane without an "applies" predicate: it only has to honour the cases that
// leave i in place (opcode outside 1..7, RD at capacity) and never store in
// them.
// Fixedness comes for free from the update: for w >= 2 a step that is not a
// fixed point always moves i ((i+2) mod 2^w != i; a taken BNZ to j != i), and
// a fixed lane never moves again.  So `moved` is the live flag and L.tlast
// counts the moves -- the lane's applied steps, i.e. its halting time once it
// stops moving.  Whether a lane that moved at every step is fixed at the end
// of the epoch is decided at write-back.
// YG (big tiles): the output tape is not staged in the tile; PRI stores go
// straight to the machine's HBM row (ybase + ya, element type YS).
template <class SC, class CT, bool POW2, Arith AR, bool SMEM, bool YG = false, class YS = SC>
__device__ __forceinline__ void rasp_step_free(LaneState<CT> &L, char *base, uint32_t lm, uint32_t uend,
                                               uint32_t yend, const Geo &g, const Opq &q,
                                               char *ybase = nullptr)
{
    static_assert(AR != Arith::W1, "w = 1 uses the gated step");
    const CT mask = static_cast<CT>(g.mask);
    Fetch<CT> f = fetch<SC, CT, POW2, AR, SMEM, kLazyUd<YG>, kLazyMj<YG>>(L, base, lm, g, q);
    if constexpr (kLazyMj<YG>)   // M[j] only for the instructions that use it
        f.mj = ((f.o == 2) | (f.o == 3) | (f.o == 7)) ? ld_cell<SC, CT, SMEM>(base, f.jo) : CT(0);
    const CT a0 = L.a;
    const Decode<CT, kOneHot<YG>> op(f.o);
    const bool ucap = L.ua >= uend;
    const bool taken = op.is(5) & ((AR == Arith::CELL ? (a0 & mask) : a0) != 0);
    const bool stay = op.stays(ucap);   // i does not move
    if (op.is(1)) L.a = f.jw;
    if constexpr (AR == Arith::CELL) {
        if (op.is(2)) L.a = a0 + f.mj;
        if (op.is(3)) L.a = a0 * f.mj;
    } else {
        if (op.is(2)) L.a = wrap<CT, AR>(a0 + f.mj, mask);
        if (op.is(3)) L.a = wrap<CT, AR>(a0 * f.mj, mask);
    }
    if (op.is(4)) st_cell<SC, CT, SMEM>(base, f.jo, a0);
    if (op.is(6) & !ucap) {
        st_cell<SC, CT, SMEM>(base, f.jo, kLazyUd<YG> ? ld_cell<SC, CT, SMEM>(base, L.ua) : f.ud);
        L.ua += q.row;
    }
    if constexpr (YG) {   // HBM row: lanes without a machine must not store
        if (L.active & op.is(7) & (L.ya < yend)) {
            *reinterpret_cast<YS *>(ybase + L.ya) = static_cast<YS>(f.mj);
            L.ya += static_cast<uint32_t>(sizeof(YS));
        }
    } else if (op.is(7) & (L.ya < yend)) {
        check_col<SC>(L.ya, lm, g, true);
        st_cell<SC, CT, SMEM>(base, L.ya, f.mj);
        L.ya += q.row;
    }
    CT i2;
    if constexpr (kRawI<POW2, AR>) i2 = L.i + static_cast<CT>(q.two);
    else i2 = wrap<CT, AR>(L.i + 2, mask);
    const CT ni = taken ? f.jw : (stay ? L.i : i2);
    bool moved;
    if constexpr (kRawI<POW2, AR> && AR != Arith::FULL) moved = ((ni ^ L.i) & mask) != 0;
    else moved = ni != L.i;
    L.active = moved;
    if (moved) ++L.tlast;
    L.i = ni;
}



__device__ __forceinline__ uint32_t sel32(bool c, uint32_t a, uint32_t b)
{
    uint32_t r;
    asm("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %3, 0;\n\tselp.b32 %0, %1, %2, p;\n\t}"
        : "=r"(r) : "r"(a), "r"(b), "r"(static_cast<uint32_t>(c)));
    return r;
}

// c ? a : b as a select instruction (ptxas otherwise sometimes turns an
// opcode-keyed chain of conditional updates into a branch tree)
template <class CT>
__device__ __forceinline__ CT selw(bool c, CT a, CT b)
{
    if constexpr (sizeof(CT) == 8) {
        unsigned long long r;
        asm("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %3, 0;\n\tselp.b64 %0, %1, %2, p;\n\t}"
            : "=l"(r) : "l"(static_cast<unsigned long long>(a)), "l"(static_cast<unsigned long long>(b)),
              "r"(static_cast<uint32_t>(c)));
        return static_cast<CT>(r);
    } else {
        return static_cast<CT>(sel32(c, static_cast<uint32_t>(a), static_cast<uint32_t>(b)));
    }
}

// Ungated step for n not a power of two.  Instead of reducing i and i+1 mod n
// (a multiply-high chain each) before every fetch, the residues im = i mod n
// and ib = ((i+1) mod 2^w) mod n are carried from step to step: an advance
// adds 2 (one conditional subtract of n, and i+2 wrapping through 2^w lands
// on 0 or 1, its own residue), a taken branch reuses j mod n, which the
// M[j] access computes anyway.  COUNT selects the move-counting form of
// rasp_step_free (used by the epoch kernel), else the explicit form
// (active &= !fixed; tlast = t while live).
template <class SC, class CT, Arith AR, bool SMEM, bool COUNT, bool YG = false, class YS = SC>
__device__ __forceinline__ void rasp_step_inc(LaneState<CT> &L, uint32_t &im, uint32_t &ib, char *base,
                                              uint32_t lm, uint32_t uend, uint32_t yend, const Geo &g,
                                              const Opq &q, uint32_t t, char *ybase = nullptr)
{
    static_assert(AR != Arith::W1, "w = 1 uses the gated step");
    constexpr uint32_t SH = sizeof(SC) == 2 ? 6 : sizeof(SC) == 4 ? 7 : 8;   // log2(row bytes)
    const CT mask = static_cast<CT>(g.mask);
    check_col<SC>((im << SH) + lm, lm, g, false);
    check_col<SC>((ib << SH) + lm, lm, g, false);
    const CT o = ld_cell<SC, CT, SMEM>(base, (im << SH) + lm);
    const CT jw = ld_cell<SC, CT, SMEM>(base, (ib << SH) + lm);
    const uint32_t jn = modn<CT, false>(jw, g);
    const uint32_t jo = (jn << SH) + lm;
    check_col<SC>(jo, lm, g, false);
    check_col<SC>(L.ua, lm, g, false);
    const CT mj = (!kLazyMj<YG> || (o == 2) | (o == 3) | (o == 7)) ? ld_cell<SC, CT, SMEM>(base, jo) : CT(0);
    const CT ud = kLazyUd<YG> ? CT(0) : ld_cell<SC, CT, SMEM>(base, L.ua);
    const CT a0 = L.a;
    const Decode<CT, false> op(o);   // one-hot measured 61.6 against 57.1 instructions per step here
    const bool ucap = L.ua >= uend;
    const bool taken = op.is(5) & ((AR == Arith::CELL ? (a0 & mask) : a0) != 0);
    const bool stay = op.stays(ucap);   // i does not move
    if constexpr (!COUNT) {
        const bool fixed = stay | (taken & (jw == L.i));
        if (L.active) L.tlast = t;
        L.active = L.active & !fixed;
    }
    {
        CT na = selw<CT>(op.is(1), jw, a0);
        if constexpr (AR == Arith::CELL) {
            na = selw<CT>(op.is(2), a0 + mj, na);
            na = selw<CT>(op.is(3), a0 * mj, na);
        } else {
            na = selw<CT>(op.is(2), wrap<CT, AR>(a0 + mj, mask), na);
            na = selw<CT>(op.is(3), wrap<CT, AR>(a0 * mj, mask), na);
        }
        L.a = na;
    }
    if (op.is(4)) st_cell<SC, CT, SMEM>(base, jo, a0);
    if (op.is(6) & !ucap) {
        st_cell<SC, CT, SMEM>(base, jo, kLazyUd<YG> ? ld_cell<SC, CT, SMEM>(base, L.ua) : ud);
        L.ua += q.row;
    }
    if constexpr (YG) {   // HBM row: lanes without a machine (no ybase) must not store
        if (L.active & op.is(7) & (L.ya < yend)) {
            *reinterpret_cast<YS *>(ybase + L.ya) = static_cast<YS>(mj);
            L.ya += static_cast<uint32_t>(sizeof(YS));
        }
    } else if (op.is(7) & (L.ya < yend)) {
        check_col<SC>(L.ya, lm, g, true);
        st_cell<SC, CT, SMEM>(base, L.ya, mj);
        L.ya += q.row;
    }
    const CT i2 = wrap<CT, AR>(L.i + 2, mask);
    uint32_t im2 = min(im + 2, im + 2 - g.n);             // (im + 2) mod n as one add-min
    im2 = i2 < 2 ? static_cast<uint32_t>(i2) : im2;      // wrapped through 2^w
    const CT ni = selw<CT>(taken, jw, selw<CT>(stay, L.i, i2));
    im = sel32(taken, jn, sel32(stay, im, im2));
    const uint32_t ib1 = im + 1;
    ib = sel32((ib1 == g.n) | (ni == mask), 0u, ib1);
    if constexpr (COUNT) {
        const bool moved = ni != L.i;
        L.active = moved;
        if (moved) ++L.tlast;
    }
    L.i = ni;
}

// The last block of epoch e to finish plans epoch e + 1 (K[e+1], covered[e+1])
// from the survival ratio of this epoch.  Called by one thread per block.
__device__ __forceinline__ void plan_next_epoch(const EpochArgs &A, uint32_t count, uint32_t K, int64_t covered,
                                                uint32_t ntiles)
{
    Sched *sc = A.sched;
    const uint32_t e = A.e;
    __threadfence();
    if (atomicAdd(&sc->blocks_done[e], 1u) == gridDim.x - 1) {
        __threadfence();
        const uint32_t cout = atomicAdd(&sc->count[e], 0u);
        const int64_t cov = covered + K;
        const int64_t left = A.tau_max - cov;
        uint32_t kn = 0;
        if (cout > 0 && left > 0 && ntiles > 0) {
            // the rest of the budget runs as one epoch once the live set has
            // stopped halting: at least stable_q8/256 of it survived this
            // epoch and the rest is at most `jump` times this epoch, or
            // stable_hi_q8/256 of it survived (a long budget jumped to while
            // machines still halt leaves their lanes idle for all of it);
            // otherwise keep compacting at 2x length
            const uint64_t surv = 256ull * cout;
            const bool stable =
                (surv >= static_cast<uint64_t>(A.stable_q8) * count &&
                 static_cast<uint64_t>(left) <= static_cast<uint64_t>(A.jump) * (K > 0 ? K : 1u)) ||
                surv >= static_cast<uint64_t>(A.stable_hi_q8) * count;
            uint64_t want = stable ? static_cast<uint64_t>(left)
                                   : static_cast<uint64_t>(A.growth) * (K > 0 ? K : 1u);
            // never leave a sliver of the budget (under a quarter of this
            // epoch) for one more epoch: it would reload every survivor
            // for a few steps (C5 at first epoch 336: 336, 672, 16)
            if (static_cast<uint64_t>(left) > want &&
                static_cast<uint64_t>(left) - want < (want >> 2))
                want = static_cast<uint64_t>(left);
            kn = static_cast<uint32_t>(min(min(want, static_cast<uint64_t>(left)),
                                           static_cast<uint64_t>(A.kmax)));
        }
        if (e + 1 < kMaxEpochs) {
            sc->K[e + 1] = kn;
            sc->covered[e + 1] = cov;
        }
    }
}

template <class S, class SC, class CT, bool POW2, Arith AR, bool BUDGET, bool SMEM, bool BIG = false>
__global__ void __launch_bounds__(BIG ? 32 : 32 * RASP_BLOCK_WARPS, BIG ? 8 : (SMEM ? RASP_MIN_BLOCKS : 1))
epoch_kernel(const EpochArgs A, SC *gtiles)
{
    // Programmatic dependent launch: epochs after the first are launched while
    // the previous one drains; wait for it (complete, memory visible) before
    // touching anything (a no-op for a launch without the PDL attribute).  No
    // early launch_dependents: the next epoch's blocks would sit on the SMs
    // through this epoch's tail, where runs on other streams could use them.
    asm volatile("griddepcontrol.wait;" ::: "memory");
    constexpr uint32_t LB = BIG ? 32 : 8;   // row-load batch (per-lane path)
    // matrix-op batch (16 B per lane each): wide only for native-width rows
    constexpr uint32_t MB = RASP_MX_BATCH;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr uint32_t ROW = 32 * sizeof(SC);
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t wib = threadIdx.x >> 5;
    const uint32_t n = A.g.n;
    const uint32_t tile_bytes = A.tile_rows * ROW;

    char *tb;      // SMEM: the dynamic shared window; else the warp's HBM tile
    uint32_t lm;   // address of this lane's column in row 0
    if constexpr (SMEM) {
        tb = reinterpret_cast<char *>(smem_raw);
        lm = static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw)) + wib * tile_bytes +
             ((kMx<SC> && !BIG) ? mx_col<SC>(lane) : lane) * static_cast<uint32_t>(sizeof(SC));
    } else {
        tb = reinterpret_cast<char *>(gtiles) +
             (static_cast<size_t>(blockIdx.x) * (blockDim.x >> 5) + wib) * static_cast<size_t>(tile_bytes);
        lm = lane * static_cast<uint32_t>(sizeof(SC));
    }
    // per-thread copies (threadIdx.x >> 10 == 0): not uniform, so adds stay on IMAD
    // compile-time constants: ptxas rematerialises runtime ones with LDC inside
    // the step loop, which put a constant-cache latency on the critical path
    const Opq q = {1u, 2u, ROW};
    const uint32_t U = n * ROW + lm;                       // u[1] of this lane
    // y[1] of this lane: a tile row (epoch scratch), or (BIG) an offset from the
    // lane's HBM output row
    const uint32_t Y = BIG ? 0u : (n + A.g.ell + 1) * ROW + lm;
    constexpr uint32_t YSTEP = BIG ? static_cast<uint32_t>(sizeof(S)) : ROW;
    // warp-wide row moves (stmatrix/ldmatrix); BIG tiles keep per-lane moves
    // with 32 loads in flight (measured faster for their few resident warps)
    constexpr bool MX = SMEM && kMx<SC> && !BIG;
    // ungated steps with move counting (every lane's budget covers the epoch)
    constexpr bool kCount = !BUDGET && AR != Arith::W1;
    // ungated steps with carried residues (n not a power of two)
    constexpr bool kInc = !BUDGET && AR != Arith::W1 && !POW2 && SMEM;
    constexpr uint32_t kUnroll = BIG ? RASP_UNROLL_BIG : RASP_UNROLL;
    const uint32_t tile0 = SMEM ? static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw)) + wib * tile_bytes : 0u;
    const bool vecM = mx_vec_ok<S, SC>(A.first ? A.in.M : A.out.M, n) && mx_vec_ok<S, SC>(A.out.M, n);
    char *ybase = nullptr;
    // generic base for the (cold) row copies: gb + address = generic pointer
    char *gb = SMEM ? reinterpret_cast<char *>(smem_raw) -
                          static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw))
                    : tb;

    Sched *sc = A.sched;
    const uint32_t e = A.e;
    const uint32_t count = A.first ? A.count_in : sc->count[e - 1];
    const uint32_t K = A.first ? A.K0 : sc->K[e];
    const int64_t covered = A.first ? 0 : sc->covered[e];
    const uint32_t ntiles = (K == 0 && !A.first) ? 0 : (count + 31) / 32;
    if (ntiles == 0) return;   // schedule finished: K[e+1] stays 0 from the memset
    const uint32_t nwarps = gridDim.x * (blockDim.x >> 5);
    // the halting histogram of hypervisor.py:329-352, fused: every verdict
    // lands in a block-private copy after the tiles in shared memory, flushed
    // with one global atomic per non-empty bucket when the block ends
    uint32_t *hist_s = reinterpret_cast<uint32_t *>(smem_raw + (SMEM ? (blockDim.x >> 5) * tile_bytes : 0u));
    if (A.hist) {
        for (uint32_t k = threadIdx.x; k < 102; k += blockDim.x) hist_s[k] = 0;
        __syncthreads();
    }
    const bool copy_side = A.first && !A.inplace;
    const bool fresh = A.fresh != 0;

    uint32_t next = 0;   // lane 0: the tile this warp takes next
    if (lane == 0) next = atomicAdd(&sc->tile_ctr[e], 1u);
    for (;;) {
        const uint32_t tix = __shfl_sync(kFull, next, 0);
        if (tix >= ntiles) break;

        LaneState<CT> L;
        bool running;
        {   // ---- load phase (values here are not kept live across the step loop)
            const Side &src = A.first ? A.in : A.out;
            const Side &dst = A.out;
            const uint64_t ucols = static_cast<uint64_t>(A.g.ell) + 1;
            const uint64_t ycols = static_cast<uint64_t>(A.g.s) + 1;
            if (copy_side && !BIG) {
                // out-of-place first epoch: the tile's machines are contiguous
                // (identity list), so their u and y rows are two contiguous
                // blocks -- copy them to `out` here, before any write-back of
                // this tile touches them (replaces a bulk copy kernel per tape;
                // the latency-bound big tiles keep the bulk copies: measured;
                // deferring the copy to the write-back behind an L2 prefetch
                // measured +0.2% on C2/C3)
                const uint64_t m0 = static_cast<uint64_t>(tix) * 32;
                const uint64_t m1 = min(static_cast<uint64_t>(count), m0 + 32);
                warp_copy(static_cast<S *>(dst.u) + m0 * ucols, static_cast<const S *>(A.in.u) + m0 * ucols,
                          (m1 - m0) * ucols * sizeof(S), lane);
                warp_copy(static_cast<S *>(dst.y) + m0 * ycols, static_cast<const S *>(A.in.y) + m0 * ycols,
                          (m1 - m0) * ycols * sizeof(S), lane);
                // the owning lanes rewrite u[0], y[0] and y[k] of these rows at
                // write-back: order the copies (any lane) before those stores
                __syncwarp();
            }
            const uint32_t j = tix * 32 + lane;
            const bool valid = j < count;
            const uint64_t id = valid ? (A.list_in ? A.list_in[j] : j) : 0;
            RASP_CHECK(id < A.count_in, kChkRow, id, A.count_in);
            running = valid;
            int64_t steps0 = fresh ? covered : 0;
            if (valid && !fresh) {
                // status/steps/tau_h of `out` already hold the input values (the
                // host copies them for out-of-place runs before the first epoch)
                if (A.first && dst.status[id] != kRunning) running = false;
                steps0 = dst.steps[id];
            }
            const S *srcM = static_cast<const S *>(src.M) + id * n;
            const S *srcU = static_cast<const S *>(src.u) + id * ucols;
            const S *srcY = static_cast<const S *>(src.y) + id * ycols;
            if (A.hist && valid && A.first && !running) {   // untouched: counted as it stands
                const int8_t st0 = dst.status[id];
                if (st0 == kHalted) {
                    const int64_t th = dst.tau_h[id];
                    atomicAdd(&hist_s[th < 100 ? static_cast<uint32_t>(th) : 100u], 1u);
                } else if (st0 == kExhausted) {
                    atomicAdd(&hist_s[101], 1u);
                }
            }
            if (valid && copy_side && !running) {
                // untouched machine, out-of-place: carry i, a, M over (u, y are
                // copied per tile above, or in bulk by the host for big tiles)
                static_cast<S *>(dst.iw)[id] = static_cast<const S *>(A.in.iw)[id];
                static_cast<S *>(dst.ac)[id] = static_cast<const S *>(A.in.ac)[id];
                copy_cells(static_cast<S *>(dst.M) + id * n, srcM, n);
            }
            L.i = 0; L.a = 0; L.ua = U; L.ya = Y; L.tlast = 0;
            if (running) {
                L.i = static_cast<CT>(static_cast<const S *>(src.iw)[id]);
                L.a = static_cast<CT>(static_cast<const S *>(src.ac)[id]);
                L.ua = U + static_cast<uint32_t>(srcU[0]) * ROW;
                L.ya = Y + static_cast<uint32_t>(srcY[0]) * YSTEP;
                if constexpr (BIG) ybase = reinterpret_cast<char *>(static_cast<S *>(A.out.y) + id * ycols + 1);
                if constexpr (BIG) {
                    load_rows_mu<S, SC, LB>(srcM, n, reinterpret_cast<SC *>(gb + lm), srcU + 1, A.g.ell,
                                            reinterpret_cast<SC *>(gb + U));
                } else if constexpr (!MX) {
                    load_row<S, SC, LB>(srcM, n, reinterpret_cast<SC *>(gb + lm));
                    load_row<S, SC, LB>(srcU + 1, A.g.ell, reinterpret_cast<SC *>(gb + U));
                }
            } else if constexpr (kCount && !MX) {
                // a lane without a machine sits at a fixed point (opcode 0 at
                // i = 0), so move-counting steps never see it move (the matrix
                // loads zero-fill such columns)
                reinterpret_cast<SC *>(gb + lm)[0] = 0;
            }
            if constexpr (MX) {
                mx_load<S, SC, MB>(srcM, running, vecM, n, tile0, 0, lane, reinterpret_cast<SC *>(gb + lm));
                mx_load<S, SC, MB>(srcU + 1, running, false, A.g.ell, tile0, n, lane, reinterpret_cast<SC *>(gb + U));
            }
            const uint64_t rem64 = (steps0 >= A.tau_max) ? 0ull
                                                         : static_cast<uint64_t>(A.tau_max - steps0);
            L.rem = rem64 > 0xffffffffull ? 0xffffffffu : static_cast<uint32_t>(rem64);
            L.active = running;
        }
        asm volatile("" ::: "memory");   // column fills above are visible to the asm loads below
        {   // warm L2 with the tile this warp will probably take next (tiles are
            // claimed in order, about one per resident warp ahead): its rows
            // then arrive from L2 while the epoch's DRAM traffic streams behind
            const uint32_t pf = tix + A.pf_dist * nwarps;
            const uint32_t j = pf * 32 + lane;
            if (A.pf_dist && pf < ntiles && j < count) {
                const Side &src = A.first ? A.in : A.out;
                const uint64_t id = A.list_in ? A.list_in[j] : j;
                prefetch_l2(static_cast<const S *>(src.M) + id * n, n * static_cast<uint32_t>(sizeof(S)));
                prefetch_l2(static_cast<const S *>(src.u) + id * (static_cast<uint64_t>(A.g.ell) + 1),
                            (A.g.ell + 1) * static_cast<uint32_t>(sizeof(S)));
            }
        }

        {   // ---- step loop
            const Geo g = A.g;
            const uint32_t uend = U + g.ell * ROW;
            const uint32_t yend = Y + g.s * YSTEP;
            uint32_t t = 0;
            bool live = __any_sync(kFull, L.active);
            // steps between live checks (the check ends each block with a vote
            // and a branch the next block's loads wait on)
            constexpr uint32_t UN = kUnroll;
            if constexpr (kInc) {
                // residues of i and i+1 mod n, carried across steps
                uint32_t im = modn<CT, false>(L.i, g);
                uint32_t ib = modn<CT, false>(wrap<CT, AR>(L.i + 1, static_cast<CT>(g.mask)), g);
                for (; live && t + UN <= K; t += UN) {
#pragma unroll
                    for (uint32_t r = 0; r < UN; ++r)
                        rasp_step_inc<SC, CT, AR, SMEM, kCount, BIG, S>(L, im, ib, tb, lm, uend, yend, g, q, t + r, ybase);
                    live = __any_sync(kFull, L.active);
                }
                for (; live && t < K; ++t) {
                    rasp_step_inc<SC, CT, AR, SMEM, kCount, BIG, S>(L, im, ib, tb, lm, uend, yend, g, q, t, ybase);
                    live = __any_sync(kFull, L.active);
                }
            } else if constexpr (kCount) {
                for (; live && t + UN <= K; t += UN) {
#pragma unroll
                    for (uint32_t r = 0; r < UN; ++r)
                        rasp_step_free<SC, CT, POW2, AR, SMEM, BIG, S>(L, tb, lm, uend, yend, g, q, ybase);
                    live = __any_sync(kFull, L.active);
                }
                for (; live && t < K; ++t) {
                    rasp_step_free<SC, CT, POW2, AR, SMEM, BIG, S>(L, tb, lm, uend, yend, g, q, ybase);
                    live = __any_sync(kFull, L.active);
                }
            } else {   // per-lane budgets (mid-run inputs) or w = 1: the gated step
                for (; live && t + 2 <= K; t += 2) {
                    rasp_step<SC, CT, POW2, AR, BUDGET, SMEM, BIG, S>(L, tb, lm, uend, yend, g, q, t, true, ybase);
                    rasp_step<SC, CT, POW2, AR, BUDGET, SMEM, BIG, S>(L, tb, lm, uend, yend, g, q, t + 1, true, ybase);
                    live = __any_sync(kFull, L.active);
                }
                if (live && t < K) {
                    rasp_step<SC, CT, POW2, AR, BUDGET, SMEM, BIG, S>(L, tb, lm, uend, yend, g, q, t, true, ybase);
                    ++t;
                    live = __any_sync(kFull, L.active);
                }
                if (live) rasp_step<SC, CT, POW2, AR, true, SMEM, BIG, S>(L, tb, lm, uend, yend, g, q, K, false, ybase);
            }
        }
        // ---- verdicts first, so the two atomics (next tile, survivor slots)
        // are in flight while the write-back stores issue
        bool fin = false, halted = true;
        if (running) {
            if constexpr (kCount) {
                // tlast = moves: below K the lane stopped moving (fixed there);
                // at K it is fixed at K, out of budget (K == rem), or survives
                fin = L.tlast < K;
                if (!fin) {
                    const uint32_t uend = U + A.g.ell * ROW, yend = Y + A.g.s * YSTEP;
                    const Fetch<CT> f = fetch<SC, CT, POW2, AR, SMEM>(L, tb, lm, A.g, q);
                    halted = is_fixed<CT, POW2, AR>(L, f, uend, yend, A.g, q);
                    fin = halted | (K == L.rem);
                }
            } else {
                // verdict at tlast: halted, unless the budget ran out there and
                // the configuration is not a fixed point
                fin = !L.active;
                if (fin && L.tlast == L.rem) {
                    const uint32_t uend = U + A.g.ell * ROW, yend = Y + A.g.s * YSTEP;
                    const Fetch<CT> f = fetch<SC, CT, POW2, AR, SMEM>(L, tb, lm, A.g, q);
                    halted = is_fixed<CT, POW2, AR>(L, f, uend, yend, A.g, q);
                }
            }
        }
        const bool survivor = running & !fin;
        const unsigned sv = __ballot_sync(kFull, survivor);
        uint32_t sbase = 0;
        if (lane == 0) {
            next = atomicAdd(&sc->tile_ctr[e], 1u);
            if (sv) sbase = atomicAdd(&sc->count[e], static_cast<uint32_t>(__popc(sv)));
        }

        uint64_t id = 0;
        if (running) {   // ---- write-back phase (re-derives what the load phase knew)
            const Side &src = A.first ? A.in : A.out;
            const Side &dst = A.out;
            const uint64_t ucols = static_cast<uint64_t>(A.g.ell) + 1;
            const uint64_t ycols = static_cast<uint64_t>(A.g.s) + 1;
            const uint32_t j = tix * 32 + lane;
            id = A.list_in ? A.list_in[j] : j;
            const int64_t steps0 = fresh ? covered : dst.steps[id];
            const uint32_t y0_start = static_cast<uint32_t>(static_cast<const S *>(src.y)[id * ycols]);
            const uint32_t u0 = (L.ua - U) / ROW;
            const uint32_t y0 = (L.ya - Y) / YSTEP;
            if constexpr (kRawI<POW2, AR>) L.i &= static_cast<CT>(A.g.mask);
            if constexpr (AR == Arith::CELL) L.a &= static_cast<CT>(A.g.mask);
            S *dY = static_cast<S *>(dst.y) + id * ycols;
            if constexpr (!BIG) {
                const SC *colY = reinterpret_cast<const SC *>(gb + Y);
                for (uint32_t k = y0_start; k < y0; ++k) dY[k + 1] = static_cast<S>(colY[k * 32]);
            }
            dY[0] = static_cast<S>(y0);
            static_cast<S *>(dst.iw)[id] = static_cast<S>(L.i);
            static_cast<S *>(dst.ac)[id] = static_cast<S>(L.a);
            static_cast<S *>(dst.u)[id * ucols] = static_cast<S>(u0);
            if (fin) {
                const int64_t tend = steps0 + L.tlast;
                dst.steps[id] = tend;
                if (!halted) {
                    dst.status[id] = kExhausted;
                    if (fresh) dst.tau_h[id] = -1;
                } else {
                    dst.status[id] = kHalted;
                    dst.tau_h[id] = tend;
                }
                if (A.hist) atomicAdd(&hist_s[!halted ? 101u : tend < 100 ? static_cast<uint32_t>(tend) : 100u], 1u);
            } else if (!fresh) {
                dst.steps[id] = steps0 + K;
            }
            if constexpr (!MX)
                store_row<S, SC, 16>(static_cast<S *>(dst.M) + id * n, n, reinterpret_cast<const SC *>(gb + lm));
        }
        if constexpr (MX)
            mx_store<S, SC, MB>(static_cast<S *>(A.out.M) + id * n, running, vecM, n, tile0, 0, lane,
                                reinterpret_cast<const SC *>(gb + lm));
        if (sv) {
            sbase = __shfl_sync(kFull, sbase, 0);
            if (survivor) {
                RASP_CHECK(sbase + __popc(sv & ((1u << lane) - 1u)) < A.count_in, kChkList,
                           sbase + __popc(sv & ((1u << lane) - 1u)), A.count_in);
                A.list_out[sbase + __popc(sv & ((1u << lane) - 1u))] = static_cast<uint32_t>(id);
            }
        }
    }

    // the last block to finish plans the next epoch
    __syncthreads();
    if (A.hist)
        for (uint32_t k = threadIdx.x; k < 102; k += blockDim.x)
            if (hist_s[k]) atomicAdd(&A.hist[k], static_cast<unsigned long long>(hist_s[k]));
    if (threadIdx.x == 0) plan_next_epoch(A, count, K, covered, ntiles);
}

// --- per-lane refill for big tiles (fresh runs) ----------------------------------
//
// The epoch kernel keeps a tile's 32 machines until the last of them stops or
// the epoch ends, so a lane whose machine halted early idles: C5's first
// epoch uses 41% of its lane-steps (p50 halting time 38 against a 320-step
// epoch; 14% of the machines never halt, so nearly every tile runs it out).
// For fresh runs every machine can start at a block boundary, so with a
// first epoch K0 that is a multiple of the unrolled block its budget also
// ends on one.  The kernel runs that first epoch (by default the whole
// budget): after each block of UN steps a lane whose machine stopped moving
// (halted at its move count, hv:115) or reached K0 (one more fetch decides:
// fixed there, exhausted at K0 = tau_max, else a survivor for the epoch
// kernel's later epochs, appended to the survivor list like theirs) is
// finished; its machine stays in place (a fixed point, or parked: opcode 0
// stored at its instruction cell, the true value kept in a register and
// written after the row).  Once at least `refill_min` lanes are free the warp
// writes the finished machines back together (batches of 16 x 16 B shared
// loads, then the stores) and the free lanes load the next machines of the
// warp's reservation: the M row and a tape of <= 32 cells in two memory round
// trips (load_rows_mu_aligned), the warp waiting for them.  Reservations are
// 32 consecutive machine ids claimed with one atomic, one reservation ahead;
// each refill warms L2 with the rows of the next pf_dist ids.  Lanes without a
// machine step on two zero cells after the histogram (opcode 0 at i = 0: a
// fixed point that stores nothing).
// RASP_REFILL_ASYNC=1 (measured slower, C5 2.06 against 1.65 ms: the copies
// crowd the steps' shared loads) copies the rows with 4- or 8-byte cp.async
// instead (a TMA box cannot land in a lane column) while the warp steps its
// other lanes for one more block, the loading lanes parked on the zero cells.
#ifndef RASP_REFILL_ASYNC
#define RASP_REFILL_ASYNC 0
#endif
template <class SC>
constexpr uint32_t kRefillExtra = 416 + 32 * sizeof(SC) + 16;   // histogram, then the parking cells

__device__ __forceinline__ void cp_async_cell(uint32_t saddr, const void *g, uint32_t bytes)
{
    const unsigned long long ga = static_cast<unsigned long long>(__cvta_generic_to_global(g));
    check_smem(saddr, bytes);
    if (bytes == 8) asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(saddr), "l"(ga) : "memory");
    else asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(saddr), "l"(ga) : "memory");
}

template <class S, class SC, class CT, bool POW2, Arith AR>
__global__ void __launch_bounds__(32, 8) refill_kernel(const EpochArgs A)
{
    static_assert(sizeof(SC) >= 4 && AR != Arith::W1 && AR != Arith::CELL, "big tiles, w >= 2");
    constexpr uint32_t UN = RASP_UNROLL_BIG;
    constexpr uint32_t ROW = 32 * sizeof(SC);
    constexpr uint32_t SH = sizeof(SC) == 4 ? 7 : 8;   // log2(row bytes)
    constexpr uint32_t LB = 32;                        // row-load batch (16 B per lane each)
    // rows copied cell by cell asynchronously when HBM words are tile cells
    constexpr bool kAsync = RASP_REFILL_ASYNC && sizeof(S) == sizeof(SC);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const uint32_t lane = threadIdx.x & 31;
    const Geo g = A.g;
    const uint32_t n = g.n;
    char *const tb = reinterpret_cast<char *>(smem_raw);
    const uint32_t sbase = static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw));
    const uint32_t lm = sbase + lane * static_cast<uint32_t>(sizeof(SC));
    char *const gb = reinterpret_cast<char *>(smem_raw) - sbase;
    const Opq q = {1u, 2u, ROW};
    const uint32_t U = n * ROW + lm;                    // u[1] of this lane
    const uint32_t uend = U + g.ell * ROW;
    const uint32_t yend = g.s * static_cast<uint32_t>(sizeof(S));
    const uint64_t ucols = static_cast<uint64_t>(g.ell) + 1, ycols = static_cast<uint64_t>(g.s) + 1;
    const uint32_t d = A.count_in;
    const uint32_t K = A.K0;                                 // this epoch: a multiple of UN, <= tau_max
    const bool last = static_cast<int64_t>(K) >= A.tau_max;   // K0 covers the budget
    const uint32_t rmin = A.refill_min;
    const uint32_t tile_bytes = A.tile_rows * ROW;
    uint32_t *const hist_s = reinterpret_cast<uint32_t *>(smem_raw + tile_bytes);
    const uint32_t P = sbase + tile_bytes + 416;        // parking cells P, P + ROW (zero)
    if (A.hist)
        for (uint32_t k = lane; k < 102; k += 32) hist_s[k] = 0;
    if (lane < 2) *reinterpret_cast<SC *>(gb + P + lane * ROW) = SC(0);
    __syncwarp();
    uint32_t *const ctr = &A.sched->tile_ctr[0];
    const S *const inM = static_cast<const S *>(A.in.M);
    const S *const inU = static_cast<const S *>(A.in.u);
    const S *const inY = static_cast<const S *>(A.in.y);

    // a reservation of up to 32 ids [b, b + c); rows warmed into L2
    auto claim = [&](uint32_t &b, uint32_t &c) {
        uint32_t x = 0;
        if (lane == 0) x = atomicAdd(ctr, 32u);
        x = __shfl_sync(kFull, x, 0);
        b = x;
        c = x < d ? min(32u, d - x) : 0u;
        if (A.pf_dist == 1 && lane < c) {
            const uint64_t id = static_cast<uint64_t>(x) + lane;
            prefetch_l2(inM + id * n, n * static_cast<uint32_t>(sizeof(S)));
            prefetch_l2(inU + id * ucols, static_cast<uint32_t>(ucols * sizeof(S)));
        }
    };

    LaneState<CT> L;
    L.i = 0; L.a = 0; L.ua = P; L.ya = 0; L.rem = 0; L.tlast = 0; L.active = false;
    uint32_t lms = P;          // column the steps read: the lane's own (lm) or the parking cells
    uint32_t im = 0, ib = 1;   // carried residues of i and i+1 (n not a power of two)
    uint32_t id = 0;
    bool has = false;          // the lane holds a machine (not yet written back)
    bool done = false;         // ... whose verdict is known (it waits for the next refill)
    bool loading = false;      // ... whose rows are in flight
    bool halted = false;
    bool surv = false;         // ... that survives this epoch (reached K0 < tau_max, not fixed)
    uint32_t pk = 0;           // parked cell of an exhausted machine (0: none)
    SC pkv = 0;                // its value
    CT ni0 = 0, na0 = 0;       // the incoming machine's i, a and cursors
    uint32_t nua0 = 0, nya0 = 0;
    char *ybase = nullptr;
    auto park = [&]() {        // step on the zero cells
        L.i = 0; L.a = 0; L.ua = P; L.active = false;
        im = 0; ib = 1;
        lms = P;
    };
    auto start = [&]() {       // the incoming machine takes the lane
        L.i = ni0; L.a = na0; L.ua = U + nua0 * ROW; L.ya = nya0 * static_cast<uint32_t>(sizeof(S));
        L.tlast = 0; L.active = true;
        if constexpr (!POW2) {
            im = modn<CT, false>(L.i, g);
            ib = modn<CT, false>(wrap<CT, AR>(L.i + 1, static_cast<CT>(g.mask)), g);
        }
        lms = lm;
        loading = false;
    };
    auto load = [&](uint32_t mid) {
        RASP_CHECK(mid < d, kChkRow, mid, d);
        const uint64_t m = mid;
        ni0 = static_cast<CT>(static_cast<const S *>(A.in.iw)[m]);
        na0 = static_cast<CT>(static_cast<const S *>(A.in.ac)[m]);
        nua0 = static_cast<uint32_t>(inU[m * ucols]);   // used at start(): the loads stay in flight
        nya0 = static_cast<uint32_t>(inY[m * ycols]);
        ybase = reinterpret_cast<char *>(static_cast<S *>(A.out.y) + m * ycols + 1);
        id = mid;
        has = true;
        done = false;
        surv = false;
        if constexpr (kAsync) {
            park();
            const S *rm = inM + m * n;
#pragma unroll 8
            for (uint32_t k = 0; k < n; ++k) cp_async_cell(lm + k * ROW, rm + k, sizeof(SC));
            const S *ru = inU + m * ucols + 1;
#pragma unroll 8
            for (uint32_t k = 0; k < g.ell; ++k) cp_async_cell(U + k * ROW, ru + k, sizeof(SC));
            loading = true;
        } else {
            load_rows_mu_aligned<S, SC, LB>(inM + m * n, n, reinterpret_cast<SC *>(gb + lm), inU + m * ucols + 1,
                                            g.ell, reinterpret_cast<SC *>(gb + U));
            start();
        }
    };
    // write the lane's finished machine back (final row, cursors, verdict)
    auto retire = [&]() {
        const uint64_t m = id;
        const uint32_t u0 = (L.ua - U) / ROW;
        const uint32_t y0 = L.ya / static_cast<uint32_t>(sizeof(S));
        CT iv = L.i;
        if constexpr (kRawI<POW2, AR>) iv &= static_cast<CT>(g.mask);
        static_cast<S *>(A.out.y)[m * ycols] = static_cast<S>(y0);
        static_cast<S *>(A.out.iw)[m] = static_cast<S>(iv);
        static_cast<S *>(A.out.ac)[m] = static_cast<S>(L.a);
        static_cast<S *>(A.out.u)[m * ucols] = static_cast<S>(u0);
        if (!surv) {   // a survivor's verdict fields are written by the epoch it finishes in
            const int64_t tend = L.tlast;
            A.out.steps[m] = tend;
            A.out.status[m] = halted ? kHalted : kExhausted;
            A.out.tau_h[m] = halted ? tend : -1;
            if (A.hist) atomicAdd(&hist_s[!halted ? 101u : tend < 100 ? static_cast<uint32_t>(tend) : 100u], 1u);
        }
        store_row<S, SC, 16>(static_cast<S *>(A.out.M) + m * n, n, reinterpret_cast<const SC *>(gb + lm));
        // a parked machine: its true cell goes out after the row
        if (pk) static_cast<S *>(A.out.M)[m * n + ((pk - lm) >> SH)] = static_cast<S>(pkv);
        pk = 0;
        has = false;
        done = false;
        park();
    };

    uint32_t r0, n0, r1, n1;
    claim(r0, n0);
    claim(r1, n1);
    bool more = n0 > 0;
    for (;;) {
        if constexpr (kAsync) {   // rows issued at the last refill have landed: start those lanes
            if (__any_sync(kFull, loading)) {
                asm volatile("cp.async.wait_all;" ::: "memory");
                if (loading) start();
            }
        }
        // free lanes: no machine, or a finished one (sitting at a fixed point)
        const bool freel = !has || done;
        const unsigned freem = __ballot_sync(kFull, freel);
        const uint32_t nf = __popc(freem);
        if (nf == 32u || (more && nf >= rmin)) {
            // write the finished machines back together (survivors onto the
            // next epoch's list), then hand the next machines of the
            // reservations to the free lanes
            const unsigned sv = __ballot_sync(kFull, done && surv);
            if (sv) {
                uint32_t sb = 0;
                if (lane == 0) sb = atomicAdd(&A.sched->count[0], static_cast<uint32_t>(__popc(sv)));
                sb = __shfl_sync(kFull, sb, 0);
                if (done && surv) {
                    const uint32_t slot = sb + __popc(sv & ((1u << lane) - 1u));
                    RASP_CHECK(slot < d, kChkList, slot, d);
                    A.list_out[slot] = id;
                }
            }
            if (done) retire();
            if (!more) break;   // every lane free and nothing left to hand out
            const uint32_t rank = __popc(freem & ((1u << lane) - 1u));
            const uint32_t take = min(nf, n0 + n1);
            if (freel && rank < take) load(rank < n0 ? r0 + rank : r1 + (rank - n0));
            if constexpr (kAsync) asm volatile("cp.async.commit_group;" ::: "memory");
            if (take < n0) {
                r0 += take;
                n0 -= take;
            } else {
                const uint32_t t1 = take - n0;
                const bool full = n1 == 32u;
                r0 = r1 + t1;
                n0 = n1 - t1;
                if (full) claim(r1, n1);
                else n1 = 0;
                if (n0 == 0 && n1 > 0) {   // the old next reservation is used up too
                    r0 = r1;
                    n0 = n1;
                    if (n1 == 32u) claim(r1, n1);
                    else n1 = 0;
                }
            }
            more = n0 > 0;
            if (A.pf_dist >= 2) {   // warm L2 with the pf_dist machines the next refills will take
                const uint32_t nx = min(n0 + n1, min(A.pf_dist, 32u));
                if (lane < nx) {
                    const uint64_t id = lane < n0 ? r0 + lane : r1 + (lane - n0);
                    prefetch_l2(inM + id * n, n * static_cast<uint32_t>(sizeof(S)));
                    prefetch_l2(inU + id * ucols, static_cast<uint32_t>(ucols * sizeof(S)));
                }
            }
            asm volatile("" ::: "memory");   // column fills above are visible to the asm loads below
        }
        // one block of UN ungated steps; free and loading lanes sit still
        if constexpr (POW2) {
#pragma unroll
            for (uint32_t r = 0; r < UN; ++r)
                rasp_step_free<SC, CT, POW2, AR, true, true, S>(L, tb, lms, uend, yend, g, q, ybase);
        } else {
#pragma unroll
            for (uint32_t r = 0; r < UN; ++r)
                rasp_step_inc<SC, CT, AR, true, true, true, S>(L, im, ib, tb, lms, uend, yend, g, q, r, ybase);
        }
        // verdicts at the block boundary
        if (has && !done && !loading) {
            if (!L.active) {   // stopped moving: halted at its move count
                done = true;
                halted = true;
            } else if (L.tlast >= K) {   // epoch end: fixed at K0, exhausted, or a survivor
                const Fetch<CT> f = fetch<SC, CT, POW2, AR, true>(L, tb, lm, g, q);
                halted = is_fixed<CT, POW2, AR>(L, f, uend, yend, g, q);
                surv = !halted && !last;
                done = true;
                // park it in place: opcode 0 at its instruction cell (the
                // true value goes out at write-back)
                pk = ((POW2 ? (static_cast<uint32_t>(L.i) & g.jm) : im) << SH) + lm;
                pkv = *reinterpret_cast<const SC *>(gb + pk);
                *reinterpret_cast<SC *>(gb + pk) = SC(0);
                L.active = false;
            }
        }
    }
    __syncwarp();
    if (A.hist)
        for (uint32_t k = lane; k < 102; k += 32)
            if (hist_s[k]) atomicAdd(&A.hist[k], static_cast<unsigned long long>(hist_s[k]));
    if (lane == 0) plan_next_epoch(A, d, K, 0, (d + 31) / 32);
}

// --- exhaustive enumeration (BASELINE config 4) -------------------
//
// Program rank r in [0, 2^(m*(ob+pb))): pair k occupies bits [k*(ob+pb), ...)
// of r, opcode = low ob bits, operand = next pb bits.  Machine (r, x) is
// c0(P_r, (x)) with ell = s = 1 and x in [0, 2^w) (init_config, m:289-309).
// A warp takes whole programs; its lanes take the program's inputs one after
// the other: a lane whose machine stopped (fixed point or budget) folds it
// into the record, claims the next input of the program and restores its own
// column of the tile to the program (the columns are independent machines),
// so no lane waits for the slowest input of a group.  Per program one record:
//   bit 63     all inputs reached a fixed point within tau_max
//   bits 0..62 sum over x of fmix32(x | halted << 8 | y0 << 9 | y1 << 10 | tau_h << 18)
// (a sum, so the order the lanes finish in cannot change it; y1 and tau_h
// count only when written / halted; the key fits 32 bits for w <= 8 and
// tau_max < 2^14).

struct EnumArgs {
    Geo g;
    uint64_t first;          // first program rank
    uint64_t count;          // programs
    uint64_t *records;       // [count]
    unsigned long long *steps_total;
    uint32_t m, ob, pb;      // pairs, opcode bits, operand bits
    uint32_t tau;            // step budget
};

__device__ __forceinline__ uint64_t mix64(uint64_t z)
{
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

// murmur3's 32-bit finaliser: the per-input fingerprint of the C4 records
__device__ __forceinline__ uint32_t fmix32(uint32_t h)
{
    h ^= h >> 16;
    h *= 0x85ebca6bu;
    h ^= h >> 13;
    h *= 0xc2b2ae35u;
    h ^= h >> 16;
    return h;
}

// resident 8-warp blocks per SM of the enumeration kernel (C4: 5 -> 0.896 s;
// 6 / 4 / 3 / 2 -> 0.941 / 0.991 / 0.989 / 1.000 s: unlike the epoch
// kernel's small tiles, this ALU-bound kernel wants its 40 warps)
#ifndef RASP_ENUM_MIN_BLOCKS
#define RASP_ENUM_MIN_BLOCKS 5
#endif
template <bool POW2, Arith AR, uint32_t UN>
__global__ void __launch_bounds__(256, RASP_ENUM_MIN_BLOCKS)
enum_kernel(const EnumArgs A)
{
    using SC = uint16_t;
    using CT = uint32_t;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ unsigned long long red_steps[8];
    constexpr uint32_t ROW = 32 * sizeof(SC);
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t wib = threadIdx.x >> 5;
    const Geo g = A.g;
    const uint32_t n = g.n;
    const uint32_t tile_bytes = (n + 3) * ROW;     // M, u[1] + pad, y[1]
    const uint32_t prog_bytes = (2 * n + 15) & ~15u;   // the program, machine-major
    char *tb = reinterpret_cast<char *>(smem_raw);
    const uint32_t s0 = static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw));
    const uint32_t nwb = blockDim.x >> 5;
    const uint32_t tile0 = s0 + wib * tile_bytes;
    const uint32_t prog0 = s0 + nwb * tile_bytes + wib * prog_bytes;
    const uint32_t lm = tile0 + lane * static_cast<uint32_t>(sizeof(SC));
    const uint32_t U = n * ROW + lm, Y = (n + 2) * ROW + lm;
    const uint32_t uend = U + ROW, yend = Y + ROW;
    const Opq q = {1u, 2u, ROW};
    const uint32_t pw = A.ob + A.pb;
    const uint32_t xs = static_cast<uint32_t>(g.mask) + 1;   // inputs per program (2^w)
    const uint32_t K = A.tau;
    const uint64_t nwarps = static_cast<uint64_t>(gridDim.x) * nwb;
    unsigned long long my_steps = 0;

    // programs go to warps in groups of 4 consecutive ranks, so a warp writes
    // its 4 records as one 32-byte sector (8-byte records from different warps
    // left partial sectors for L2 to merge: 14 GB of DRAM traffic for 2 GB of
    // records)
    uint64_t myrec = 0;   // lane k < 4: the record of program k of the current group
    for (uint64_t pi = (blockIdx.x * static_cast<uint64_t>(nwb) + wib) * 4; pi < A.count;
         pi += ((pi & 3) == 3) ? 4 * nwarps - 3 : 1) {
        const uint64_t r = A.first + pi;
        // the program, once per program, machine-major (lane c writes cell c)
        for (uint32_t c = lane; c < n; c += 32) {
            uint32_t cell = 0;
            if (c < 2 * A.m) {
                const uint32_t pair = static_cast<uint32_t>(r >> ((c >> 1) * pw)) & ((1u << pw) - 1u);
                cell = (c & 1) ? (pair >> A.ob) : (pair & ((1u << A.ob) - 1u));
            }
            st_cell<SC, CT, true>(tb, prog0 + 2 * c, cell);
        }
        __syncwarp();
        uint64_t v = 0;
        bool all_halted = true;
        uint32_t next = 32;      // next input to hand out (warp-uniform)
        uint32_t x = lane;       // this lane's input
        bool has = x < xs;
        LaneState<CT> L;
        L.tlast = 0;
        L.active = false;
        // (re)start the lane's machine on input x: its column = the program,
        // u[1] = x, empty output tape
        auto start = [&](bool go) {
            if (go) {
                uint32_t c = 0;
                for (; c + 8 <= n; c += 8) {   // 8 program cells per 16-byte broadcast read
                    uint4 v8;
                    check_smem(prog0 + 2 * c, 16);
                    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                                 : "=r"(v8.x), "=r"(v8.y), "=r"(v8.z), "=r"(v8.w) : "r"(prog0 + 2 * c));
                    const uint32_t w4[4] = {v8.x, v8.y, v8.z, v8.w};
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        st_cell<SC, CT, true>(tb, lm + (c + 2 * e) * ROW, w4[e] & 0xffffu);
                        st_cell<SC, CT, true>(tb, lm + (c + 2 * e + 1) * ROW, w4[e] >> 16);
                    }
                }
                for (; c < n; ++c)
                    st_cell<SC, CT, true>(tb, lm + c * ROW, ld_cell<SC, CT, true>(tb, prog0 + 2 * c));
                st_cell<SC, CT, true>(tb, U, x);
            } else {
                st_cell<SC, CT, true>(tb, lm, 0u);   // parked: opcode 0 at i = 0, a fixed point
            }
            L.i = 0; L.a = 0; L.ua = U; L.ya = Y; L.tlast = 0; L.rem = K;
            L.active = go;
        };
        start(has);
        for (;;) {
            // UN steps (machines start at check boundaries and tau_max % UN == 0,
            // so a live lane reaches its budget exactly at a check)
            if (K > 0) {
#pragma unroll
                for (uint32_t t = 0; t < UN; ++t) rasp_step_free<SC, CT, POW2, AR, true>(L, tb, lm, uend, yend, g, q);
            }
            // lanes whose machine stopped moving (fixed point) or used its budget
            const bool done = has && (!L.active || L.tlast == K);
            const unsigned dm = __ballot_sync(kFull, done);
            if (dm) {
                if (done) {
                    bool halted = L.tlast < K || !L.active;
                    if (L.tlast == K) {   // at the budget: the final probe (hv:140-148)
                        const Fetch<CT> f = fetch<SC, CT, POW2, AR, true>(L, tb, lm, g, q);
                        halted = is_fixed<CT, POW2, AR>(L, f, uend, yend, g, q);
                    }
                    const uint32_t y0 = (L.ya - Y) / ROW;
                    const uint32_t y1 = y0 ? static_cast<uint32_t>(ld_cell<SC, CT, true>(tb, Y)) : 0u;
                    const uint32_t key = x | (static_cast<uint32_t>(halted) << 8) | (y0 << 9) | (y1 << 10) |
                                         ((halted ? L.tlast : 0u) << 18);
                    v += fmix32(key);
                    all_halted &= halted;
                    my_steps += L.tlast;
                    x = next + __popc(dm & ((1u << lane) - 1u));
                    has = x < xs;
                    start(has);
                }
                next += __popc(dm);
            }
            if (!__any_sync(kFull, has)) break;
        }
        for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(kFull, v, off);
        const unsigned all = __all_sync(kFull, all_halted);
        if (lane == static_cast<uint32_t>(pi & 3))
            myrec = (static_cast<uint64_t>(all != 0) << 63) | (v & 0x7fffffffffffffffull);
        // a full group (or the batch's last program): lanes 0-3 write the
        // group's records, one sector
        if (((pi & 3) == 3 || pi + 1 == A.count) && lane <= static_cast<uint32_t>(pi & 3))
            A.records[(pi & ~uint64_t(3)) + lane] = myrec;
        __syncwarp();   // the next program rewrites the program area
    }
    // machine-steps: one atomic per block
    for (int off = 16; off; off >>= 1) my_steps += __shfl_down_sync(kFull, my_steps, off);
    if (lane == 0) red_steps[wib] = my_steps;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long st = 0;
        for (uint32_t w2 = 0; w2 < (blockDim.x >> 5); ++w2) st += red_steps[w2];
        if (st) atomicAdd(A.steps_total, st);
    }
}

// --- on-device c0 construction -----------------------------------
//
// init_c0_kernel: the device packer of init_config (m:289-309) for a batch:
//   M = P_j || 0^(n-L), u = (0, x_j || 0^(ell-k)), y = 0^(s+1), i = a = 0,
//   status = 0, steps = 0, tau_h = -1.  Programs [d][L] and inputs [d][k] in
//   the batch word type; ranges are checked by the host surface beforehand.
// generate_kernel: generator G_dev, the device twin of generator G (SURVEY
//   §8d): program fills memory, even cells opcode uniform in 1..7, odd cells
//   operand uniform in [0, n) (BNZ operands even), ell random input words.
//   Counter-based (splitmix64 of (seed, machine, cell)), so any shard of any
//   size is generated independently; not bit-identical to numpy's G.

template <class S>
__global__ void init_c0_kernel(Side b, uint64_t d, uint32_t n, uint32_t ell, uint32_t s,
                               const S *__restrict__ prog, uint32_t L, const S *__restrict__ inp,
                               uint32_t k)
{
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    S *M = static_cast<S *>(b.M), *u = static_cast<S *>(b.u), *y = static_cast<S *>(b.y);
    for (uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; t < d * n; t += stride) {
        const uint64_t j = t / n, c = t % n;
        M[t] = c < L ? prog[j * L + c] : S(0);
    }
    const uint64_t uc = static_cast<uint64_t>(ell) + 1, yc = static_cast<uint64_t>(s) + 1;
    for (uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; t < d * uc; t += stride) {
        const uint64_t j = t / uc, c = t % uc;
        u[t] = (c >= 1 && c <= k) ? inp[j * k + (c - 1)] : S(0);
    }
    for (uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; t < d * yc; t += stride)
        y[t] = S(0);
    for (uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; j < d; j += stride) {
        static_cast<S *>(b.iw)[j] = S(0);
        static_cast<S *>(b.ac)[j] = S(0);
        b.status[j] = kRunning;
        b.steps[j] = 0;
        b.tau_h[j] = -1;
    }
}

template <class S>
__global__ void generate_kernel(Side b, uint64_t d, uint64_t first, uint32_t n, uint32_t ell,
                                uint32_t s, uint64_t mask, uint64_t seed)
{
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    S *M = static_cast<S *>(b.M), *u = static_cast<S *>(b.u), *y = static_cast<S *>(b.y);
    const uint64_t key = mix64(seed ^ 0x5241535056495352ull);   // "RASPVISR"
    const uint32_t half = n / 2;
    for (uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; t < d * half; t += stride) {
        const uint64_t j = t / half, c = t % half;
        const uint64_t r = mix64(key ^ mix64(((first + j) << 20) ^ (c << 1)));
        const uint64_t op = 1 + (r & 0xffffffffull) % 7;
        uint64_t opr = (r >> 32) % n;
        if (op == 5) opr &= ~1ull;
        M[j * n + 2 * c] = static_cast<S>(op & mask);
        M[j * n + 2 * c + 1] = static_cast<S>(opr & mask);
    }
    if (n & 1)
        for (uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; j < d; j += stride)
            M[j * n + n - 1] = S(0);
    const uint64_t uc = static_cast<uint64_t>(ell) + 1, yc = static_cast<uint64_t>(s) + 1;
    for (uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; t < d * uc; t += stride) {
        const uint64_t j = t / uc, c = t % uc;
        u[t] = c == 0 ? S(0) : static_cast<S>(mix64(key ^ mix64(((first + j) << 20) ^ (c << 1) ^ 1)) & mask);
    }
    for (uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; t < d * yc; t += stride)
        y[t] = S(0);
    for (uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; j < d; j += stride) {
        static_cast<S *>(b.iw)[j] = S(0);
        static_cast<S *>(b.ac)[j] = S(0);
        b.status[j] = kRunning;
        b.steps[j] = 0;
        b.tau_h[j] = -1;
    }
}

// Bulk device copy on the SMs (keeps the copy engines free for host traffic).
static __global__ void copy_kernel(const uint4 *__restrict__ src, uint4 *__restrict__ dst, uint64_t n16,
                            const unsigned char *__restrict__ srcb, unsigned char *__restrict__ dstb,
                            uint64_t tail)
{
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; k < n16; k += stride)
        dst[k] = src[k];
    if (blockIdx.x == 0)
        for (uint64_t k = threadIdx.x; k < tail; k += blockDim.x) dstb[k] = srcb[k];
}

// 102-bucket halting histogram (hypervisor.py:326-352).
static __global__ void __launch_bounds__(1024) histogram_kernel(const int8_t *__restrict__ status,
                                                                const int64_t *__restrict__ tau_h, uint64_t d,
                                                                unsigned long long *__restrict__ out)
{
    // one private sub-histogram per warp (low smem-atomic contention), four
    // independent loads in flight per thread, then a block reduction and one
    // global atomic per non-empty bucket (grid = one block per SM)
    constexpr int B = 102, W = 32, U = 4;
    __shared__ unsigned int h[W][B + 2];
    const int wid = threadIdx.x >> 5;
    for (int k = threadIdx.x; k < W * (B + 2); k += blockDim.x) (&h[0][0])[k] = 0;
    __syncthreads();
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t j0 = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; j0 < d; j0 += U * stride) {
        int8_t st[U];
        int64_t th[U];
#pragma unroll
        for (int r = 0; r < U; ++r) {
            const uint64_t j = j0 + r * stride;
            st[r] = j < d ? status[j] : kRunning;
            th[r] = (j < d && st[r] == kHalted) ? tau_h[j] : 0;
        }
#pragma unroll
        for (int r = 0; r < U; ++r) {
            if (st[r] == kHalted) atomicAdd(&h[wid][th[r] < 100 ? static_cast<int>(th[r]) : 100], 1u);
            else if (st[r] == kExhausted) atomicAdd(&h[wid][101], 1u);
        }
    }
    __syncthreads();
    for (int k = threadIdx.x; k < B; k += blockDim.x) {
        unsigned int v = 0;
#pragma unroll 8
        for (int w = 0; w < W; ++w) v += h[w][k];
        if (v) atomicAdd(&out[k], static_cast<unsigned long long>(v));
    }
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
