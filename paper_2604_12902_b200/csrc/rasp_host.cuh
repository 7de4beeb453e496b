// rasp_host.cuh -- host-side launch machinery shared by the ABI translation
// units: device query, tile planning, workspace layout, the epoch scheduler
// (launch_epochs) and the template dispatch.  Instantiated per HBM word type
// in rasp_inst_s*.cu so the kernels compile in parallel.
#pragma once
#include "rasp_kernels.cuh"
#include "raspvisor_b200.h"

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>

namespace rasp {
namespace host {

extern thread_local char g_cuda_err[256];
extern std::atomic<unsigned long long> g_launches;

inline int cuda_fail(cudaError_t e, const char *what)
{
    std::snprintf(g_cuda_err, sizeof g_cuda_err, "%s: %s", what, cudaGetErrorString(e));
    return RASP_ECUDA;
}

#define RASP_CUDA(call)                                   \
    do {                                                  \
        cudaError_t e_ = (call);                          \
        if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
    } while (0)

using rasp::kMaxEpochs;                 // schedule slots in the workspace
constexpr int kPollAfter = 24;          // epochs after which the host polls the schedule
constexpr uint32_t kMaxK = 1u << 24;    // longest epoch, in steps

// Programmatic dependent launch between epochs ($RASP_PDL=0 turns it off; A/B aid)
inline bool pdl_enabled()
{
    static const bool on = [] {
        const char *e = std::getenv("RASP_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}

// Longest epoch actually used: kMaxK, or $RASP_KMAX (tests shorten it to drive
// long budgets through the host's polling path with small tau_max).
inline uint32_t max_epoch_len()
{
    static const uint32_t v = [] {
        const char *e = std::getenv("RASP_KMAX");
        const unsigned long x = e ? std::strtoul(e, nullptr, 10) : 0ul;
        return x >= 1 && x <= kMaxK ? uint32_t(x) : kMaxK;
    }();
    return v;
}
constexpr int kWarpsPerBlockMax = RASP_BLOCK_WARPS;
constexpr size_t kHistSmem = 512;       // block histogram (102 x u32) after the tiles, when requested
constexpr size_t kBigTile = 16 * 1024;  // tiles above this use the one-warp, many-register kernel
constexpr size_t kGlobalTileBudget = size_t(1) << 30;  // bytes of HBM tiles for huge n

struct Device {
    int id = -1, nsm = 0, smem_optin = 0;
};

inline int device_info(Device &dv)
{
    int id = 0;
    RASP_CUDA(cudaGetDevice(&id));
    static thread_local Device cache;
    if (cache.id != id) {
        Device d;
        d.id = id;
        RASP_CUDA(cudaDeviceGetAttribute(&d.nsm, cudaDevAttrMultiProcessorCount, id));
        RASP_CUDA(cudaDeviceGetAttribute(&d.smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, id));
        cache = d;
    }
    dv = cache;
    return RASP_OK;
}

// Launch shape of a kernel for one dynamic shared-memory size per unit
// (tile or slot group): units per block and resident blocks per SM, chosen to
// maximise resident units per SM.  Process-wide cache guarded by a mutex; the
// kernel's MaxDynamicSharedMemorySize attribute is raised once per (kernel,
// device) to the opt-in maximum and never lowered, so concurrent callers on
// other threads never see a limit below their launch (occupancy queries take
// each candidate size as an argument).
struct LaunchShape { int units = 0; int per_sm = 0; };

inline std::mutex &launch_mutex()
{
    static std::mutex mu;
    return mu;
}

// Raise a kernel's dynamic shared-memory limit to the device's opt-in maximum,
// once per (kernel, device); the caller holds launch_mutex().
inline int raise_smem_limit_locked(const void *kern, const Device &dv)
{
    static std::map<std::pair<const void *, int>, bool> raised;
    if (!raised[std::make_pair(kern, dv.id)]) {
        cudaFuncAttributes fa;
        RASP_CUDA(cudaFuncGetAttributes(&fa, kern));   // static shared memory counts against the opt-in limit
        RASP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       dv.smem_optin - int(fa.sharedSizeBytes)));
        raised[std::make_pair(kern, dv.id)] = true;
    }
    return RASP_OK;
}

inline int launch_shape(const void *kern, const Device &dv, size_t unit_bytes, size_t fixed_bytes, int max_units,
                        LaunchShape &out)
{
    static std::map<std::tuple<const void *, int, size_t, size_t, int>, LaunchShape> shapes;
    std::lock_guard<std::mutex> lock(launch_mutex());
    const auto key = std::make_tuple(kern, dv.id, unit_bytes, fixed_bytes, max_units);
    const auto it = shapes.find(key);
    if (it != shapes.end()) {
        out = it->second;
        return RASP_OK;
    }
    const int rc = raise_smem_limit_locked(kern, dv);
    if (rc) return rc;
    LaunchShape best;
    for (int u = max_units; u >= 1; --u) {
        const size_t smem = fixed_bytes + unit_bytes * size_t(u);
        if (smem > size_t(dv.smem_optin)) continue;
        int per_sm = 0;
        RASP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * u, smem));
        if (per_sm * u > best.per_sm * best.units) {
            best.units = u;
            best.per_sm = per_sm;
        }
    }
    if (best.units == 0) return RASP_ECAPACITY;
    shapes[key] = best;
    out = best;
    return RASP_OK;
}

// Checked builds: wait for the launches on `st` and report the first kernel
// check violation of this translation unit's kernels (g_check is per module).
inline int checked_result(cudaStream_t st)
{
#if RASP_CHECKED
    RASP_CUDA(cudaStreamSynchronize(st));
    unsigned long long c[4] = {0, 0, 0, 0};
    RASP_CUDA(cudaMemcpyFromSymbol(c, rasp::g_check, sizeof c));
    if (c[0]) {
        static const char *what[] = {"?", "shared access outside the dynamic window",
                                     "cell access outside the lane's column", "machine index beyond the batch",
                                     "output cursor beyond the tape", "list slot beyond the batch"};
        std::snprintf(g_cuda_err, sizeof g_cuda_err, "check failed: %s (%llu, %llu; block %llu thread %llu)",
                      what[c[0] < 6 ? c[0] : 0], c[1], c[2], c[3] >> 32, c[3] & 0xffffffffull);
        const unsigned long long z[4] = {0, 0, 0, 0};
        RASP_CUDA(cudaMemcpyToSymbol(rasp::g_check, z, sizeof z));
        return RASP_ECHECK;
    }
#else
    (void)st;
#endif
    return RASP_OK;
}

inline size_t natural_bytes(uint32_t w) { return w <= 8 ? 1 : w <= 16 ? 2 : w <= 32 ? 4 : 8; }
inline size_t cell_bytes(uint32_t w) { return w <= 16 ? 2 : w <= 32 ? 4 : 8; }   // tile cell SC
inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

inline int check_params(const rasp_params *p)
{
    if (!p || p->w < 1 || p->w > 64 || p->n < 2) return RASP_EPARAM;
    if (p->n >= (1u << 31)) return RASP_ECAPACITY;   // the kernels' x mod n needs n < 2^31
    const uint64_t limit_m1 = p->w == 64 ? ~0ull : ((1ull << p->w) - 1);
    if (p->ell < 1 || p->s < 1 || p->ell > limit_m1 || p->s > limit_m1) return RASP_EPARAM;
    if (p->ell >= (1ull << 31) || p->s >= (1ull << 31)) return RASP_ECAPACITY;
    return RASP_OK;
}

struct Plan {
    bool smem = true;
    bool big = false;         // one-warp blocks, y not staged in the tile
    uint32_t tile_rows = 0;
    int warps_per_block = 1;
    int blocks = 1;
    size_t tile_bytes = 0;
    size_t dyn_smem = 0;
    size_t gtile_bytes = 0;   // workspace bytes for HBM tiles (huge n only)
};

inline uint64_t tile_rows(const rasp_params *p) { return uint64_t(p->n) + p->ell + 1 + p->s; }

// Sizing that does not need the kernel handle (workspace size).
inline void plan_shape(const rasp_params *p, const Device &dv, Plan &pl)
{
    pl.tile_rows = uint32_t(tile_rows(p));
    pl.tile_bytes = uint64_t(pl.tile_rows) * 32 * cell_bytes(p->w);
    pl.big = cell_bytes(p->w) >= 4 && pl.tile_bytes > kBigTile;
    if (pl.big) {   // PRI writes go to HBM directly: no output rows in the tile
        pl.tile_rows = uint32_t(uint64_t(p->n) + p->ell + 1);
        pl.tile_bytes = uint64_t(pl.tile_rows) * 32 * cell_bytes(p->w);
    }
    if (pl.tile_bytes <= size_t(dv.smem_optin)) {
        pl.smem = true;
        pl.warps_per_block = int(std::min<size_t>(kWarpsPerBlockMax, dv.smem_optin / pl.tile_bytes));
        pl.dyn_smem = pl.tile_bytes * pl.warps_per_block;
        pl.gtile_bytes = 0;
    } else {
        pl.smem = false;
        pl.big = false;
        pl.tile_rows = uint32_t(tile_rows(p));
        pl.tile_bytes = uint64_t(pl.tile_rows) * 32 * cell_bytes(p->w);
        pl.warps_per_block = 1;
        pl.dyn_smem = 0;
        const size_t warps = std::max<size_t>(
            dv.nsm, std::min<size_t>(size_t(dv.nsm) * 16, kGlobalTileBudget / pl.tile_bytes));
        pl.blocks = int(warps);
        pl.gtile_bytes = warps * pl.tile_bytes;
    }
}

struct Workspace {
    uint32_t *lists[2];
    rasp::Sched *sched;
    void *gtiles;
};

inline size_t workspace_layout(const rasp_params *p, uint64_t d, const Plan &pl, void *base, Workspace *ws)
{
    size_t off = 0;
    char *b = static_cast<char *>(base);
    const size_t list_bytes = align256(sizeof(uint32_t) * std::max<uint64_t>(d, 1));
    if (ws) ws->lists[0] = reinterpret_cast<uint32_t *>(b + off);
    off += list_bytes;
    if (ws) ws->lists[1] = reinterpret_cast<uint32_t *>(b + off);
    off += list_bytes;
    if (ws) ws->sched = reinterpret_cast<rasp::Sched *>(b + off);
    off += align256(sizeof(rasp::Sched));
    if (ws) ws->gtiles = pl.gtile_bytes ? b + off : nullptr;
    off += align256(pl.gtile_bytes);
    (void)p;
    return off;
}

template <class SC, rasp::Arith AR, bool BUDGET, bool SMEM, bool BIG>
constexpr bool kRefillOk = sizeof(SC) >= 4 && AR != rasp::Arith::W1 && AR != rasp::Arith::CELL && !BUDGET && SMEM && BIG;

// The refill kernel as the first epoch (big tiles, fresh runs): its launch
// shape and parameters.  Instantiated only where it applies.
template <class S, class SC, class CT, bool POW2, rasp::Arith AR>
int launch_refill_epoch(const rasp::EpochArgs &a, const Plan &pl, const Device &dv, uint64_t d, cudaStream_t st)
{
    auto kern = rasp::refill_kernel<S, SC, CT, POW2, AR>;
    LaunchShape sh;
    const size_t extra = rasp::kRefillExtra<SC>;   // histogram + parking cells
    const int rc = launch_shape(reinterpret_cast<const void *>(kern), dv, pl.tile_bytes, extra, 1, sh);
    if (rc) return rc;
    const uint64_t warps = uint64_t(sh.per_sm) * dv.nsm;
    const int grid = int(std::max<uint64_t>(1, std::min<uint64_t>(warps, (d + 31) / 32)));
    if (std::getenv("RASP_DEBUG"))
        std::fprintf(stderr, "rasp: refill epoch K0 %u, tile %zu B (%u rows), %d blocks/SM, grid %d\n", a.K0,
                     pl.tile_bytes, pl.tile_rows, sh.per_sm, grid);
    kern<<<grid, 32, pl.tile_bytes + extra, st>>>(a);
    RASP_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return RASP_OK;
}

template <class S, class SC, class CT, bool POW2, rasp::Arith AR, bool BUDGET, bool SMEM, bool BIG = false>
int launch_epochs(const rasp::EpochArgs &base, Plan pl, const Device &dv, const Workspace &ws,
                  uint64_t d, int64_t tau_max, int64_t epoch, cudaStream_t st, bool refill0 = false)
{
    auto kern = rasp::epoch_kernel<S, SC, CT, POW2, AR, BUDGET, SMEM, BIG>;
    if (SMEM) {
        // warps per block chosen to maximise resident warps per SM (ties: more
        // warps per block)
        LaunchShape sh;
        const size_t hist_bytes = base.hist ? kHistSmem : 0;
        const int rc = launch_shape(reinterpret_cast<const void *>(kern), dv, pl.tile_bytes, hist_bytes,
                                    BIG ? 1 : kWarpsPerBlockMax, sh);
        if (rc) return rc;
        pl.warps_per_block = sh.units;
        pl.dyn_smem = pl.tile_bytes * size_t(sh.units) + hist_bytes;
        pl.blocks = sh.per_sm * dv.nsm;
        if (std::getenv("RASP_DEBUG"))   // plan of this launch sequence (tuning aid)
            std::fprintf(stderr, "rasp: tile %zu B (%u rows), %d warps/block, %d blocks/SM, big %d\n",
                         pl.tile_bytes, pl.tile_rows, sh.units, sh.per_sm, int(BIG));
    }
    else if (base.hist) pl.dyn_smem = kHistSmem;   // HBM tiles: only the histogram is in shared memory
    const int threads = 32 * pl.warps_per_block;
    const uint64_t tiles = (d + 31) / 32;
    const uint64_t need_blocks = (tiles + pl.warps_per_block - 1) / pl.warps_per_block;
    const int grid = int(std::max<uint64_t>(1, std::min<uint64_t>(uint64_t(pl.blocks), need_blocks)));

    RASP_CUDA(cudaMemsetAsync(ws.sched, 0, sizeof(rasp::Sched), st));
    // Enough launches for the pure doubling schedule; the device schedule can
    // only finish sooner (it lengthens epochs once survivors stop halting).
    const uint64_t K0 = std::min<uint64_t>(uint64_t(std::min<int64_t>(std::max<int64_t>(epoch, 1), tau_max)),
                                           max_epoch_len());
    int planned = 1;
    bool covers = int64_t(K0) >= tau_max;
    {
        uint64_t cov = K0, k = std::max<uint64_t>(K0, 1);
        while (int64_t(cov) < tau_max && planned < kPollAfter) {
            k = std::min<uint64_t>(k * 2, max_epoch_len());
            cov += k;
            ++planned;
        }
        covers = int64_t(cov) >= tau_max;
    }
    // PDL only for eager launches: graph replays already launch the epochs
    // back to back (measured: eager C2 -1.5%, graph replays C2 +0.0%, C3 +0.2%)
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    bool pdl = false;
    if (pdl_enabled()) {
        if (cudaStreamIsCapturing(st, &cap) == cudaSuccess) pdl = cap == cudaStreamCaptureStatusNone;
        else (void)cudaGetLastError();   // e.g. legacy stream during a global capture
    }
    for (int e = 0;; ++e) {
        if (e >= kMaxEpochs) {
            // the schedule slots are used up: fine if the last epoch left no
            // survivors (its K[e+1] is never written), a capacity error if not
            uint32_t left = 0;
            RASP_CUDA(cudaMemcpyAsync(&left, &ws.sched->count[kMaxEpochs - 1], sizeof left, cudaMemcpyDeviceToHost, st));
            RASP_CUDA(cudaStreamSynchronize(st));
            if (left == 0) break;
            return RASP_ECAPACITY;
        }
        if (e >= planned && covers) break;   // fully asynchronous in the common case
        if (e >= planned) {
            // long budgets: ask the device whether another epoch is needed
            uint32_t knext = 0;
            RASP_CUDA(cudaMemcpyAsync(&knext, &ws.sched->K[e], sizeof knext, cudaMemcpyDeviceToHost, st));
            RASP_CUDA(cudaStreamSynchronize(st));
            if (knext == 0) break;
        }
        rasp::EpochArgs a = base;
        a.sched = ws.sched;
        a.e = uint32_t(e);
        a.first = e == 0;
        a.count_in = uint32_t(d);
        a.K0 = uint32_t(K0);
        a.kmax = max_epoch_len();
        a.list_in = e == 0 ? nullptr : ws.lists[(e - 1) & 1];
        a.list_out = ws.lists[e & 1];
        // epochs after the first chain on the previous epoch launch with
        // programmatic dependent launch (the kernel waits on it first thing),
        // so the launch overlaps the previous epoch's tail; not after a host
        // poll (the previous stream op is then a copy)
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        if (e == 0 && refill0) {
            if constexpr (kRefillOk<SC, AR, BUDGET, SMEM, BIG>) {
                a.refill_min = 12;   // C5: 8/12/16 -> 1.655/1.601/1.634 ms (tuning knob RASP_REFILL_MIN)
                if (const char *v = std::getenv("RASP_REFILL_MIN"))
                    a.refill_min = std::min<uint32_t>(32, std::max<uint32_t>(1, uint32_t(std::strtoul(v, nullptr, 10))));
                // L2 warm-up of the 16 machines the next refills take, issued at
                // each refill: C5 1.601 -> 1.585 ms (12/24/32: 1.588/1.599/1.622;
                // =1: whole reservations when claimed, 1.624; =0: off)
                a.pf_dist = 16;
                if (const char *v = std::getenv("RASP_REFILL_PREFETCH")) a.pf_dist = uint32_t(std::strtoul(v, nullptr, 10));
                const int rc = launch_refill_epoch<S, SC, CT, POW2, AR>(a, pl, dv, d, st);
                if (rc) return rc;
                continue;
            }
        }
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(unsigned(grid));
        cfg.blockDim = dim3(unsigned(threads));
        cfg.dynamicSmemBytes = pl.dyn_smem;
        cfg.stream = st;
        cfg.attrs = attr;
        cfg.numAttrs = (pdl && e > 0 && e < planned) ? 1 : 0;
        RASP_CUDA(cudaLaunchKernelEx(&cfg, kern, a, static_cast<SC *>(ws.gtiles)));
        RASP_CUDA(cudaGetLastError());
        g_launches.fetch_add(1, std::memory_order_relaxed);
    }
    return checked_result(st);
}

// Per-lane refill for big tiles (refill_kernel) as the first epoch of fresh
// runs.  Measured (first-epoch length K0 swept on both paths,
// scripts/sweep_k0.sh): C5 (tau 1024) 1.84 ms at its best epochs against 1.61
// with K0 = tau and 1.70-1.78 with K0 = 512/320 plus epochs; the paper row
// (tau 10^4) 2.60 on epochs against 2.91-3.29 refilled (K0 32..512); paper6
// (tau 10^6) within 0.3%.  So by default the refill kernel runs only when it
// can take the whole budget in one launch: tau a multiple of the block and at
// most kRefillMaxTau, and the machine rows 16-byte aligned.  $RASP_REFILL=0 keeps the epochs; =1 runs the refill
// kernel as the first epoch of any fresh big-tile run, K0 = the first-epoch
// length rounded up to the block (survivors continue on the epoch kernel).
// Read per run: tests compare the paths in one process.
constexpr int64_t kRefillMaxTau = 2048;
inline int refill_mode()
{
    const char *e = std::getenv("RASP_REFILL");
    if (e && e[0] == '0') return 0;
    if (e && e[0] == '1') return 1;
    return 2;   // auto
}

template <class S, class SC, class CT, bool POW2, rasp::Arith AR>
int dispatch_budget(const rasp::EpochArgs &a, const Plan &pl, const Device &dv, const Workspace &ws,
                    uint64_t d, int64_t tau_max, int64_t epoch, cudaStream_t st)
{
    if constexpr (kRefillOk<SC, AR, false, true, true>) {
        // the refill kernel runs the first epoch: K0 = the first-epoch length
        // rounded up to the unrolled block, or the whole budget when that
        // covers it and is a multiple of the block (else a block less)
        constexpr int64_t UN = RASP_UNROLL_BIG;
        const int mode = refill_mode();
        int64_t k0 = 0;
        // auto: machine rows on 16-byte boundaries only (the paper rows' n = 250
        // 32-bit words are not: refilled, 0.92-1.09 ms against 0.90-0.99 on
        // epochs at tau 256-1024, and 1.24-1.49 with the aligned-only loader
        // the refill kernel keeps -- scripts/refill_policy.py)
        const bool rows16 = (reinterpret_cast<uintptr_t>(a.in.M) % 16 == 0) &&
                            (uint64_t(a.g.n) * sizeof(S)) % 16 == 0;
        if (mode == 2 && rows16 && tau_max % UN == 0 && tau_max <= kRefillMaxTau) k0 = tau_max;
        if (mode == 1) {
            k0 = (std::max<int64_t>(epoch, 1) + UN - 1) / UN * UN;
            if (k0 >= tau_max) k0 = tau_max / UN * UN;
        }
        if (pl.big && a.fresh && k0 >= UN && k0 <= int64_t(max_epoch_len()) && k0 < (int64_t(1) << 31) &&
            d < (uint64_t(1) << 31))
            return launch_epochs<S, SC, CT, POW2, AR, false, true, true>(a, pl, dv, ws, d, tau_max, k0, st, true);
    }
    if (sizeof(SC) >= 4 && pl.big) {
        if (a.fresh) return launch_epochs<S, SC, CT, POW2, AR, false, true, true>(a, pl, dv, ws, d, tau_max, epoch, st);
        return launch_epochs<S, SC, CT, POW2, AR, true, true, true>(a, pl, dv, ws, d, tau_max, epoch, st);
    }
    if (a.fresh) return launch_epochs<S, SC, CT, POW2, AR, false, true>(a, pl, dv, ws, d, tau_max, epoch, st);
    return launch_epochs<S, SC, CT, POW2, AR, true, true>(a, pl, dv, ws, d, tau_max, epoch, st);
}

// S: HBM word type, SC: tile cell type, CT: arithmetic type.
template <class S, class SC, class CT>
int dispatch_flags(const rasp_params *p, const rasp::EpochArgs &a, const Plan &pl, const Device &dv,
                   const Workspace &ws, uint64_t d, int64_t tau_max, int64_t epoch, cudaStream_t st)
{
    using rasp::Arith;
    if (!pl.smem)   // huge n: tiles in HBM, generic arithmetic
        return launch_epochs<S, SC, CT, false, Arith::W1, true, false>(a, pl, dv, ws, d, tau_max, epoch, st);
    const bool pow2 = (p->n & (p->n - 1)) == 0;
    if constexpr (sizeof(SC) == 2) {
        if (p->w == 1) {
            if (pow2) return dispatch_budget<S, SC, CT, true, Arith::W1>(a, pl, dv, ws, d, tau_max, epoch, st);
            return dispatch_budget<S, SC, CT, false, Arith::W1>(a, pl, dv, ws, d, tau_max, epoch, st);
        }
        if (p->w == 16) {
            if (pow2) return dispatch_budget<S, SC, CT, true, Arith::CELL>(a, pl, dv, ws, d, tau_max, epoch, st);
            return dispatch_budget<S, SC, CT, false, Arith::CELL>(a, pl, dv, ws, d, tau_max, epoch, st);
        }
    } else {
        if (p->w == 8 * sizeof(CT)) {
            if (pow2) return dispatch_budget<S, SC, CT, true, Arith::FULL>(a, pl, dv, ws, d, tau_max, epoch, st);
            return dispatch_budget<S, SC, CT, false, Arith::FULL>(a, pl, dv, ws, d, tau_max, epoch, st);
        }
    }
    if (pow2) return dispatch_budget<S, SC, CT, true, Arith::NARROW>(a, pl, dv, ws, d, tau_max, epoch, st);
    return dispatch_budget<S, SC, CT, false, Arith::NARROW>(a, pl, dv, ws, d, tau_max, epoch, st);
}

// Device-to-device copy with a kernel (cudaMemcpyAsync D2D would occupy a copy
// engine that host<->device pipelines need).
inline int dev_copy(void *dst, const void *src, size_t bytes, const Device &dv, cudaStream_t st)
{
    if (bytes == 0) return RASP_OK;
    const uintptr_t a = reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src);
    const size_t n16 = (a & 15) ? 0 : bytes / 16;
    const size_t head = n16 * 16;
    const unsigned blocks = unsigned(std::max<size_t>(1, std::min<size_t>((n16 + 255) / 256, size_t(dv.nsm) * 8)));
    rasp::copy_kernel<<<blocks, 256, 0, st>>>(static_cast<const uint4 *>(src), static_cast<uint4 *>(dst), n16,
                                              static_cast<const unsigned char *>(src) + head,
                                              static_cast<unsigned char *>(dst) + head, bytes - head);
    RASP_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return RASP_OK;
}

inline rasp::Side side_of(const rasp_batch *b)
{
    rasp::Side s;
    s.iw = b->iw; s.ac = b->ac; s.M = b->M; s.u = b->u; s.y = b->y;
    s.status = b->status; s.steps = b->steps; s.tau_h = b->tau_h;
    return s;
}


// Run dispatch for one HBM word type (definitions in rasp_inst_s<bytes>.cu).
template <class S>
int run_typed(const rasp_params *p, const EpochArgs &a, const Plan &pl, const Device &dv,
              const Workspace &ws, uint64_t d, int64_t tau_max, int64_t epoch, cudaStream_t st);
#define RASP_DECL_RUN(S)                                                                         \
    template <>                                                                                  \
    int run_typed<S>(const rasp_params *p, const EpochArgs &a, const Plan &pl, const Device &dv, \
                     const Workspace &ws, uint64_t d, int64_t tau_max, int64_t epoch, cudaStream_t st);
RASP_DECL_RUN(uint8_t)
RASP_DECL_RUN(uint16_t)
RASP_DECL_RUN(uint32_t)
RASP_DECL_RUN(uint64_t)
#undef RASP_DECL_RUN

}  // namespace host
}  // namespace rasp
