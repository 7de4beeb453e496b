// rasp_abi.cu -- extern "C" boundary of the B200 word-RASP engine
// (declared in include/raspvisor_b200.h).  Host-side epoch scheduling,
// template dispatch and launch configuration; the kernels are in
// rasp_kernels.cuh.
#include "rasp_kernels.cuh"
#include "raspvisor_b200.h"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include <atomic>

namespace {

thread_local char g_cuda_err[256] = "";
std::atomic<unsigned long long> g_launches{0};

int cuda_fail(cudaError_t e, const char *what)
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
constexpr int kWarpsPerBlockMax = 4;
constexpr size_t kGlobalTileBudget = size_t(1) << 30;  // bytes of HBM tiles for huge n

struct Device {
    int id = -1, nsm = 0, smem_optin = 0;
};

int device_info(Device &dv)
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

size_t natural_bytes(uint32_t w) { return w <= 8 ? 1 : w <= 16 ? 2 : w <= 32 ? 4 : 8; }
size_t cell_bytes(uint32_t w) { return w <= 16 ? 2 : w <= 32 ? 4 : 8; }   // tile cell SC
size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

int check_params(const rasp_params *p)
{
    if (!p || p->w < 1 || p->w > 64 || p->n < 2) return RASP_EPARAM;
    const uint64_t limit_m1 = p->w == 64 ? ~0ull : ((1ull << p->w) - 1);
    if (p->ell < 1 || p->s < 1 || p->ell > limit_m1 || p->s > limit_m1) return RASP_EPARAM;
    if (p->ell >= (1ull << 31) || p->s >= (1ull << 31)) return RASP_ECAPACITY;
    return RASP_OK;
}

struct Plan {
    bool smem = true;
    int warps_per_block = 1;
    int blocks = 1;
    size_t tile_bytes = 0;
    size_t dyn_smem = 0;
    size_t gtile_bytes = 0;   // workspace bytes for HBM tiles (huge n only)
};

uint64_t tile_rows(const rasp_params *p) { return uint64_t(p->n) + p->ell + 1 + p->s; }

// Sizing that does not need the kernel handle (workspace size).
void plan_shape(const rasp_params *p, const Device &dv, Plan &pl)
{
    pl.tile_bytes = tile_rows(p) * 32 * cell_bytes(p->w);
    if (pl.tile_bytes <= size_t(dv.smem_optin)) {
        pl.smem = true;
        pl.warps_per_block = int(std::min<size_t>(kWarpsPerBlockMax, dv.smem_optin / pl.tile_bytes));
        pl.dyn_smem = pl.tile_bytes * pl.warps_per_block;
        pl.gtile_bytes = 0;
    } else {
        pl.smem = false;
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

size_t workspace_layout(const rasp_params *p, uint64_t d, const Plan &pl, void *base, Workspace *ws)
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

template <class S, class SC, class CT, bool POW2, rasp::Arith AR, bool BUDGET, bool SMEM>
int launch_epochs(const rasp::EpochArgs &base, Plan pl, const Device &dv, const Workspace &ws,
                  uint64_t d, int64_t tau_max, int64_t epoch, cudaStream_t st)
{
    auto kern = rasp::epoch_kernel<S, SC, CT, POW2, AR, BUDGET, SMEM>;
    if (SMEM) {
        // warps per block chosen to maximise resident warps per SM (ties: more
        // warps per block); attribute + occupancy queried once per
        // (instantiation, device, tile size)
        struct Cached { int dev = -1; size_t tile = 0; int wpb = 0; int per_sm = 0; };
        static thread_local Cached c;
        if (c.dev != dv.id || c.tile != pl.tile_bytes) {
            int best_w = 0, best_ps = 0;
            for (int wpb = kWarpsPerBlockMax; wpb >= 1; --wpb) {
                const size_t smem = pl.tile_bytes * size_t(wpb);
                if (smem > size_t(dv.smem_optin)) continue;
                RASP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
                int per_sm = 0;
                RASP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * wpb, smem));
                if (per_sm * wpb > best_ps * best_w) {
                    best_w = wpb;
                    best_ps = per_sm;
                }
            }
            if (best_w == 0) return RASP_ECAPACITY;
            RASP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           int(pl.tile_bytes * size_t(best_w))));
            c.dev = dv.id;
            c.tile = pl.tile_bytes;
            c.wpb = best_w;
            c.per_sm = best_ps;
        }
        pl.warps_per_block = c.wpb;
        pl.dyn_smem = pl.tile_bytes * size_t(c.wpb);
        pl.blocks = c.per_sm * dv.nsm;
    }
    const int threads = 32 * pl.warps_per_block;
    const uint64_t tiles = (d + 31) / 32;
    const uint64_t need_blocks = (tiles + pl.warps_per_block - 1) / pl.warps_per_block;
    const int grid = int(std::max<uint64_t>(1, std::min<uint64_t>(uint64_t(pl.blocks), need_blocks)));

    RASP_CUDA(cudaMemsetAsync(ws.sched, 0, sizeof(rasp::Sched), st));
    // Enough launches for the pure doubling schedule; the device schedule can
    // only finish sooner (it lengthens epochs once survivors stop halting).
    const uint64_t K0 = uint64_t(std::min<int64_t>(std::max<int64_t>(epoch, 1), tau_max));
    int planned = 1;
    bool covers = int64_t(K0) >= tau_max;
    {
        uint64_t cov = K0, k = std::max<uint64_t>(K0, 1);
        while (int64_t(cov) < tau_max && planned < kPollAfter) {
            k = std::min<uint64_t>(k * 2, kMaxK);
            cov += k;
            ++planned;
        }
        covers = int64_t(cov) >= tau_max;
    }
    for (int e = 0;; ++e) {
        if (e >= kMaxEpochs) return RASP_ECAPACITY;
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
        a.kmax = kMaxK;
        a.list_in = e == 0 ? nullptr : ws.lists[(e - 1) & 1];
        a.list_out = ws.lists[e & 1];
        kern<<<grid, threads, pl.dyn_smem, st>>>(a, static_cast<SC *>(ws.gtiles));
        RASP_CUDA(cudaGetLastError());
        g_launches.fetch_add(1, std::memory_order_relaxed);
    }
    return RASP_OK;
}

template <class S, class SC, class CT, bool POW2, rasp::Arith AR>
int dispatch_budget(const rasp::EpochArgs &a, const Plan &pl, const Device &dv, const Workspace &ws,
                    uint64_t d, int64_t tau_max, int64_t epoch, cudaStream_t st)
{
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
int dev_copy(void *dst, const void *src, size_t bytes, const Device &dv, cudaStream_t st)
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

rasp::Side side_of(const rasp_batch *b)
{
    rasp::Side s;
    s.iw = b->iw; s.ac = b->ac; s.M = b->M; s.u = b->u; s.y = b->y;
    s.status = b->status; s.steps = b->steps; s.tau_h = b->tau_h;
    return s;
}

}  // namespace

extern "C" {

int rasp_abi_version(void) { return RASP_ABI_VERSION; }

unsigned long long rasp_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

const char *rasp_error_string(int code)
{
    switch (code) {
    case RASP_OK: return "ok";
    case RASP_EPARAM: return "invalid machine parameters";
    case RASP_ECAPACITY: return "batch or geometry exceeds engine capacity";
    case RASP_ECUDA: return "CUDA error";
    case RASP_EWORKSPACE: return "workspace too small";
    case RASP_EDTYPE: return "word_bytes must be 1, 2, 4 or 8 and hold w bits";
    default: return "unknown error";
    }
}

const char *rasp_last_cuda_error(void) { return g_cuda_err; }

size_t rasp_workspace_bytes(const rasp_params *p, uint64_t d)
{
    if (check_params(p) != RASP_OK) return 0;
    Device dv;
    if (device_info(dv) != RASP_OK) return 0;
    Plan pl;
    plan_shape(p, dv, pl);
    return workspace_layout(p, d, pl, nullptr, nullptr);
}

int rasp_run(const rasp_params *p, const rasp_batch *in, const rasp_batch *out, int64_t tau_max,
             int64_t epoch, uint32_t flags, void *workspace, size_t workspace_bytes, void *stream)
{
    int rc = check_params(p);
    if (rc) return rc;
    if (!in || !out || tau_max < 0 || epoch < 1) return RASP_EPARAM;
    if (in->d != out->d) return RASP_EPARAM;
    const uint64_t d = in->d;
    if (d == 0) return RASP_OK;
    if (d > 0xffffffe0ull) return RASP_ECAPACITY;
    const uint32_t wb = in->word_bytes;
    if (wb != out->word_bytes || (wb != 1 && wb != 2 && wb != 4 && wb != 8) || wb < natural_bytes(p->w))
        return RASP_EDTYPE;
    Device dv;
    rc = device_info(dv);
    if (rc) return rc;
    Plan pl;
    plan_shape(p, dv, pl);
    const size_t need = workspace_layout(p, d, pl, nullptr, nullptr);
    if (!workspace || workspace_bytes < need) return RASP_EWORKSPACE;
    Workspace ws;
    workspace_layout(p, d, pl, workspace, &ws);

    rasp::EpochArgs a;
    std::memset(&a, 0, sizeof a);
    a.g.mask = p->w == 64 ? ~0ull : ((1ull << p->w) - 1);
    a.g.n = p->n;
    a.g.nm1 = p->n - 1;
    a.g.jm = uint32_t(a.g.mask & uint64_t(p->n - 1));
    a.g.fm = ~0ull / p->n + 1;
    a.g.ell = uint32_t(p->ell);
    a.g.s = uint32_t(p->s);
    a.in = side_of(in);
    a.out = side_of(out);
    a.tau_max = tau_max;
    a.fresh = (flags & RASP_FRESH) ? 1 : 0;
    a.inplace = (in->iw == out->iw) ? 1 : 0;
    a.tile_rows = uint32_t(tile_rows(p));
    a.one = 1;
    a.two = 2;
    a.row = uint32_t(32 * cell_bytes(p->w));
    a.stable_q8 = 128;                       // 0.5 (measured best on C2 and C5): tuning knob RASP_STABLE_Q8
    if (const char *e = std::getenv("RASP_STABLE_Q8")) a.stable_q8 = uint32_t(std::strtoul(e, nullptr, 10));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (!a.inplace) {
        // out-of-place: the input tapes and the bookkeeping arrays move in bulk;
        // the kernels then treat `out` as the working copy
        const size_t ub = size_t(d) * (p->ell + 1) * wb, yb = size_t(d) * (p->s + 1) * wb;
        int rc2 = dev_copy(out->u, in->u, ub, dv, st);
        if (!rc2) rc2 = dev_copy(out->y, in->y, yb, dv, st);
        if (!rc2 && !a.fresh) {
            rc2 = dev_copy(out->status, in->status, size_t(d), dv, st);
            if (!rc2) rc2 = dev_copy(out->steps, in->steps, size_t(d) * 8, dv, st);
            if (!rc2) rc2 = dev_copy(out->tau_h, in->tau_h, size_t(d) * 8, dv, st);
        }
        if (rc2) return rc2;
    }
    if (p->w <= 16) {
        switch (wb) {
        case 1: return dispatch_flags<uint8_t, uint16_t, uint32_t>(p, a, pl, dv, ws, d, tau_max, epoch, st);
        case 2: return dispatch_flags<uint16_t, uint16_t, uint32_t>(p, a, pl, dv, ws, d, tau_max, epoch, st);
        case 4: return dispatch_flags<uint32_t, uint16_t, uint32_t>(p, a, pl, dv, ws, d, tau_max, epoch, st);
        default: return dispatch_flags<uint64_t, uint16_t, uint32_t>(p, a, pl, dv, ws, d, tau_max, epoch, st);
        }
    }
    if (p->w <= 32) {
        if (wb == 4) return dispatch_flags<uint32_t, uint32_t, uint32_t>(p, a, pl, dv, ws, d, tau_max, epoch, st);
        return dispatch_flags<uint64_t, uint32_t, uint32_t>(p, a, pl, dv, ws, d, tau_max, epoch, st);
    }
    return dispatch_flags<uint64_t, uint64_t, uint64_t>(p, a, pl, dv, ws, d, tau_max, epoch, st);
}

int rasp_enumerate(const rasp_enum_params *ep, uint64_t first_rank, uint64_t count, uint64_t *records,
                   unsigned long long *steps_total, void *stream)
{
    if (!ep || !records || !steps_total) return RASP_EPARAM;
    if (ep->w < 2 || ep->w > 8 || ep->n < 2 || ep->n > 4096 || ep->m < 1 || ep->opcode_bits < 1 ||
        ep->operand_bits < 1 || ep->opcode_bits > ep->w || ep->operand_bits > ep->w ||
        uint64_t(ep->m) * (ep->opcode_bits + ep->operand_bits) > 63)
        return RASP_EPARAM;
    if (2 * ep->m > ep->n) return RASP_ECAPACITY;
    if (count == 0) return RASP_OK;
    Device dv;
    int rc = device_info(dv);
    if (rc) return rc;
    rasp::EnumArgs a;
    std::memset(&a, 0, sizeof a);
    a.g.mask = (1ull << ep->w) - 1;
    a.g.n = ep->n;
    a.g.nm1 = ep->n - 1;
    a.g.jm = uint32_t(a.g.mask & uint64_t(ep->n - 1));
    a.g.fm = ~0ull / ep->n + 1;
    a.g.ell = 1;
    a.g.s = 1;
    a.first = first_rank;
    a.count = count;
    a.records = records;
    a.steps_total = steps_total;
    a.m = ep->m;
    a.ob = ep->opcode_bits;
    a.pb = ep->operand_bits;
    a.tau = ep->tau_max;
    a.one = 1;
    a.two = 2;
    a.row = 64;
    const size_t smem = size_t(8) * (ep->n + 3) * 64;
    const bool pow2 = (ep->n & (ep->n - 1)) == 0;
    auto kern = pow2 ? rasp::enum_kernel<true, rasp::Arith::NARROW> : rasp::enum_kernel<false, rasp::Arith::NARROW>;
    RASP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    int per_sm = 0;
    RASP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, smem));
    if (per_sm < 1) return RASP_ECAPACITY;
    const uint64_t grid = std::min<uint64_t>(count, uint64_t(per_sm) * dv.nsm * 8);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    kern<<<unsigned(grid), 256, smem, st>>>(a);
    RASP_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return RASP_OK;
}

int rasp_init_c0(const rasp_params *p, const void *programs, uint32_t prog_len, const void *inputs,
                 uint32_t input_len, const rasp_batch *out, void *stream)
{
    int rc = check_params(p);
    if (rc) return rc;
    if (!out || (prog_len && !programs) || (input_len && !inputs)) return RASP_EPARAM;
    if (prog_len > p->n || input_len > p->ell) return RASP_ECAPACITY;
    const uint32_t wb = out->word_bytes;
    if ((wb != 1 && wb != 2 && wb != 4 && wb != 8) || wb < natural_bytes(p->w)) return RASP_EDTYPE;
    if (out->d == 0) return RASP_OK;
    Device dv;
    rc = device_info(dv);
    if (rc) return rc;
    const unsigned blocks = unsigned(std::min<uint64_t>((out->d * p->n + 255) / 256, uint64_t(dv.nsm) * 16));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const rasp::Side sd = side_of(out);
    const uint32_t ell = uint32_t(p->ell), s = uint32_t(p->s);
    switch (wb) {
    case 1: rasp::init_c0_kernel<uint8_t><<<blocks, 256, 0, st>>>(sd, out->d, p->n, ell, s, static_cast<const uint8_t *>(programs), prog_len, static_cast<const uint8_t *>(inputs), input_len); break;
    case 2: rasp::init_c0_kernel<uint16_t><<<blocks, 256, 0, st>>>(sd, out->d, p->n, ell, s, static_cast<const uint16_t *>(programs), prog_len, static_cast<const uint16_t *>(inputs), input_len); break;
    case 4: rasp::init_c0_kernel<uint32_t><<<blocks, 256, 0, st>>>(sd, out->d, p->n, ell, s, static_cast<const uint32_t *>(programs), prog_len, static_cast<const uint32_t *>(inputs), input_len); break;
    default: rasp::init_c0_kernel<uint64_t><<<blocks, 256, 0, st>>>(sd, out->d, p->n, ell, s, static_cast<const uint64_t *>(programs), prog_len, static_cast<const uint64_t *>(inputs), input_len); break;
    }
    RASP_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return RASP_OK;
}

int rasp_generate(const rasp_params *p, uint64_t seed, uint64_t first_machine, const rasp_batch *out,
                  void *stream)
{
    int rc = check_params(p);
    if (rc) return rc;
    if (!out) return RASP_EPARAM;
    const uint32_t wb = out->word_bytes;
    if ((wb != 1 && wb != 2 && wb != 4 && wb != 8) || wb < natural_bytes(p->w)) return RASP_EDTYPE;
    if (out->d == 0) return RASP_OK;
    Device dv;
    rc = device_info(dv);
    if (rc) return rc;
    const unsigned blocks = unsigned(std::min<uint64_t>((out->d * p->n + 255) / 256, uint64_t(dv.nsm) * 16));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const rasp::Side sd = side_of(out);
    const uint64_t mask = p->w == 64 ? ~0ull : ((1ull << p->w) - 1);
    const uint32_t ell = uint32_t(p->ell), s = uint32_t(p->s);
    switch (wb) {
    case 1: rasp::generate_kernel<uint8_t><<<blocks, 256, 0, st>>>(sd, out->d, first_machine, p->n, ell, s, mask, seed); break;
    case 2: rasp::generate_kernel<uint16_t><<<blocks, 256, 0, st>>>(sd, out->d, first_machine, p->n, ell, s, mask, seed); break;
    case 4: rasp::generate_kernel<uint32_t><<<blocks, 256, 0, st>>>(sd, out->d, first_machine, p->n, ell, s, mask, seed); break;
    default: rasp::generate_kernel<uint64_t><<<blocks, 256, 0, st>>>(sd, out->d, first_machine, p->n, ell, s, mask, seed); break;
    }
    RASP_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return RASP_OK;
}

int rasp_histogram(const int8_t *status, const int64_t *tau_h, uint64_t d, int64_t *out, void *stream)
{
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (!out) return RASP_EPARAM;
    RASP_CUDA(cudaMemsetAsync(out, 0, sizeof(int64_t) * 102, st));
    if (d == 0) return RASP_OK;
    Device dv;
    int rc = device_info(dv);
    if (rc) return rc;
    const uint64_t blocks = std::min<uint64_t>((d + 255) / 256, uint64_t(dv.nsm) * 8);
    rasp::histogram_kernel<<<unsigned(blocks), 256, 0, st>>>(
        status, tau_h, d, reinterpret_cast<unsigned long long *>(out));
    RASP_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return RASP_OK;
}

int rasp_validate(const rasp_params *p, const rasp_batch *b, int64_t *out, void *stream)
{
    int rc = check_params(p);
    if (rc) return rc;
    if (!b || !out) return RASP_EPARAM;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    RASP_CUDA(cudaMemsetAsync(out, 0, sizeof(int64_t) * 8, st));
    if (b->d == 0) return RASP_OK;
    Device dv;
    rc = device_info(dv);
    if (rc) return rc;
    const uint64_t mask = p->w == 64 ? ~0ull : ((1ull << p->w) - 1);
    const unsigned blocks = unsigned(std::min<uint64_t>((b->d * p->n + 255) / 256, uint64_t(dv.nsm) * 8));
    auto *o = reinterpret_cast<unsigned long long *>(out);
    const rasp::Side s = side_of(b);
    switch (b->word_bytes) {
    case 1: rasp::validate_kernel<uint8_t><<<blocks, 256, 0, st>>>(s, b->d, p->n, p->ell + 1, p->s + 1, mask, p->ell, p->s, o); break;
    case 2: rasp::validate_kernel<uint16_t><<<blocks, 256, 0, st>>>(s, b->d, p->n, p->ell + 1, p->s + 1, mask, p->ell, p->s, o); break;
    case 4: rasp::validate_kernel<uint32_t><<<blocks, 256, 0, st>>>(s, b->d, p->n, p->ell + 1, p->s + 1, mask, p->ell, p->s, o); break;
    case 8: rasp::validate_kernel<uint64_t><<<blocks, 256, 0, st>>>(s, b->d, p->n, p->ell + 1, p->s + 1, mask, p->ell, p->s, o); break;
    default: return RASP_EDTYPE;
    }
    RASP_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return RASP_OK;
}

}  // extern "C"
