// rasp_abi.cu -- extern "C" boundary of the B200 word-RASP engine
// (declared in include/raspvisor_b200.h).  The launch machinery is in
// rasp_host.cuh; the kernels in rasp_kernels.cuh.
#include "rasp_host.cuh"

namespace rasp {
namespace host {
thread_local char g_cuda_err[256] = "";
std::atomic<unsigned long long> g_launches{0};
}  // namespace host
}  // namespace rasp

using namespace rasp::host;

extern "C" {

int rasp_abi_version(void) { return RASP_ABI_VERSION; }

int rasp_checked_build(void) { return RASP_CHECKED; }

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
    case RASP_ENCCL: return "NCCL unavailable or an NCCL call failed";
    case RASP_ECHECK: return "kernel bounds/ownership check failed (checked build)";
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
    return rasp_run_hist(p, in, out, tau_max, epoch, flags, nullptr, workspace, workspace_bytes, stream);
}

int rasp_run_hist(const rasp_params *p, const rasp_batch *in, const rasp_batch *out, int64_t tau_max,
                  int64_t epoch, uint32_t flags, int64_t *hist, void *workspace, size_t workspace_bytes,
                  void *stream)
{
    int rc = check_params(p);
    if (rc) return rc;
    if (!in || !out || tau_max < 0 || epoch < 1) return RASP_EPARAM;
    if (in->d != out->d) return RASP_EPARAM;
    const uint64_t d = in->d;
    if (hist) RASP_CUDA(cudaMemsetAsync(hist, 0, sizeof(int64_t) * 102, static_cast<cudaStream_t>(stream)));
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
    a.g.m32 = uint32_t((1ull << 32) / p->n);
    a.g.ell = uint32_t(p->ell);
    a.g.s = uint32_t(p->s);
    a.in = side_of(in);
    a.out = side_of(out);
    a.tau_max = tau_max;
    a.hist = reinterpret_cast<unsigned long long *>(hist);
    a.fresh = (flags & RASP_FRESH) ? 1 : 0;
    a.inplace = (in->iw == out->iw) ? 1 : 0;
    a.tile_rows = pl.tile_rows;
    a.stable_q8 = 128;                       // 0.5 (measured best on C2 and C5): tuning knob RASP_STABLE_Q8
    if (const char *e = std::getenv("RASP_STABLE_Q8")) a.stable_q8 = uint32_t(std::strtoul(e, nullptr, 10));
    a.stable_hi_q8 = 243;                    // 0.95: tuning knob RASP_STABLE_HI_Q8
    if (const char *e = std::getenv("RASP_STABLE_HI_Q8")) a.stable_hi_q8 = uint32_t(std::strtoul(e, nullptr, 10));
    a.growth = 2;                            // tuning knob RASP_GROWTH (>= 2: the host plans for doubling)
    if (const char *e = std::getenv("RASP_GROWTH")) a.growth = std::max<uint32_t>(2, uint32_t(std::strtoul(e, nullptr, 10)));
    a.jump = 16;                             // tuning knob RASP_JUMP
    if (const char *e = std::getenv("RASP_JUMP")) a.jump = uint32_t(std::strtoul(e, nullptr, 10));
    a.pf_dist = 1;                           // tuning knob RASP_PREFETCH (0 disables)
    if (const char *e = std::getenv("RASP_PREFETCH")) a.pf_dist = uint32_t(std::strtoul(e, nullptr, 10));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (!a.inplace) {
        // out-of-place: the bookkeeping arrays move in bulk (non-fresh runs);
        // u and y rows are copied by the first epoch, tile by tile (bulk
        // copies here for big tiles); the kernels then treat `out` as the
        // working copy
        int rc2 = RASP_OK;
        if (pl.smem && pl.big) {
            const size_t ub = size_t(d) * (p->ell + 1) * wb, yb = size_t(d) * (p->s + 1) * wb;
            rc2 = dev_copy(out->u, in->u, ub, dv, st);
            if (!rc2) rc2 = dev_copy(out->y, in->y, yb, dv, st);
        }
        if (!rc2 && !a.fresh) {
            rc2 = dev_copy(out->status, in->status, size_t(d), dv, st);
            if (!rc2) rc2 = dev_copy(out->steps, in->steps, size_t(d) * 8, dv, st);
            if (!rc2) rc2 = dev_copy(out->tau_h, in->tau_h, size_t(d) * 8, dv, st);
        }
        if (rc2) return rc2;
    }
    switch (wb) {
    case 1: return run_typed<uint8_t>(p, a, pl, dv, ws, d, tau_max, epoch, st);
    case 2: return run_typed<uint16_t>(p, a, pl, dv, ws, d, tau_max, epoch, st);
    case 4: return run_typed<uint32_t>(p, a, pl, dv, ws, d, tau_max, epoch, st);
    default: return run_typed<uint64_t>(p, a, pl, dv, ws, d, tau_max, epoch, st);
    }
}

int rasp_enumerate(const rasp_enum_params *ep, uint64_t first_rank, uint64_t count, uint64_t *records,
                   unsigned long long *steps_total, void *stream)
{
    if (!ep || !records || !steps_total) return RASP_EPARAM;
    if (ep->w < 2 || ep->w > 8 || ep->n < 2 || ep->n > 4096 || ep->m < 1 || ep->opcode_bits < 1 ||
        ep->operand_bits < 1 || ep->opcode_bits > ep->w || ep->operand_bits > ep->w ||
        uint64_t(ep->m) * (ep->opcode_bits + ep->operand_bits) > 63)
        return RASP_EPARAM;
    if (ep->tau_max >= (1u << 14)) return RASP_EPARAM;   // tau_h must fit the record key's 14 bits
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
    a.g.m32 = uint32_t((1ull << 32) / ep->n);
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
    // per warp: its tile (n + 3 rows of 32 u16 cells) + the program (n cells)
    const size_t smem = size_t(8) * ((ep->n + 3) * 64 + ((2 * ep->n + 15) & ~15u));
    const bool pow2 = (ep->n & (ep->n - 1)) == 0;
    // steps between lane checks: 2, or 1 when tau_max is odd (machines start at
    // checks and must reach their budget exactly at one)
#ifndef RASP_ENUM_CHECK
#define RASP_ENUM_CHECK 2
#endif
    const bool even = RASP_ENUM_CHECK == 2 && (ep->tau_max & 1) == 0;
    auto kern = pow2 ? (even ? rasp::enum_kernel<true, rasp::Arith::NARROW, 2> : rasp::enum_kernel<true, rasp::Arith::NARROW, 1>)
                     : (even ? rasp::enum_kernel<false, rasp::Arith::NARROW, 2> : rasp::enum_kernel<false, rasp::Arith::NARROW, 1>);
    if (smem > size_t(dv.smem_optin)) return RASP_ECAPACITY;
    int per_sm = 0;
    {
        std::lock_guard<std::mutex> lock(launch_mutex());
        rc = raise_smem_limit_locked(reinterpret_cast<const void *>(kern), dv);
        if (rc) return rc;
        RASP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, smem));
    }
    if (per_sm < 1) return RASP_ECAPACITY;
    // one resident wave of blocks; every warp loops over whole programs
    const uint64_t grid = std::min<uint64_t>((count + 7) / 8, uint64_t(per_sm) * dv.nsm);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    kern<<<unsigned(grid), 256, smem, st>>>(a);
    RASP_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return checked_result(st);
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
    const uint64_t blocks = std::min<uint64_t>((d + 1023) / 1024, uint64_t(dv.nsm));
    rasp::histogram_kernel<<<unsigned(blocks), 1024, 0, st>>>(
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
