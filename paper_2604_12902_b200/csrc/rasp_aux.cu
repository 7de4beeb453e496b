// rasp_aux.cu -- the boundary's auxiliary entry points (include/raspvisor_b200.h):
//   * rasp_pack / rasp_unpack: word-width conversion between the reference's
//     uint64 SoA arrays (hv:280-284) and the engine's natural-width arrays;
//   * rasp_topk: bb-search's "K longest halting runs" (cli.py:195-230) on the
//     device: a radix select on tau_h, an index-ordered compaction of the
//     threshold ties, and a one-block bitonic sort of the K survivors;
//   * rasp_nccl_* / rasp_shard_*: the post-run collectives of a sharded run
//      on an NCCL communicator, NCCL resolved at run time.
#include "rasp_host.cuh"

#include <climits>
#include <cstddef>
#include <dlfcn.h>

using namespace rasp::host;

namespace {

// ---------------------------------------------------------------- pack/unpack
// One grid-stride sweep per field; every element is read and written once
// (HBM-bound: src + dst bytes per word).
template <class Si, class So>
__global__ void convert_kernel(rasp::Side src, rasp::Side dst, uint64_t d, uint64_t ncols, uint64_t ucols,
                               uint64_t ycols)
{
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    const uint64_t t0 = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    const Si *si[5] = {static_cast<const Si *>(src.iw), static_cast<const Si *>(src.ac),
                       static_cast<const Si *>(src.M), static_cast<const Si *>(src.u),
                       static_cast<const Si *>(src.y)};
    So *so[5] = {static_cast<So *>(dst.iw), static_cast<So *>(dst.ac), static_cast<So *>(dst.M),
                 static_cast<So *>(dst.u), static_cast<So *>(dst.y)};
    const uint64_t len[5] = {d, d, d * ncols, d * ucols, d * ycols};
#pragma unroll
    for (int f = 0; f < 5; ++f)
        for (uint64_t k = t0; k < len[f]; k += stride) so[f][k] = static_cast<So>(si[f][k]);
}

template <class Si>
int convert_from(const rasp_params *p, const rasp_batch *src, const rasp_batch *dst, unsigned blocks,
                 cudaStream_t st)
{
    const rasp::Side a = side_of(src), b = side_of(dst);
    const uint64_t d = src->d, n = p->n, uc = p->ell + 1, yc = p->s + 1;
    switch (dst->word_bytes) {
    case 1: convert_kernel<Si, uint8_t><<<blocks, 256, 0, st>>>(a, b, d, n, uc, yc); break;
    case 2: convert_kernel<Si, uint16_t><<<blocks, 256, 0, st>>>(a, b, d, n, uc, yc); break;
    case 4: convert_kernel<Si, uint32_t><<<blocks, 256, 0, st>>>(a, b, d, n, uc, yc); break;
    default: convert_kernel<Si, uint64_t><<<blocks, 256, 0, st>>>(a, b, d, n, uc, yc); break;
    }
    RASP_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return RASP_OK;
}

bool word_bytes_ok(uint32_t wb) { return wb == 1 || wb == 2 || wb == 4 || wb == 8; }

int convert(const rasp_params *p, const rasp_batch *src, const rasp_batch *dst, void *stream)
{
    int rc = check_params(p);
    if (rc) return rc;
    if (!src || !dst || src->d != dst->d) return RASP_EPARAM;
    if (!word_bytes_ok(src->word_bytes) || !word_bytes_ok(dst->word_bytes) ||
        dst->word_bytes < natural_bytes(p->w))
        return RASP_EDTYPE;
    const uint64_t d = src->d;
    if (d == 0) return RASP_OK;
    Device dv;
    rc = device_info(dv);
    if (rc) return rc;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const unsigned blocks = unsigned(std::min<uint64_t>((d * p->n + 255) / 256, uint64_t(dv.nsm) * 16));
    switch (src->word_bytes) {
    case 1: rc = convert_from<uint8_t>(p, src, dst, blocks, st); break;
    case 2: rc = convert_from<uint16_t>(p, src, dst, blocks, st); break;
    case 4: rc = convert_from<uint32_t>(p, src, dst, blocks, st); break;
    default: rc = convert_from<uint64_t>(p, src, dst, blocks, st); break;
    }
    if (rc) return rc;
    // run bookkeeping is width-independent: plain copies when both sides have it
    if (src->status && dst->status && src->status != dst->status)
        if ((rc = dev_copy(dst->status, src->status, d, dv, st))) return rc;
    if (src->steps && dst->steps && src->steps != dst->steps)
        if ((rc = dev_copy(dst->steps, src->steps, d * 8, dv, st))) return rc;
    if (src->tau_h && dst->tau_h && src->tau_h != dst->tau_h)
        if ((rc = dev_copy(dst->tau_h, src->tau_h, d * 8, dv, st))) return rc;
    return RASP_OK;
}

// ----------------------------------------------------------------------- top-k
constexpr int kRadixBits = 11;
constexpr int kBins = 1 << kRadixBits;
constexpr int kMaxPasses = (64 + kRadixBits - 1) / kRadixBits;
constexpr int kTopkBlocks = 1024;       // compaction blocks (contiguous index chunks)
constexpr int kTopkMax = 2048;          // largest K (one-block sort in shared memory)

struct TopkState {
    unsigned long long hist[kMaxPasses][kBins];
    unsigned long long prefix, mask;    // key bits fixed so far
    long long need;                     // ties still to take at the threshold
    unsigned long long gt;              // candidates strictly above the threshold (appended)
    int all;                            // fewer halted machines than K: take them all
    int pad_;
};

size_t topk_layout(uint32_t k, size_t *off_blocks, size_t *off_cand)
{
    size_t off = align256(sizeof(TopkState));
    if (off_blocks) *off_blocks = off;
    off += align256(sizeof(unsigned long long) * kTopkBlocks);
    if (off_cand) *off_cand = off;
    off += align256(sizeof(long long) * 2 * std::max<uint32_t>(k, 1));
    return off;
}

// Histogram of the current digit of tau_h over the halted machines whose
// higher digits match the prefix selected so far.
__global__ void __launch_bounds__(1024) topk_hist_kernel(const int8_t *__restrict__ status,
                                                         const int64_t *__restrict__ tau_h, uint64_t d,
                                                         TopkState *stt, int pass, int shift)
{
    __shared__ unsigned int h[kBins];
    if (stt->all) return;
    for (int k = threadIdx.x; k < kBins; k += blockDim.x) h[k] = 0;
    __syncthreads();
    const unsigned long long prefix = stt->prefix, mask = stt->mask;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; j < d; j += stride) {
        if (status[j] != rasp::kHalted) continue;
        const unsigned long long key = static_cast<unsigned long long>(tau_h[j]);
        if ((key & mask) == prefix) atomicAdd(&h[(key >> shift) & (kBins - 1)], 1u);
    }
    __syncthreads();
    for (int k = threadIdx.x; k < kBins; k += blockDim.x)
        if (h[k]) atomicAdd(&stt->hist[pass][k], static_cast<unsigned long long>(h[k]));
}

// Pick the digit holding the K-th largest key: suffix sums over the bins
// (descending digit order), one block.
__global__ void __launch_bounds__(1024) topk_select_kernel(TopkState *stt, int pass, int shift, uint32_t k)
{
    __shared__ unsigned long long cnt[kBins];
    __shared__ unsigned long long suf[1024];
    if (stt->all) return;
    const long long need = pass == 0 ? static_cast<long long>(k) : stt->need;  // read before any write
    const int t = threadIdx.x;   // thread t owns descending bins 2t, 2t+1
    for (int b = t; b < kBins; b += blockDim.x) cnt[b] = stt->hist[pass][kBins - 1 - b];
    __syncthreads();
    suf[t] = cnt[2 * t] + cnt[2 * t + 1];
    __syncthreads();
    for (int off = 1; off < 1024; off <<= 1) {   // inclusive scan (Hillis-Steele)
        const unsigned long long v = t >= off ? suf[t - off] : 0;
        __syncthreads();
        suf[t] += v;
        __syncthreads();
    }
    const unsigned long long total = suf[1023];
    if (pass == 0 && total <= static_cast<unsigned long long>(need)) {
        if (t == 0) stt->all = 1;
        return;
    }
    const unsigned long long before = t ? suf[t - 1] : 0;   // keys in higher bins
    for (int q = 0; q < 2; ++q) {
        const unsigned long long above = before + (q ? cnt[2 * t] : 0);
        const unsigned long long here = cnt[2 * t + q];
        if (here && above < static_cast<unsigned long long>(need) &&
            static_cast<unsigned long long>(need) <= above + here) {
            const unsigned long long digit = kBins - 1 - (2 * t + q);
            stt->prefix |= digit << shift;
            stt->mask |= static_cast<unsigned long long>(kBins - 1) << shift;
            stt->need = need - static_cast<long long>(above);
        }
    }
}

// Candidates strictly above the threshold are appended (fewer than K); ties
// at the threshold are counted per contiguous index chunk.
__global__ void __launch_bounds__(1024) topk_gather_kernel(const int8_t *__restrict__ status,
                                                           const int64_t *__restrict__ tau_h, uint64_t d,
                                                           uint64_t chunk, unsigned long long limit,
                                                           TopkState *stt,
                                                           unsigned long long *__restrict__ blockcount,
                                                           long long *__restrict__ cand)
{
    __shared__ unsigned int ties;
    if (threadIdx.x == 0) ties = 0;
    __syncthreads();
    const int all = stt->all;
    const unsigned long long thr = stt->prefix;
    const uint64_t lo = blockIdx.x * chunk, hi = std::min<uint64_t>(d, lo + chunk);
    unsigned int mine = 0;
    for (uint64_t j = lo + threadIdx.x; j < hi; j += blockDim.x) {
        if (status[j] != rasp::kHalted) continue;
        const unsigned long long key = static_cast<unsigned long long>(tau_h[j]);
        if (key > limit) continue;   // outside the contract (tau_h <= tau_max); never selected
        if (all || key > thr) {
            const unsigned long long at = atomicAdd(&stt->gt, 1ull);
            cand[2 * at] = static_cast<long long>(key);
            cand[2 * at + 1] = static_cast<long long>(j);
        } else if (key == thr) {
            ++mine;
        }
    }
    if (mine) atomicAdd(&ties, mine);
    __syncthreads();
    if (threadIdx.x == 0) blockcount[blockIdx.x] = ties;
}

// The `need` lowest-index ties, in index order: each block ranks its chunk's
// ties after the ties of all lower chunks.
__global__ void __launch_bounds__(1024) topk_ties_kernel(const int8_t *__restrict__ status,
                                                         const int64_t *__restrict__ tau_h, uint64_t d,
                                                         uint64_t chunk, TopkState *stt,
                                                         const unsigned long long *__restrict__ blockcount,
                                                         long long *__restrict__ cand)
{
    __shared__ unsigned long long part[32];
    __shared__ unsigned int wsum[32];
    if (stt->all) return;
    const long long need = stt->need;
    const unsigned long long gt = stt->gt, thr = stt->prefix;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    unsigned long long s = 0;
    for (unsigned b = threadIdx.x; b < blockIdx.x; b += blockDim.x) s += blockcount[b];
    for (int off = 16; off; off >>= 1) s += __shfl_down_sync(rasp::kFull, s, off);
    if (lane == 0) part[wid] = s;
    __syncthreads();
    unsigned long long base = 0;
    for (int w = 0; w < nw; ++w) base += part[w];
    if (base >= static_cast<unsigned long long>(need) || blockcount[blockIdx.x] == 0) return;
    const uint64_t lo = blockIdx.x * chunk, hi = std::min<uint64_t>(d, lo + chunk);
    for (uint64_t j0 = lo; j0 < hi && base < static_cast<unsigned long long>(need); j0 += blockDim.x) {
        const uint64_t j = j0 + threadIdx.x;
        const bool tie = j < hi && status[j] == rasp::kHalted &&
                         static_cast<unsigned long long>(tau_h[j]) == thr;
        const unsigned int bal = __ballot_sync(rasp::kFull, tie);
        if (lane == 0) wsum[wid] = __popc(bal);
        __syncthreads();
        unsigned int before = 0, total = 0;
        for (int w = 0; w < nw; ++w) {
            before += w < wid ? wsum[w] : 0;
            total += wsum[w];
        }
        const unsigned long long rank = base + before + __popc(bal & ((1u << lane) - 1));
        if (tie && rank < static_cast<unsigned long long>(need)) {
            cand[2 * (gt + rank)] = static_cast<long long>(thr);
            cand[2 * (gt + rank) + 1] = static_cast<long long>(j);
        }
        base += total;
        __syncthreads();
    }
}

// Bitonic sort of the (at most K) candidates: tau_h descending, index
// ascending -- the order of sorted(heap, reverse=True) over (tau_h, -index).
__global__ void __launch_bounds__(1024) topk_sort_kernel(const TopkState *stt, const long long *__restrict__ cand,
                                                         uint32_t k, int64_t *__restrict__ out_index,
                                                         int64_t *__restrict__ out_tau)
{
    __shared__ long long key[kTopkMax], idx[kTopkMax];
    const unsigned long long have = stt->all ? stt->gt : static_cast<unsigned long long>(k);
    uint32_t P = 1;
    while (P < have) P <<= 1;
    for (uint32_t r = threadIdx.x; r < P; r += blockDim.x) {
        key[r] = r < have ? cand[2 * r] : -1;
        idx[r] = r < have ? cand[2 * r + 1] : LLONG_MAX;
    }
    __syncthreads();
    for (uint32_t size = 2; size <= P; size <<= 1)
        for (uint32_t stride = size >> 1; stride; stride >>= 1) {
            for (uint32_t r = threadIdx.x; r < P; r += blockDim.x) {
                const uint32_t q = r ^ stride;
                if (q > r) {
                    // "a before b": larger tau first, then smaller index
                    const bool first_ok = key[r] > key[q] || (key[r] == key[q] && idx[r] < idx[q]);
                    const bool up = (r & size) == 0;
                    if (first_ok != up) {
                        const long long tk = key[r], ti = idx[r];
                        key[r] = key[q]; idx[r] = idx[q];
                        key[q] = tk; idx[q] = ti;
                    }
                }
            }
            __syncthreads();
        }
    for (uint32_t r = threadIdx.x; r < k; r += blockDim.x) {
        out_tau[r] = r < have ? key[r] : -1;
        out_index[r] = r < have ? idx[r] : -1;
    }
}

// ------------------------------------------------------------------------ NCCL
// The few NCCL entry points the shard collectives use, resolved with dlsym
// from the process's libnccl.so.2 (the one torch already loaded, else the
// first on the loader path or $RASP_NCCL_LIBRARY).  Types follow nccl.h:
// ncclUniqueId is 128 opaque bytes; results, data types and ops are ints.
struct NcclUid { char internal[128]; };
using nccl_res = int;
struct Nccl {
    bool tried = false, ok = false;
    nccl_res (*get_unique_id)(NcclUid *) = nullptr;
    nccl_res (*comm_init_rank)(void **, int, NcclUid, int) = nullptr;
    nccl_res (*comm_destroy)(void *) = nullptr;
    nccl_res (*comm_count)(void *, int *) = nullptr;
    nccl_res (*user_rank)(void *, int *) = nullptr;
    nccl_res (*all_reduce)(const void *, void *, size_t, int, int, void *, cudaStream_t) = nullptr;
    nccl_res (*send)(const void *, size_t, int, int, void *, cudaStream_t) = nullptr;
    nccl_res (*recv)(void *, size_t, int, int, void *, cudaStream_t) = nullptr;
    nccl_res (*group_start)() = nullptr;
    nccl_res (*group_end)() = nullptr;
    const char *(*error_string)(nccl_res) = nullptr;
};
constexpr int kNcclUint8 = 1, kNcclInt64 = 4, kNcclSum = 0;

Nccl &nccl()
{
    static Nccl n;
    if (n.tried) return n;
    n.tried = true;
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) {
        const char *env = std::getenv("RASP_NCCL_LIBRARY");
        h = dlopen(env && *env ? env : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    }
    if (!h) {
        std::snprintf(g_cuda_err, sizeof g_cuda_err, "NCCL not loadable: %s", dlerror());
        return n;
    }
#define RASP_SYM(field, name) n.field = reinterpret_cast<decltype(n.field)>(dlsym(h, name))
    RASP_SYM(get_unique_id, "ncclGetUniqueId");
    RASP_SYM(comm_init_rank, "ncclCommInitRank");
    RASP_SYM(comm_destroy, "ncclCommDestroy");
    RASP_SYM(comm_count, "ncclCommCount");
    RASP_SYM(user_rank, "ncclCommUserRank");
    RASP_SYM(all_reduce, "ncclAllReduce");
    RASP_SYM(send, "ncclSend");
    RASP_SYM(recv, "ncclRecv");
    RASP_SYM(group_start, "ncclGroupStart");
    RASP_SYM(group_end, "ncclGroupEnd");
    RASP_SYM(error_string, "ncclGetErrorString");
#undef RASP_SYM
    n.ok = n.get_unique_id && n.comm_init_rank && n.comm_destroy && n.comm_count && n.user_rank &&
           n.all_reduce && n.send && n.recv && n.group_start && n.group_end && n.error_string;
    if (!n.ok) std::snprintf(g_cuda_err, sizeof g_cuda_err, "NCCL library lacks a required symbol");
    return n;
}

int nccl_fail(nccl_res r, const char *what)
{
    std::snprintf(g_cuda_err, sizeof g_cuda_err, "%s: %s", what, nccl().error_string(r));
    return RASP_ENCCL;
}

#define RASP_NCCL(call)                                  \
    do {                                                 \
        nccl_res r_ = (call);                            \
        if (r_ != 0) return nccl_fail(r_, #call);        \
    } while (0)

void bounds(uint64_t d, int world, int rank, uint64_t &lo, uint64_t &hi)
{
    const uint64_t per = d ? (d + world - 1) / world : 0;
    lo = std::min<uint64_t>(d, uint64_t(rank) * per);
    hi = std::min<uint64_t>(d, lo + per);
}

}  // namespace

extern "C" {

int rasp_pack(const rasp_params *p, const rasp_batch *src, const rasp_batch *dst, void *stream)
{
    return convert(p, src, dst, stream);
}

int rasp_unpack(const rasp_params *p, const rasp_batch *src, const rasp_batch *dst, void *stream)
{
    return convert(p, src, dst, stream);
}

size_t rasp_topk_workspace_bytes(uint32_t k) { return topk_layout(k, nullptr, nullptr); }

int rasp_topk(const int8_t *status, const int64_t *tau_h, uint64_t d, int64_t tau_max, uint32_t k,
              int64_t *out_index, int64_t *out_tau, void *workspace, size_t workspace_bytes, void *stream)
{
    if (k == 0) return RASP_OK;
    if (!out_index || !out_tau || tau_max < 0 || (d && (!status || !tau_h))) return RASP_EPARAM;
    if (k > uint32_t(kTopkMax)) return RASP_ECAPACITY;
    size_t off_blocks = 0, off_cand = 0;
    const size_t need_bytes = topk_layout(k, &off_blocks, &off_cand);
    if (!workspace || workspace_bytes < need_bytes) return RASP_EWORKSPACE;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    auto *base = static_cast<unsigned char *>(workspace);
    auto *stt = reinterpret_cast<TopkState *>(base);
    auto *blockcount = reinterpret_cast<unsigned long long *>(base + off_blocks);
    auto *cand = reinterpret_cast<long long *>(base + off_cand);
    Device dv;
    int rc = device_info(dv);
    if (rc) return rc;
    // key bits: every halted tau_h is <= tau_max; the prefix starts with the
    // bits above them fixed at 0
    const int bits = tau_max ? 64 - __builtin_clzll(static_cast<unsigned long long>(tau_max)) : 1;
    const int passes = (bits + kRadixBits - 1) / kRadixBits;
    TopkState init{};
    init.mask = bits >= 64 ? 0ull : ~((1ull << bits) - 1);
    RASP_CUDA(cudaMemsetAsync(stt, 0, sizeof(TopkState), st));
    RASP_CUDA(cudaMemcpyAsync(&stt->mask, &init.mask, sizeof init.mask, cudaMemcpyHostToDevice, st));
    const unsigned hblocks = unsigned(std::max<uint64_t>(1, std::min<uint64_t>((d + 1023) / 1024, uint64_t(dv.nsm))));
    for (int q = 0; q < passes; ++q) {
        const int shift = (passes - 1 - q) * kRadixBits;
        topk_hist_kernel<<<hblocks, 1024, 0, st>>>(status, tau_h, d, stt, q, shift);
        topk_select_kernel<<<1, 1024, 0, st>>>(stt, q, shift, k);
        g_launches.fetch_add(2, std::memory_order_relaxed);
    }
    const uint64_t chunk = std::max<uint64_t>(1024, ((d + kTopkBlocks - 1) / kTopkBlocks + 1023) / 1024 * 1024);
    const unsigned cblocks = unsigned(std::max<uint64_t>(1, (d + chunk - 1) / chunk));
    topk_gather_kernel<<<cblocks, 1024, 0, st>>>(status, tau_h, d, chunk, ~init.mask, stt, blockcount, cand);
    topk_ties_kernel<<<cblocks, 1024, 0, st>>>(status, tau_h, d, chunk, stt, blockcount, cand);
    topk_sort_kernel<<<1, 1024, 0, st>>>(stt, cand, k, out_index, out_tau);
    RASP_CUDA(cudaGetLastError());
    g_launches.fetch_add(3, std::memory_order_relaxed);
    return RASP_OK;
}

int rasp_nccl_unique_id(void *id_out)
{
    if (!id_out) return RASP_EPARAM;
    Nccl &n = nccl();
    if (!n.ok) return RASP_ENCCL;
    NcclUid id;
    RASP_NCCL(n.get_unique_id(&id));
    std::memcpy(id_out, &id, sizeof id);
    return RASP_OK;
}

int rasp_nccl_comm_init(int nranks, const void *id, int rank, void **comm_out)
{
    if (!id || !comm_out || nranks < 1 || rank < 0 || rank >= nranks) return RASP_EPARAM;
    Nccl &n = nccl();
    if (!n.ok) return RASP_ENCCL;
    NcclUid uid;
    std::memcpy(&uid, id, sizeof uid);
    RASP_NCCL(n.comm_init_rank(comm_out, nranks, uid, rank));
    return RASP_OK;
}

int rasp_nccl_comm_destroy(void *comm)
{
    if (!comm) return RASP_OK;
    Nccl &n = nccl();
    if (!n.ok) return RASP_ENCCL;
    RASP_NCCL(n.comm_destroy(comm));
    return RASP_OK;
}

int rasp_shard_allreduce(void *comm, int64_t *counters, uint64_t count, void *stream)
{
    if (!comm || (count && !counters)) return RASP_EPARAM;
    Nccl &n = nccl();
    if (!n.ok) return RASP_ENCCL;
    if (count == 0) return RASP_OK;
    RASP_NCCL(n.all_reduce(counters, counters, count, kNcclInt64, kNcclSum, comm, static_cast<cudaStream_t>(stream)));
    return RASP_OK;
}

int rasp_shard_gather(void *comm, int root, const rasp_params *p, uint64_t d_total, const rasp_batch *shard,
                      const rasp_batch *full, uint32_t fields, void *stream)
{
    int rc = check_params(p);
    if (rc) return rc;
    if (!comm || !shard) return RASP_EPARAM;
    Nccl &n = nccl();
    if (!n.ok) return RASP_ENCCL;
    int world = 0, rank = 0;
    RASP_NCCL(n.comm_count(comm, &world));
    RASP_NCCL(n.user_rank(comm, &rank));
    if (root < 0 || root >= world) return RASP_EPARAM;
    uint64_t lo, hi;
    bounds(d_total, world, rank, lo, hi);
    if (shard->d != hi - lo) return RASP_EPARAM;
    if (rank == root && (!full || full->d != d_total || full->word_bytes != shard->word_bytes)) return RASP_EPARAM;
    if (!word_bytes_ok(shard->word_bytes)) return RASP_EDTYPE;
    const size_t wb = shard->word_bytes;
    // per-machine extents of the gathered fields (bytes), in a fixed order
    struct F { size_t per; size_t off; bool on; };
    const F f[8] = {
        {1, offsetof(rasp_batch, status), (fields & RASP_GATHER_RESULTS) != 0},
        {8, offsetof(rasp_batch, steps), (fields & RASP_GATHER_RESULTS) != 0},
        {8, offsetof(rasp_batch, tau_h), (fields & RASP_GATHER_RESULTS) != 0},
        {wb * (p->s + 1), offsetof(rasp_batch, y), (fields & RASP_GATHER_OUTPUT) != 0},
        {wb, offsetof(rasp_batch, iw), (fields & RASP_GATHER_CONFIG) != 0},
        {wb, offsetof(rasp_batch, ac), (fields & RASP_GATHER_CONFIG) != 0},
        {wb * p->n, offsetof(rasp_batch, M), (fields & RASP_GATHER_CONFIG) != 0},
        {wb * (p->ell + 1), offsetof(rasp_batch, u), (fields & RASP_GATHER_CONFIG) != 0},
    };
    auto ptr = [](const rasp_batch *b, size_t off) {
        return *reinterpret_cast<unsigned char *const *>(reinterpret_cast<const unsigned char *>(b) + off);
    };
    for (const F &x : f)
        if (x.on && (!ptr(shard, x.off) || (rank == root && !ptr(full, x.off)))) return RASP_EPARAM;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    Device dv;
    if ((rc = device_info(dv))) return rc;
    if (rank == root)
        for (const F &x : f)
            if (x.on && (rc = dev_copy(ptr(full, x.off) + lo * x.per, ptr(shard, x.off), shard->d * x.per, dv, st)))
                return rc;
    if (world == 1) return RASP_OK;
    RASP_NCCL(n.group_start());
    for (const F &x : f) {
        if (!x.on) continue;
        if (rank != root) {
            if (shard->d) RASP_NCCL(n.send(ptr(shard, x.off), shard->d * x.per, kNcclUint8, root, comm, st));
        } else {
            for (int r = 0; r < world; ++r) {
                if (r == root) continue;
                uint64_t rl, rh;
                bounds(d_total, world, r, rl, rh);
                if (rh > rl) RASP_NCCL(n.recv(ptr(full, x.off) + rl * x.per, (rh - rl) * x.per, kNcclUint8, r, comm, st));
            }
        }
    }
    RASP_NCCL(n.group_end());
    return RASP_OK;
}

}  // extern "C"
