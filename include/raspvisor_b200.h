/*
 * raspvisor_b200.h -- C ABI of the B200 word-RASP batch engine.
 *
 * Drop-in boundary for the reference's batch kernel.  The reference binds
 * exactly one native entry point on this path,
 *
 *     _worker(iw, ac, M, u, y, status, steps, tau_h, g, W, q, rounds,
 *             tau_max, wmask, n, ell, s)
 *         /root/reference/pkg/src/raspvisor/hypervisor.py:128-164
 *
 * called once per host thread from run_batch (hypervisor.py:305-314) on
 * C-contiguous SoA arrays it allocated itself.  rasp_run below replaces the
 * W concurrent _worker calls with one device-side run over the whole batch:
 * same arrays (device pointers, element width `word_bytes`), same in-place
 * contract, same per-machine results, independent of `epoch` the way the
 * reference is independent of (W, q) (hypervisor.py:1-9).
 *
 * Conventions: every pointer is a DEVICE pointer owned by the caller (torch
 * tensors on the Python side); nothing here frees caller memory.  Every
 * function returns 0 on success or a negative RASP_E* code; no exception
 * crosses the ABI.  `stream` is a cudaStream_t passed as void*.  All work is
 * enqueued on `stream`; nothing synchronises unless documented.
 */
#ifndef RASPVISOR_B200_H
#define RASPVISOR_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RASP_ABI_VERSION 3

/* error codes */
#define RASP_OK 0
#define RASP_EPARAM -1      /* bad machine params (hv:299-300 scalars / m:72-86) */
#define RASP_ECAPACITY -2   /* batch or geometry beyond what the engine supports */
#define RASP_ECUDA -3       /* a CUDA call failed; see rasp_last_cuda_error */
#define RASP_EWORKSPACE -4  /* workspace too small */
#define RASP_EDTYPE -5      /* word_bytes not in {1,2,4,8} or narrower than w */
#define RASP_ENCCL -6       /* NCCL missing or an NCCL call failed; see rasp_last_cuda_error */
#define RASP_ECHECK -7      /* checked build only: a kernel bounds/ownership check failed;
                               details in rasp_last_cuda_error */

/* VM status codes: hypervisor.py:63-69 */
#define RASP_RUNNING 0
#define RASP_HALTED 1
#define RASP_EXHAUSTED 2

/* Machine geometry: the (wmask, n, ell, s) scalars of _worker
 * (hypervisor.py:299-300), with w instead of wmask. */
typedef struct rasp_params {
    uint32_t w;    /* word width, 1..64 */
    uint32_t n;    /* memory cells, >= 2 */
    uint64_t ell;  /* input capacity, 1 <= ell < 2^w */
    uint64_t s;    /* output capacity, 1 <= s < 2^w */
} rasp_params;

/* One batch of d machines in the reference's SoA layout (hypervisor.py:280-293):
 * iw[d], ac[d], M[d][n], u[d][ell+1] (u[.][0] = read cursor),
 * y[d][s+1] (y[.][0] = write count), all words of `word_bytes` bytes
 * (1, 2, 4 or 8; at least ceil(w/8) rounded up to a power of two);
 * status int8[d], steps int64[d], tau_h int64[d]. */
typedef struct rasp_batch {
    void *iw, *ac, *M, *u, *y;
    int8_t *status;
    int64_t *steps;
    int64_t *tau_h;
    uint64_t d;
    uint32_t word_bytes;
    uint32_t _pad;
} rasp_batch;

/* rasp_run flags */
#define RASP_FRESH 1u   /* caller guarantees status == 0, steps == 0 on input
                           (run_batch's fresh arrays, hv:291-293): skip reading them */

/* Bytes of device workspace rasp_run needs for a batch of d machines. */
size_t rasp_workspace_bytes(const rasp_params *p, uint64_t d);

/* Run every RUNNING machine of `in` to a fixed point or tau_max total steps.
 * Replaces the W calls of _worker (hypervisor.py:128-164 via :305-314).
 *   in, out : may be the same batch (in-place, the reference's contract) or
 *             two distinct batches of the same shape (out-of-place: `in` is
 *             only read; every field of `out` is written).
 *   Results per machine j, for any `epoch` >= 1:
 *     HALTED    (status 1): tau_h = steps = least t with Phi^t(c) fixed, t <= tau_max
 *     EXHAUSTED (status 2): steps = tau_max, tau_h unchanged (-1 from run_batch)
 *     final config = Phi^steps(c);  machines entering with status != 0 are untouched.
 *   epoch   : length of the first on-device epoch (the reference's q); later
 *             epochs double it.  Performance knob only: a fresh run of big
 *             machines (u32/u64 tiles) whose budget is a multiple of 16 and at
 *             most 2048, on 16-byte aligned rows, runs as one per-lane refill
 *             launch over the whole budget instead (same results).
 *   workspace: device buffer of at least rasp_workspace_bytes(p, d) bytes.
 * Asynchronous on `stream` (may synchronise internally only when tau_max is
 * too large for a fixed epoch schedule, to poll the live count).  A machine
 * can run at most 1024 epochs of at most 2^24 steps (~1.7e10 steps): larger
 * budgets on machines that never halt return RASP_ECAPACITY. */
int rasp_run(const rasp_params *p, const rasp_batch *in, const rasp_batch *out,
             int64_t tau_max, int64_t epoch, uint32_t flags,
             void *workspace, size_t workspace_bytes, void *stream);

/* rasp_run plus the halting histogram of the batch after the run, computed
 * inside the epoch kernels (each verdict counted as it is written; machines
 * entering with status != 0 counted as they stand): hist[0..99] = machines
 * HALTED with tau_h = k, hist[100] = HALTED with tau_h >= 100, hist[101] =
 * EXHAUSTED -- collect_histogram / HISTOGRAM_KEYS (hypervisor.py:326-352).
 * `hist` is a device int64[102], zeroed by the call; NULL = plain rasp_run.
 * Replaces rasp_run + rasp_histogram (one launch and a 9 B/machine re-read
 * fewer). */
int rasp_run_hist(const rasp_params *p, const rasp_batch *in, const rasp_batch *out,
                  int64_t tau_max, int64_t epoch, uint32_t flags, int64_t *hist,
                  void *workspace, size_t workspace_bytes, void *stream);

/* Device packer of init_config (machine.py:289-309) for a whole batch:
 * M = program || 0, u = (0, inputs || 0), y = 0, i = a = 0, status = 0,
 * steps = 0, tau_h = -1.  programs: [d][prog_len], inputs: [d][input_len],
 * both device buffers of out->word_bytes words (range-checked by the caller).
 * Lets a caller ship only programs and inputs over PCIe. */
int rasp_init_c0(const rasp_params *p, const void *programs, uint32_t prog_len,
                 const void *inputs, uint32_t input_len, const rasp_batch *out, void *stream);

/* Generator G_dev (SURVEY §8d generator G, on the device): every program
 * fills memory with opcode/operand pairs (opcode uniform in 1..7, operand
 * uniform in [0, n), BNZ operands even), ell uniform input words, i = a = 0.
 * Machine j of the batch is machine first_machine + j of the stream `seed`
 * (counter-based splitmix64), so shards generate independently. */
int rasp_generate(const rasp_params *p, uint64_t seed, uint64_t first_machine,
                  const rasp_batch *out, void *stream);

/* Exhaustive program enumeration (BASELINE config 4).
 * Program rank r: pair k = bits [k*(ob+pb), (k+1)*(ob+pb)) of r, opcode = the
 * low ob bits, operand = the next pb bits.  Machine (r, x) is
 * init_config(P_r, [x]) (machine.py:289-309) with ell = s = 1, for every
 * input word x in [0, 2^w), run for at most tau_max steps.  Per program, one
 * record: bit 63 = every input reached a fixed point within tau_max; bits
 * 0..62 = sum over x of fmix32(x | halted<<8 | y0<<9 | y1<<10 | tau_h<<18)
 * (murmur3's 32-bit finaliser of a 32-bit key; y1 and tau_h count only when
 * written / halted).  records: uint64[count] device buffer; steps_total:
 * device counter that accumulates the applied machine-steps.  2 <= w <= 8,
 * tau_max < 2^14. */
typedef struct rasp_enum_params {
    uint32_t m;             /* instruction pairs */
    uint32_t opcode_bits;   /* ob */
    uint32_t operand_bits;  /* pb */
    uint32_t w;             /* word width, 2..8 */
    uint32_t n;             /* memory cells, >= 2m */
    uint32_t tau_max;
} rasp_enum_params;

int rasp_enumerate(const rasp_enum_params *p, uint64_t first_rank, uint64_t count,
                   uint64_t *records, unsigned long long *steps_total, void *stream);

/* Bucketed halting-time histogram (hypervisor.py:326-352): out[0..99] exact
 * tau_h, out[100] tau_h >= 100, out[101] EXHAUSTED count.  out: int64[102]
 * device buffer, overwritten. */
int rasp_histogram(const int8_t *status, const int64_t *tau_h, uint64_t d,
                   int64_t *out, void *stream);

/* Batch validation for run_batch (validate_config cursor ranges m:324-327 and
 * the word-range check hv:285-290).  out: int64[8] device buffer, overwritten:
 *   out[0..4] = count of words > 2^w-1 in iw, ac, M, u, y;
 *   out[5] = count of u[.][0] > ell;  out[6] = count of y[.][0] > s;  out[7] = 0. */
int rasp_validate(const rasp_params *p, const rasp_batch *b, int64_t *out, void *stream);

/* Word-width conversion between the reference's uint64 arrays and the
 * engine's natural-width arrays (the packing step of run_batch,
 * hypervisor.py:280-284, and its inverse when results are read back as
 * uint64).  Converts iw, ac, M, u, y from src->word_bytes to dst->word_bytes
 * (narrowing truncates: validate first with rasp_validate); status, steps and
 * tau_h are copied when both batches carry them at different addresses.
 * dst->word_bytes must hold w bits.  rasp_pack and rasp_unpack are the same
 * operation, named for the two directions a caller uses them in. */
int rasp_pack(const rasp_params *p, const rasp_batch *src, const rasp_batch *dst, void *stream);
int rasp_unpack(const rasp_params *p, const rasp_batch *src, const rasp_batch *dst, void *stream);

/* The k longest halting runs, for bb-search's report (cli.py:195-230): among
 * machines with status HALTED, the k largest tau_h, ties broken by the lower
 * machine index, in the order of sorted(best, reverse=True) over the
 * reference's (tau_h, -index) heap.  out_index/out_tau: int64[k] device
 * buffers; entries past the number of halted machines are -1.  tau_max bounds
 * every halted tau_h (rasp_run's contract) and sets the radix-select depth.
 * k <= 2048.  workspace: device buffer of rasp_topk_workspace_bytes(k). */
size_t rasp_topk_workspace_bytes(uint32_t k);
int rasp_topk(const int8_t *status, const int64_t *tau_h, uint64_t d, int64_t tau_max, uint32_t k,
              int64_t *out_index, int64_t *out_tau, void *workspace, size_t workspace_bytes, void *stream);

/* Post-run collectives of a sharded run on an NCCL
 * communicator (ncclComm_t passed as void*).  NCCL is resolved at run time from
 * the process (the libnccl.so.2 torch loaded) or $RASP_NCCL_LIBRARY.
 * Shard k of a d_total-machine batch over W ranks is the contiguous block
 * [k*ceil(d_total/W), (k+1)*ceil(d_total/W)) clipped to d_total. */
int rasp_nccl_unique_id(void *id_out /* 128 bytes */);
int rasp_nccl_comm_init(int nranks, const void *id, int rank, void **comm_out);
int rasp_nccl_comm_destroy(void *comm);
/* In-place sum over ranks of `count` int64 device counters (the 102-bucket
 * histogram plus whatever totals the caller appends). */
int rasp_shard_allreduce(void *comm, int64_t *counters, uint64_t count, void *stream);
/* Gather every rank's shard fields into `full` (d_total machines) on `root`;
 * `full` is ignored on other ranks.  fields: a mask of RASP_GATHER_*. */
#define RASP_GATHER_RESULTS 1u   /* status, steps, tau_h */
#define RASP_GATHER_OUTPUT 2u    /* y */
#define RASP_GATHER_CONFIG 4u    /* iw, ac, M, u */
int rasp_shard_gather(void *comm, int root, const rasp_params *p, uint64_t d_total, const rasp_batch *shard,
                      const rasp_batch *full, uint32_t fields, void *stream);

/* Text for a RASP_E* code, and the last CUDA error string seen by this library. */
const char *rasp_error_string(int code);
const char *rasp_last_cuda_error(void);

/* 1 if this library was built with the kernel bounds/ownership checks
 * (-DRASP_CHECKED=1, the checked build tests/test_checked_build.py runs). */
int rasp_checked_build(void);

/* ABI version (RASP_ABI_VERSION) of the loaded library. */
int rasp_abi_version(void);

/* Cumulative number of kernels this library has launched (all threads). */
unsigned long long rasp_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* RASPVISOR_B200_H */
