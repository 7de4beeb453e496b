/*
 * rasp_oracle.c -- CPU restatement of the reference's batch transition map.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker and the CPU
 * baseline ("port") for the B200 hot path.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  The product
 * path (paper_2604_12902_b200) never links or calls it.
 *
 * It restates, in C over the reference's own uint64 SoA layout:
 *   oracle_advance  <- raspvisor/hypervisor.py:72-125   (_advance)
 *   oracle_worker   <- raspvisor/hypervisor.py:128-164  (_worker)
 *   oracle_run      <- raspvisor/hypervisor.py:295-314  (the W-thread
 *                      striped dispatch inside run_batch)
 * Semantics of one step follow raspvisor/machine.py:169-211
 * (step_reference); the five-candidate fixedness test is hv:115-116.
 *
 * Parity pin: tests/test_oracle_golden.py checks every function here
 * against fixtures produced by the reference itself
 * (tests/golden/make_golden.py imports /root/reference/pkg/src).
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef uint64_t u64;
typedef int64_t i64;

enum { RUNNING = 0, HALTED = 1, EXHAUSTED = 2 };

typedef struct {
    u64 *iw, *ac, *M, *u, *y;     /* [d], [d], [d,n], [d,ell+1], [d,s+1] */
    int8_t *status;               /* [d] */
    i64 *steps, *tau_h;           /* [d] */
    i64 d;
    u64 wmask, n, ell, s;
} oracle_state;

/* x mod n with a 32-bit divide when both fit (the same value; 64-bit
 * division is several times slower on x86, which LLVM -- and so the numba
 * reference -- also special-cases). */
static inline u64 umod(u64 x, u64 n)
{
    if (((x | n) >> 32) == 0) return (uint32_t)x % (uint32_t)n;
    return x % n;
}

/* hypervisor.py:72-125.  Returns 1 iff VM j is at a fixed point; otherwise
 * applies one step when do_apply. */
static inline int oracle_advance(const oracle_state *st, i64 j, int do_apply)
{
    const u64 n = st->n, wmask = st->wmask;
    u64 *Mj = st->M + (size_t)j * n;
    u64 *uj = st->u + (size_t)j * (st->ell + 1);
    u64 *yj = st->y + (size_t)j * (st->s + 1);
    const u64 i0 = st->iw[j];
    const u64 a0 = st->ac[j];
    const u64 o = Mj[umod(i0, n)];                       /* hv:78 */
    const u64 jw = Mj[umod((i0 + 1) & wmask, n)];        /* hv:79 */
    const u64 jn = umod(jw, n);                          /* hv:80 */
    const u64 mj = Mj[jn];                          /* hv:81 */
    const u64 u0 = uj[0], y0 = yj[0];

    u64 ni = (i0 + 2) & wmask;                      /* hv:85 */
    u64 na = a0, nm = mj, nu0 = u0, ny0 = y0;
    int write_out = 0;
    switch (o) {                                    /* hv:91-113 */
    case 1: na = jw; break;                         /* LOD */
    case 2: na = (a0 + mj) & wmask; break;          /* ADD */
    case 3: na = (a0 * mj) & wmask; break;          /* MUL (wraps mod 2^64 first, as numpy) */
    case 4: nm = a0; break;                         /* STO */
    case 5: if (a0 != 0) ni = jw; break;            /* BNZ */
    case 6:                                         /* RD */
        if (u0 < st->ell) { nm = uj[u0 + 1]; nu0 = u0 + 1; }
        else ni = i0;
        break;
    case 7:                                         /* PRI */
        if (y0 < st->s) { ny0 = y0 + 1; write_out = 1; }
        break;
    default: ni = i0;
    }
    if (ni == i0 && na == a0 && nm == mj && nu0 == u0 && ny0 == y0)  /* hv:115 */
        return 1;
    if (do_apply) {                                 /* hv:117-124 */
        st->iw[j] = ni;
        st->ac[j] = na;
        Mj[jn] = nm;
        uj[0] = nu0;
        if (write_out) yj[y0 + 1] = mj;
        yj[0] = ny0;
    }
    return 0;
}

/* One visit of machine j (the body of the `while applied < q` loop of
 * hypervisor.py:138-154): up to q steps with i, a and the cursors held in
 * locals, exactly the per-step logic of oracle_advance (hv:72-125).
 * Returns the new status (RUNNING if the visit ended on q). */
static int oracle_visit(const oracle_state *st, i64 j, i64 q, i64 tau_max)
{
    const u64 n = st->n, wmask = st->wmask, ell = st->ell, s = st->s;
    u64 *Mj = st->M + (size_t)j * n;
    u64 *uj = st->u + (size_t)j * (ell + 1);
    u64 *yj = st->y + (size_t)j * (s + 1);
    u64 i0 = st->iw[j], a0 = st->ac[j], u0 = uj[0], y0 = yj[0];
    i64 steps = st->steps[j];
    int status = RUNNING;
    for (i64 applied = 0; applied < q; ++applied) {
        const u64 o = Mj[umod(i0, n)];
        const u64 jw = Mj[umod((i0 + 1) & wmask, n)];
        const u64 jn = umod(jw, n);
        const u64 mj = Mj[jn];
        u64 ni = (i0 + 2) & wmask, na = a0, nm = mj, nu0 = u0, ny0 = y0;
        int write_out = 0;
        switch (o) {
        case 1: na = jw; break;
        case 2: na = (a0 + mj) & wmask; break;
        case 3: na = (a0 * mj) & wmask; break;
        case 4: nm = a0; break;
        case 5: if (a0 != 0) ni = jw; break;
        case 6:
            if (u0 < ell) { nm = uj[u0 + 1]; nu0 = u0 + 1; }
            else ni = i0;
            break;
        case 7:
            if (y0 < s) { ny0 = y0 + 1; write_out = 1; }
            break;
        default: ni = i0;
        }
        const int fixed = ni == i0 && na == a0 && nm == mj && nu0 == u0 && ny0 == y0;
        if (steps >= tau_max) {                      /* hv:140-148: probe only */
            status = fixed ? HALTED : EXHAUSTED;
            break;
        }
        if (fixed) { status = HALTED; break; }       /* hv:149-152 */
        i0 = ni; a0 = na; Mj[jn] = nm; u0 = nu0;     /* hv:117-124 */
        if (write_out) yj[y0 + 1] = mj;
        y0 = ny0;
        ++steps;                                     /* hv:153 */
    }
    st->iw[j] = i0; st->ac[j] = a0; uj[0] = u0; yj[0] = y0;
    st->steps[j] = steps;
    if (status == HALTED) st->tau_h[j] = steps;
    if (status != RUNNING) st->status[j] = (int8_t)status;
    return status;
}

/* hypervisor.py:128-164: stripe {g + kW}, `rounds` sweeps of at most q
 * steps per visit, budget probe, final classification sweep. */
void oracle_worker(const oracle_state *st, i64 g, i64 W, i64 q, i64 rounds, i64 tau_max)
{
    const i64 d = st->d;
    const i64 stripe = d > g ? (d - g + W - 1) / W : 0;
    for (i64 r = 0; r < rounds; ++r) {
        for (i64 k = 0; k < stripe; ++k) {
            const i64 j = g + k * W;
            if (st->status[j] != RUNNING) continue;
            oracle_visit(st, j, q, tau_max);
        }
    }
    for (i64 k = 0; k < stripe; ++k) {                   /* hv:157-164 */
        const i64 j = g + k * W;
        if (st->status[j] == RUNNING) {
            if (oracle_advance(st, j, 0)) {
                st->status[j] = HALTED;
                st->tau_h[j] = st->steps[j];
            } else {
                st->status[j] = EXHAUSTED;
            }
        }
    }
}

typedef struct {
    const oracle_state *st;
    i64 g, W, q, rounds, tau_max;
} worker_arg;

static void *worker_main(void *p)
{
    const worker_arg *a = (const worker_arg *)p;
    oracle_worker(a->st, a->g, a->W, a->q, a->rounds, a->tau_max);
    return NULL;
}

/* hypervisor.py:295-314: W = min(W, d) interleaved stripes, one thread each,
 * epoch q, rounds = ceil(tau_max / q).  Returns 0 on success. */
int oracle_run(u64 *iw, u64 *ac, u64 *M, u64 *u, u64 *y, int8_t *status,
               i64 *steps, i64 *tau_h, i64 d, u64 wmask, u64 n, u64 ell, u64 s,
               i64 tau_max, i64 q, i64 W)
{
    if (d <= 0) return 0;
    if (q < 1 || tau_max < 0 || n < 2) return -1;
    if (W < 1) W = 1;
    if (W > d) W = d;
    oracle_state st = {iw, ac, M, u, y, status, steps, tau_h, d, wmask, n, ell, s};
    const i64 rounds = (tau_max + q - 1) / q;
    if (W == 1) {
        oracle_worker(&st, 0, 1, q, rounds, tau_max);
        return 0;
    }
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)W);
    worker_arg *args = (worker_arg *)malloc(sizeof(worker_arg) * (size_t)W);
    if (!th || !args) { free(th); free(args); return -2; }
    i64 started = 0;
    for (i64 g = 0; g < W; ++g) {
        args[g] = (worker_arg){&st, g, W, q, rounds, tau_max};
        if (pthread_create(&th[g], NULL, worker_main, &args[g]) != 0) break;
        ++started;
    }
    /* any stripe whose thread failed to start runs here, serially */
    for (i64 g = started; g < W; ++g) worker_main(&args[g]);
    for (i64 g = 0; g < started; ++g) pthread_join(th[g], NULL);
    free(th);
    free(args);
    return 0;
}

/* Single step of one config held in caller arrays (machine.py:169-211).
 * Writes the successor into the same arrays when not fixed; returns 1 iff
 * the config is a fixed point.  Used by tests to cross-check KATs. */
int oracle_step(u64 *i, u64 *a, u64 *M, u64 *u, u64 *y,
                u64 wmask, u64 n, u64 ell, u64 s)
{
    int8_t status = 0;
    i64 steps = 0, tau = -1;
    oracle_state st = {i, a, M, u, y, &status, &steps, &tau, 1, wmask, n, ell, s};
    return oracle_advance(&st, 0, 1);
}

/* ---- exhaustive enumeration (BASELINE config 4) -------------------------------
 * Same machine semantics (oracle_advance) driven per (program rank, input x),
 * run_to_fixpoint style (machine.py:336-357) with budget tau; the per-program
 * record definition mirrors include/raspvisor_b200.h (rasp_enumerate). */
/* murmur3's 32-bit finaliser: the per-input fingerprint of a record */
static uint32_t fmix32(uint32_t h)
{
    h ^= h >> 16;
    h *= 0x85ebca6bu;
    h ^= h >> 13;
    h *= 0xc2b2ae35u;
    h ^= h >> 16;
    return h;
}

typedef struct {
    u64 m, ob, pb, w, n, tau, first, count;
    u64 *records;
    u64 steps;
    i64 g, W;
} enum_arg;

static void *enum_main(void *p)
{
    enum_arg *a = (enum_arg *)p;
    const u64 n = a->n, mask = (a->w == 64) ? ~0ull : ((1ull << a->w) - 1);
    const u64 pw = a->ob + a->pb;
    u64 *M = (u64 *)calloc(n, sizeof(u64));
    u64 iw, ac, u[2], y[2];
    int8_t st;
    i64 steps, tau_h;
    oracle_state s = {&iw, &ac, M, u, y, &st, &steps, &tau_h, 1, mask, n, 1, 1};
    a->steps = 0;
    for (u64 pi = (u64)a->g; pi < a->count; pi += (u64)a->W) {
        const u64 r = a->first + pi;
        u64 sum = 0;
        int all = 1;
        for (u64 x = 0; x <= mask && x < 256; ++x) {
            memset(M, 0, n * sizeof(u64));
            for (u64 k = 0; k < a->m && 2 * k + 1 < n; ++k) {
                const u64 pair = (r >> (k * pw)) & ((1ull << pw) - 1);
                M[2 * k] = pair & ((1ull << a->ob) - 1);
                M[2 * k + 1] = pair >> a->ob;
            }
            iw = 0; ac = 0; u[0] = 0; u[1] = x; y[0] = 0; y[1] = 0;
            u64 t = 0;
            int halted = 0;
            for (;;) {                           /* run_to_fixpoint, m:345-357 */
                if (oracle_advance(&s, 0, 0)) { halted = 1; break; }
                if (t == a->tau) break;
                oracle_advance(&s, 0, 1);
                ++t;
            }
            a->steps += t;
            if (!halted) all = 0;
            const u64 key = x | ((u64)halted << 8) | (y[0] << 9) | ((y[0] ? y[1] : 0) << 10) |
                            ((u64)(halted ? t : 0) << 18);
            sum += fmix32((uint32_t)key);
        }
        a->records[pi] = ((u64)all << 63) | (sum & 0x7fffffffffffffffull);
    }
    free(M);
    return NULL;
}

/* records[count]; returns the applied machine-steps. */
u64 oracle_enumerate(u64 m, u64 ob, u64 pb, u64 w, u64 n, u64 tau, u64 first, u64 count,
                     u64 *records, i64 threads)
{
    if (threads < 1) threads = 1;
    enum_arg *args = (enum_arg *)calloc((size_t)threads, sizeof(enum_arg));
    pthread_t *th = (pthread_t *)calloc((size_t)threads, sizeof(pthread_t));
    for (i64 g = 0; g < threads; ++g) {
        args[g] = (enum_arg){m, ob, pb, w, n, tau, first, count, records, 0, g, threads};
        if (threads > 1) pthread_create(&th[g], NULL, enum_main, &args[g]);
        else enum_main(&args[g]);
    }
    u64 total = 0;
    for (i64 g = 0; g < threads; ++g) {
        if (threads > 1) pthread_join(th[g], NULL);
        total += args[g].steps;
    }
    free(args);
    free(th);
    return total;
}
