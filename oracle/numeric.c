/* CPU numeric oracle — TEST INFRASTRUCTURE ONLY (see numeric.h for the
 * contract, the parity pinning and who may call it).
 *
 * Layout of this file:
 *   premises()       restates CheckCollective        semantics.cc:203-257
 *   apply_bits()     restates ApplyCollectiveInPlace semantics.cc:259-310
 *   group_tasks()    data meaning of each rule over the row chunking
 *   oracle_execute() the RunLowered fold               dsl.cc:142-164
 */
#define _GNU_SOURCE
#include "numeric.h"

#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

enum { OP_AR = 0, OP_RS = 1, OP_AG = 2, OP_REDUCE = 3, OP_BCAST = 4 };
enum {
  V_NONE = 0, V_GROUP_TOO_SMALL, V_OUT_OF_RANGE, V_ROWSET_MISMATCH, V_CHUNK_OVERLAP,
  V_INDIVISIBLE, V_ROWSET_OVERLAP, V_BCAST_MISSING, V_BCAST_NO_NEW
};

#define MAXK 64

/* held[d*K + r]: column mask of device d's row r (0 = row not held). */
typedef struct {
  int K;
  uint64_t held[MAXK * MAXK];
} State;

static int row_count(const State* st, int d) {
  int n = 0;
  for (int r = 0; r < st->K; ++r) n += st->held[d * st->K + r] != 0;
  return n;
}

/* semantics.cc:156-191 (RowSetsEqual, RowsPairwiseDisjoint). */
static int reduce_premise(const State* st, const int32_t* g, int n) {
  const int K = st->K;
  for (int r = 0; r < K; ++r) {
    const int lead = st->held[g[0] * K + r] != 0;
    for (int m = 1; m < n; ++m)
      if ((st->held[g[m] * K + r] != 0) != lead) return V_ROWSET_MISMATCH;
  }
  for (int r = 0; r < K; ++r) {
    uint64_t seen = 0;
    for (int m = 0; m < n; ++m) {
      const uint64_t b = st->held[g[m] * K + r];
      if (b & seen) return V_CHUNK_OVERLAP;
      seen |= b;
    }
  }
  return V_NONE;
}

/* semantics.cc:203-257. */
static int premises(const State* st, const int32_t* g, int n, int op) {
  const int K = st->K;
  if (n < 2) return V_GROUP_TOO_SMALL;
  for (int m = 0; m < n; ++m)
    if (g[m] < 0 || g[m] >= K) return V_OUT_OF_RANGE;
  switch (op) {
    case OP_AR:
    case OP_REDUCE:
      return reduce_premise(st, g, n);
    case OP_RS: {
      int v = reduce_premise(st, g, n);
      if (v) return v;
      return row_count(st, g[0]) % n ? V_INDIVISIBLE : V_NONE;
    }
    case OP_AG:
      for (int r = 0; r < K; ++r) {
        int holders = 0;
        for (int m = 0; m < n; ++m) holders += st->held[g[m] * K + r] != 0;
        if (holders > 1) return V_ROWSET_OVERLAP;
      }
      return V_NONE;
    case OP_BCAST: {
      int gains = 0;
      for (int m = 1; m < n; ++m) {
        int equal = 1;
        for (int r = 0; r < K; ++r) {
          const uint64_t root = st->held[g[0] * K + r], mem = st->held[g[m] * K + r];
          if (mem & ~root) return V_BCAST_MISSING;
          equal &= mem == root;
        }
        gains |= !equal;
      }
      return gains ? V_NONE : V_BCAST_NO_NEW;
    }
    default:
      return -1;
  }
}

/* semantics.cc:259-310 (postconditions). Premises already hold. */
static void apply_bits(State* st, const int32_t* g, int n, int op) {
  const int K = st->K;
  uint64_t uni[MAXK];
  for (int r = 0; r < K; ++r) {
    uni[r] = 0;
    for (int m = 0; m < n; ++m) uni[r] |= st->held[g[m] * K + r];
  }
  switch (op) {
    case OP_AR:
    case OP_AG:
      for (int m = 0; m < n; ++m) memcpy(&st->held[g[m] * K], uni, sizeof(uint64_t) * K);
      break;
    case OP_RS: {
      int rows[MAXK], cnt = 0;
      for (int r = 0; r < K; ++r)
        if (st->held[g[0] * K + r]) rows[cnt++] = r;
      const int run = cnt / n;
      for (int m = 0; m < n; ++m) {
        memcpy(&st->held[g[m] * K], uni, sizeof(uint64_t) * K);
        for (int i = 0; i < cnt; ++i)
          if (i < m * run || i >= (m + 1) * run) st->held[g[m] * K + rows[i]] = 0;
      }
      break;
    }
    case OP_REDUCE:
      for (int m = 1; m < n; ++m) memset(&st->held[g[m] * K], 0, sizeof(uint64_t) * K);
      memcpy(&st->held[g[0] * K], uni, sizeof(uint64_t) * K);
      break;
    case OP_BCAST:
      for (int m = 1; m < n; ++m)
        memcpy(&st->held[g[m] * K], &st->held[g[0] * K], sizeof(uint64_t) * K);
      break;
  }
}

/* ------------------------------------------------------------ data tasks */

typedef struct {
  size_t lo, hi;    /* element range (same offsets on every buffer) */
  int nsrc, ndst;
  int src[MAXK];    /* device ids, summation order */
  int dst[MAXK];
} Task;

typedef struct {
  Task* v;
  size_t n, cap;
} TaskList;

static void push_task(TaskList* tl, size_t lo, size_t hi, const int* src, int nsrc,
                      const int* dst, int ndst) {
  if (hi <= lo || ndst == 0) return;
  if (tl->n == tl->cap) {
    tl->cap = tl->cap ? tl->cap * 2 : 64;
    tl->v = (Task*)realloc(tl->v, tl->cap * sizeof(Task));
  }
  Task* t = &tl->v[tl->n++];
  t->lo = lo;
  t->hi = hi;
  t->nsrc = nsrc;
  t->ndst = ndst;
  memcpy(t->src, src, sizeof(int) * nsrc);
  memcpy(t->dst, dst, sizeof(int) * ndst);
}

static size_t row_lo(int r, size_t N, int K) { return (size_t)(((unsigned __int128)r * N) / K); }

/* Data meaning of one group's rule, emitted from the PRE-state `st`. */
static void group_tasks(const State* st, const int32_t* g, int n, int op, size_t N,
                        TaskList* tl) {
  const int K = st->K;
  int all[MAXK];
  for (int m = 0; m < n; ++m) all[m] = g[m];
  switch (op) {
    case OP_AR: /* every member <- ordered sum over R, R = held rows (equal) */
      for (int r = 0; r < K; ++r)
        if (st->held[g[0] * K + r]) push_task(tl, row_lo(r, N, K), row_lo(r + 1, N, K), all, n, all, n);
      break;
    case OP_REDUCE: /* root <- ordered sum over R; others become empty */
      for (int r = 0; r < K; ++r)
        if (st->held[g[0] * K + r]) push_task(tl, row_lo(r, N, K), row_lo(r + 1, N, K), all, n, all, 1);
      break;
    case OP_RS: { /* member m <- ordered sum over its run of R */
      int rows[MAXK], cnt = 0;
      for (int r = 0; r < K; ++r)
        if (st->held[g[0] * K + r]) rows[cnt++] = r;
      const int run = cnt / n;
      for (int i = 0; i < cnt; ++i) {
        const int m = i / run;
        push_task(tl, row_lo(rows[i], N, K), row_lo(rows[i] + 1, N, K), all, n, &all[m], 1);
      }
      break;
    }
    case OP_AG: /* each held row copied from its unique holder to the others */
      for (int r = 0; r < K; ++r) {
        int holder = -1, others[MAXK], no = 0;
        for (int m = 0; m < n; ++m) {
          if (st->held[g[m] * K + r]) holder = g[m];
          else others[no++] = g[m];
        }
        if (holder >= 0) push_task(tl, row_lo(r, N, K), row_lo(r + 1, N, K), &holder, 1, others, no);
      }
      break;
    case OP_BCAST: /* every root row overwrites that row on every member */
      for (int r = 0; r < K; ++r)
        if (st->held[g[0] * K + r]) push_task(tl, row_lo(r, N, K), row_lo(r + 1, N, K), all, 1, &all[1], n - 1);
      break;
  }
}

static inline float bf16_to_f32(uint16_t h) {
  uint32_t u = (uint32_t)h << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

static inline uint16_t f32_to_bf16_rne(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return (uint16_t)((u >> 16) | 0x40); /* quiet NaN */
  u += 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

#define BLK 2048

static void run_range(const Task* t, size_t lo, size_t hi, int dtype, void* const* bufs) {
  if (t->nsrc == 1) { /* copy: raw bits */
    const size_t es = dtype == ORACLE_BF16 ? 2 : 4;
    const char* s = (const char*)bufs[t->src[0]];
    for (int d = 0; d < t->ndst; ++d)
      memmove((char*)bufs[t->dst[d]] + lo * es, s + lo * es, (hi - lo) * es);
    return;
  }
  for (size_t b = lo; b < hi; b += BLK) {
    const size_t e = hi - b < BLK ? hi - b : BLK;
    if (dtype == ORACLE_F32) {
      float acc[BLK];
      const float* s0 = (const float*)bufs[t->src[0]] + b;
      for (size_t j = 0; j < e; ++j) acc[j] = s0[j];
      for (int i = 1; i < t->nsrc; ++i) {
        const float* si = (const float*)bufs[t->src[i]] + b;
        for (size_t j = 0; j < e; ++j) acc[j] = acc[j] + si[j];
      }
      for (int d = 0; d < t->ndst; ++d) memcpy((float*)bufs[t->dst[d]] + b, acc, e * 4);
    } else if (dtype == ORACLE_BF16) {
      float acc[BLK];
      uint16_t out[BLK];
      const uint16_t* s0 = (const uint16_t*)bufs[t->src[0]] + b;
      for (size_t j = 0; j < e; ++j) acc[j] = bf16_to_f32(s0[j]);
      for (int i = 1; i < t->nsrc; ++i) {
        const uint16_t* si = (const uint16_t*)bufs[t->src[i]] + b;
        for (size_t j = 0; j < e; ++j) acc[j] = acc[j] + bf16_to_f32(si[j]);
      }
      for (size_t j = 0; j < e; ++j) out[j] = f32_to_bf16_rne(acc[j]);
      for (int d = 0; d < t->ndst; ++d) memcpy((uint16_t*)bufs[t->dst[d]] + b, out, e * 2);
    } else {
      uint32_t acc[BLK];
      const uint32_t* s0 = (const uint32_t*)bufs[t->src[0]] + b;
      for (size_t j = 0; j < e; ++j) acc[j] = s0[j];
      for (int i = 1; i < t->nsrc; ++i) {
        const uint32_t* si = (const uint32_t*)bufs[t->src[i]] + b;
        for (size_t j = 0; j < e; ++j) acc[j] += si[j];
      }
      for (int d = 0; d < t->ndst; ++d) memcpy((uint32_t*)bufs[t->dst[d]] + b, acc, e * 4);
    }
  }
}

typedef struct {
  const TaskList* tl;
  const size_t* prefix; /* prefix[i] = elements before task i */
  size_t begin, end;    /* this worker's slice of the concatenated space */
  int dtype;
  void* const* bufs;
} Work;

static void* worker(void* arg) {
  const Work* w = (const Work*)arg;
  for (size_t i = 0; i < w->tl->n; ++i) {
    const size_t t0 = w->prefix[i], t1 = w->prefix[i + 1];
    const size_t a = t0 > w->begin ? t0 : w->begin, b = t1 < w->end ? t1 : w->end;
    if (a >= b) continue;
    const Task* t = &w->tl->v[i];
    run_range(t, t->lo + (a - t0), t->lo + (b - t0), w->dtype, w->bufs);
  }
  return NULL;
}

/* Elements of one task are processed by exactly one thread each, which is
 * what makes in-place sums/copies safe (every element reads all its sources
 * before writing its destinations). */
static void run_tasks(const TaskList* tl, int dtype, void* const* bufs, int nthreads) {
  if (tl->n == 0) return;
  size_t* prefix = (size_t*)malloc((tl->n + 1) * sizeof(size_t));
  prefix[0] = 0;
  for (size_t i = 0; i < tl->n; ++i) prefix[i + 1] = prefix[i] + (tl->v[i].hi - tl->v[i].lo);
  const size_t total = prefix[tl->n];
  int T = nthreads;
  if ((size_t)T > total / 65536 + 1) T = (int)(total / 65536 + 1);
  if (T < 1) T = 1;
  Work* ws = (Work*)calloc((size_t)T, sizeof(Work));
  pthread_t* th = (pthread_t*)calloc((size_t)T, sizeof(pthread_t));
  for (int i = 0; i < T; ++i) {
    ws[i].tl = tl;
    ws[i].prefix = prefix;
    ws[i].begin = total * (size_t)i / (size_t)T;
    ws[i].end = total * (size_t)(i + 1) / (size_t)T;
    ws[i].dtype = dtype;
    ws[i].bufs = bufs;
  }
  for (int i = 1; i < T; ++i) pthread_create(&th[i], NULL, worker, &ws[i]);
  worker(&ws[0]);
  for (int i = 1; i < T; ++i) pthread_join(th[i], NULL);
  free(th);
  free(ws);
  free(prefix);
}

int oracle_hardware_threads(void) {
  long n = sysconf(_SC_NPROCESSORS_ONLN);
  return n > 0 ? (int)n : 1;
}

static int fold(int K, int num_steps, const int32_t* step_op, const int32_t* sgp,
                const int32_t* gmp, const int32_t* members, size_t elems, int dtype,
                void* const* bufs, int nthreads, int* fail_step, int* fail_violation,
                uint64_t* held_out) {
  if (K < 1 || K > MAXK || num_steps < 0) return 3;
  if (nthreads <= 0) nthreads = oracle_hardware_threads();
  State* st = (State*)calloc(1, sizeof(State));
  st->K = K;
  for (int d = 0; d < K; ++d) /* InitialContext, semantics.cc:128-136 */
    for (int r = 0; r < K; ++r) st->held[d * K + r] = 1ull << d;
  TaskList tl = {0};
  int rc = 0;
  for (int s = 0; s < num_steps && rc == 0; ++s) {
    const int op = step_op[s];
    if (op < 0 || op > 4) { rc = 3; break; }
    if (sgp[s + 1] <= sgp[s]) { rc = 3; break; } /* dsl.cc:147-150 */
    tl.n = 0;
    for (int g = sgp[s]; g < sgp[s + 1]; ++g) {
      const int32_t* grp = members + gmp[g];
      const int n = gmp[g + 1] - gmp[g];
      const int v = premises(st, grp, n, op);
      if (v != V_NONE) {
        if (fail_step) *fail_step = s;
        if (fail_violation) *fail_violation = v;
        rc = 9;
        break;
      }
      if (bufs) {
        /* Groups of a step are disjoint (dsl.h:104-107), so emitting from the
         * state after earlier groups equals emitting from the step's pre-state;
         * run the pending tasks first if this group touches an earlier one. */
        group_tasks(st, grp, n, op, elems, &tl);
        run_tasks(&tl, dtype, bufs, nthreads);
        tl.n = 0;
      }
      apply_bits(st, grp, n, op);
    }
  }
  if (rc == 0 && held_out) memcpy(held_out, st->held, sizeof(uint64_t) * (size_t)K * K);
  free(tl.v);
  free(st);
  return rc;
}

int oracle_execute(int K, int num_steps, const int32_t* step_op, const int32_t* step_group_ptr,
                   const int32_t* group_member_ptr, const int32_t* members, size_t elems,
                   int dtype, void* const* bufs, int nthreads, int* fail_step,
                   int* fail_violation, uint64_t* held_out) {
  if (!bufs || dtype < 0 || dtype > 2) return 3;
  return fold(K, num_steps, step_op, step_group_ptr, group_member_ptr, members, elems, dtype,
              bufs, nthreads, fail_step, fail_violation, held_out);
}

int oracle_check(int K, int num_steps, const int32_t* step_op, const int32_t* step_group_ptr,
                 const int32_t* group_member_ptr, const int32_t* members, int* fail_step,
                 int* fail_violation, uint64_t* held_out) {
  return fold(K, num_steps, step_op, step_group_ptr, group_member_ptr, members, 0, 0, NULL, 1,
              fail_step, fail_violation, held_out);
}
