/*
 * oracle.c -- plain, slow, sequential CPU oracle for the GTaP hot path.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product path (paper_2604_05982_b200/, include/gtap.h) never links,
 * imports or calls it, and this file shares no code, header, table or
 * constant with the CUDA path.
 *
 * Every function restates what the paper (reference/PAPER.md, cited "P:n" =
 * line n) defines, written the obvious way: plain recursion, plain loops,
 * fp64 accumulation where the paper leaves floating point open. Readings of
 * ambiguous passages are the ones listed in DESIGN.md "Readings".
 *
 * Pins (tests/test_oracle_*.py, -m "not gpu"):
 *   fib        -- iterative F(n), OEIS/SPEC values, closed-form call counts
 *   mergesort  -- numpy sort, exhaustive permutations, closed-form task count
 *   spmv       -- dense fp64 matmul on tiny matrices, identity / ones rows
 *   bfs        -- all-pairs shortest paths (scipy) on every 5-vertex graph,
 *                 Graph500-style validity on RMAT graphs
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ fib */
/*
 * P:1023-1033 (Prog. fib, §5.1.2):
 *     if (n < 2) return n;  a = fib(n-1);  b = fib(n-2);  taskwait;  return a+b;
 * Every call is one task ("we disable the cutoff and spawn a task at every
 * recursive call"). Invocations follow the transformed state machine
 * (P:1168-1190): a call with n < 2 finishes in case 0 (1 invocation); any
 * other call runs case 0 (spawn + prepare_for_join) and case 1 (load the two
 * child results, finish) -- 2 invocations.
 */
static int64_t fib_rec(int32_t n, int64_t *calls, int64_t *invocations)
{
    *calls += 1;
    if (n < 2) {
        *invocations += 1;
        return n;
    }
    int64_t a = fib_rec(n - 1, calls, invocations);
    int64_t b = fib_rec(n - 2, calls, invocations);
    *invocations += 2;
    return a + b;
}

int oracle_fib(int32_t n, int64_t *value, int64_t *calls, int64_t *invocations)
{
    if (n < 0 || n > 92) return -1;
    *calls = 0;
    *invocations = 0;
    *value = fib_rec(n, calls, invocations);
    return 0;
}

/*
 * fib with a cutoff (EPAQ experiment): a task
 * with n < cutoff runs the serial recursion ("tasks that reach the cutoff
 * execute additional serial work") and finishes; otherwise it spawns
 * fib(n-1), fib(n-2), joins and returns a + b. cutoff <= 2 is the no-cutoff
 * program above. Also counts the serial calls made inside cutoff tasks.
 */
static int64_t fib_serial(int32_t n, int64_t *serial_calls)
{
    *serial_calls += 1;
    if (n < 2) return n;
    return fib_serial(n - 1, serial_calls) + fib_serial(n - 2, serial_calls);
}

static int64_t fib_cut_rec(int32_t n, int32_t cutoff, int64_t *tasks, int64_t *invocations, int64_t *serial)
{
    *tasks += 1;
    if (n < cutoff || n < 2) {
        *invocations += 1;
        return fib_serial(n, serial);
    }
    int64_t a = fib_cut_rec(n - 1, cutoff, tasks, invocations, serial);
    int64_t b = fib_cut_rec(n - 2, cutoff, tasks, invocations, serial);
    *invocations += 2;
    return a + b;
}

int oracle_fib_cutoff(int32_t n, int32_t cutoff, int64_t *value, int64_t *tasks, int64_t *invocations,
                      int64_t *serial_calls)
{
    if (n < 0 || n > 92 || cutoff < 0) return -1;
    *tasks = *invocations = *serial_calls = 0;
    *value = fib_cut_rec(n, cutoff, tasks, invocations, serial_calls);
    return 0;
}

/* ------------------------------------------------------- synthetic trees */
/*
 * Synthetic tree benchmark (§6.3): "Each node in a tree
 * corresponds to one task. A task spawns child tasks (if any), performs
 * taskwait, and then executes do_memory_and_compute"; the work is
 * `mem_ops` pseudo-random 64-bit global loads and `compute_iters` FP64 FMAs
 * (P:611). Full binary tree of depth D: 2^(D+1) - 1 tasks. Pruned
 * B-ary tree (B = 3): at depth d each child is generated with probability
 * p(d) = 1 - d/D. Readings (R27):
 *   - node ids: full tree heap ids (root 1, children 2i, 2i+1); B-ary ids
 *     (root 0, children B*i + 1 + k); a child exists iff
 *     mix(seed ^ child_id) >> 11 < floor((D - d) * 2^53 / D) (counter-based:
 *     the shape does not depend on the schedule);
 *   - do_memory_and_compute(id) = sum_i buf[mix(id * G + i) mod len]
 *     + the bits of the final value of each of the min(64, compute_iters)
 *     independent FMA chains (chain c: f = 1 + ((id + c) & 1023) / 1024, then
 *     f = fma(f, 0.999999, 1e-7) repeated compute_iters / 64 (+1 for
 *     c < compute_iters mod 64) times, i.e. compute_iters FMAs in total),
 *     all mod 2^64; the run's value is the sum over all nodes.
 */
static uint64_t t_mix(uint64_t z)
{
    z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 27; z *= 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static uint64_t tree_work(uint64_t id, const uint64_t *buf, uint64_t len, int64_t mem_ops, int64_t compute_iters)
{
    uint64_t s = 0;
    for (int64_t i = 0; i < mem_ops; i++)
        s += buf[t_mix(id * 0x9E3779B97F4A7C15ull + (uint64_t)i) % len];
    for (int c = 0; c < 64 && c < compute_iters; c++) {
        double f = 1.0 + (double)((id + (uint64_t)c) & 1023u) / 1024.0;
        int64_t it = compute_iters / 64 + (c < compute_iters % 64 ? 1 : 0);
        for (int64_t j = 0; j < it; j++) f = fma(f, 0.999999, 1e-7);
        uint64_t bits;
        memcpy(&bits, &f, 8);
        s += bits;
    }
    return s;
}

typedef struct {
    const uint64_t *buf; uint64_t len; int64_t mem_ops, compute_iters;
    int32_t D, B, pruned; uint64_t seed;
    uint64_t total; int64_t tasks;
} tree_ctx;

static int tree_child_exists(const tree_ctx *t, uint64_t child, int32_t depth)
{   /* depth = the parent's depth d; p(d) = 1 - d/D */
    const uint64_t thr = (uint64_t)(((unsigned __int128)(uint64_t)(t->D - depth) << 53) / (uint64_t)t->D);
    return (t_mix(t->seed ^ child) >> 11) < thr;
}

static void tree_node(tree_ctx *t, uint64_t id, int32_t depth)
{
    t->tasks += 1;
    if (depth < t->D) {
        if (!t->pruned) {
            tree_node(t, 2 * id, depth + 1);
            tree_node(t, 2 * id + 1, depth + 1);
        } else {
            for (int k = 0; k < t->B; k++) {
                const uint64_t c = (uint64_t)t->B * id + 1 + (uint64_t)k;
                if (tree_child_exists(t, c, depth)) tree_node(t, c, depth + 1);
            }
        }
    }
    t->total += tree_work(id, t->buf, t->len, t->mem_ops, t->compute_iters);  /* after the join */
}

int oracle_tree(int32_t D, int32_t B, int32_t pruned, uint64_t seed, const uint64_t *buf, uint64_t len,
                int64_t mem_ops, int64_t compute_iters, uint64_t *total, int64_t *tasks)
{
    if (D < 0 || D > 40 || len == 0 || mem_ops < 0 || compute_iters < 0 || (pruned && (B < 1 || D < 1)))
        return -1;
    tree_ctx t = {buf, len, mem_ops, compute_iters, D, B, pruned, seed, 0, 0};
    tree_node(&t, pruned ? 0 : 1, 0);
    *total = t.total;
    *tasks = t.tasks;
    return 0;
}

/* ------------------------------------------------------------- N-Queens */
/*
 * N-Queens by bitmask backtracking with a cutoff depth (PAPER.md P:465,
 * "count solutions via bitmask-based backtracking with a fixed
 * cutoff depth (7)", no taskwait): a task at row r < cutoff spawns one child
 * task per free column of row r; a task at row >= cutoff counts the solutions
 * below it serially; the counts are summed (no join needed). Reading R25:
 * cols / left / right diagonals as bitmasks, the diagonals shifted per row.
 */
static int64_t nq_serial(int32_t n, int32_t row, uint32_t cols, uint32_t d1, uint32_t d2)
{
    if (row == n) return 1;
    const uint32_t full = (n >= 32) ? 0xFFFFFFFFu : ((1u << n) - 1u);
    uint32_t avail = ~(cols | d1 | d2) & full;
    int64_t c = 0;
    while (avail) {
        uint32_t bit = avail & (0u - avail);
        avail ^= bit;
        c += nq_serial(n, row + 1, cols | bit, (d1 | bit) << 1, (d2 | bit) >> 1);
    }
    return c;
}

static int64_t nq_task(int32_t n, int32_t cutoff, int32_t row, uint32_t cols, uint32_t d1, uint32_t d2,
                       int64_t *tasks)
{
    *tasks += 1;
    if (row == n || row >= cutoff) return nq_serial(n, row, cols, d1, d2);
    const uint32_t full = (n >= 32) ? 0xFFFFFFFFu : ((1u << n) - 1u);
    uint32_t avail = ~(cols | d1 | d2) & full;
    int64_t c = 0;
    while (avail) {
        uint32_t bit = avail & (0u - avail);
        avail ^= bit;
        c += nq_task(n, cutoff, row + 1, cols | bit, (d1 | bit) << 1, (d2 | bit) >> 1, tasks);
    }
    return c;
}

int oracle_nqueens(int32_t n, int32_t cutoff, int64_t *solutions, int64_t *tasks)
{
    if (n < 1 || n > 32 || cutoff < 0) return -1;
    *tasks = 0;
    *solutions = nq_task(n, cutoff, 0, 0u, 0u, 0u, tasks);
    return 0;
}

/* ------------------------------------------------------------ mergesort */
/*
 * P:153-165 (Prog. cutoff mergesort, §4.4) with the state machine of
 * P:59-74 (§4.2):
 *     if (right - left <= CUTOFF) { sequential_sort(data, left, right); return; }
 *     mid = (left + right) / 2;  fork ms(left, mid);  fork ms(mid, right);
 *     join;  merge(data, left, mid, right);
 * Readings (R14, R15): half-open [l, r); mid = l + (r - l) / 2;
 * sequential_sort = insertion sort; merge = two-pointer merge into scratch
 * taking the left element on ties, then copy back.
 * Tasks = calls; invocations: a leaf runs once, an internal node twice
 * (case 0 spawns, case 1 merges).
 */
static void insertion_sort(int32_t *a, int64_t l, int64_t r)
{
    for (int64_t i = l + 1; i < r; i++) {
        int32_t v = a[i];
        int64_t j = i - 1;
        while (j >= l && a[j] > v) {
            a[j + 1] = a[j];
            j--;
        }
        a[j + 1] = v;
    }
}

static void merge_runs(int32_t *a, int32_t *tmp, int64_t l, int64_t m, int64_t r)
{
    int64_t i = l, j = m, k = l;
    while (i < m && j < r) {
        if (a[j] < a[i]) tmp[k++] = a[j++];
        else             tmp[k++] = a[i++];
    }
    while (i < m) tmp[k++] = a[i++];
    while (j < r) tmp[k++] = a[j++];
    memcpy(a + l, tmp + l, (size_t)(r - l) * sizeof(int32_t));
}

static void ms_rec(int32_t *a, int32_t *tmp, int64_t l, int64_t r, int64_t cutoff,
                   int64_t *tasks, int64_t *invocations)
{
    *tasks += 1;
    if (r - l <= cutoff) {
        insertion_sort(a, l, r);
        *invocations += 1;
        return;
    }
    int64_t m = l + (r - l) / 2;
    ms_rec(a, tmp, l, m, cutoff, tasks, invocations);
    ms_rec(a, tmp, m, r, cutoff, tasks, invocations);
    merge_runs(a, tmp, l, m, r);
    *invocations += 2;
}

int oracle_mergesort(int32_t *data, int32_t *scratch, int64_t n, int64_t cutoff,
                     int64_t *tasks, int64_t *invocations)
{
    if (n < 0 || cutoff < 1) return -1;
    *tasks = 0;
    *invocations = 0;
    ms_rec(data, scratch, 0, n, cutoff, tasks, invocations);
    return 0;
}

/* ------------------------------------------------------------- Cilksort */
/*
 * Cilksort (mergesort whose merge is parallelised;
 * CUTOFF_SORT = 64, CUTOFF_MERGE = 256). Readings (R26):
 *   sort(l, r): if r - l <= CUTOFF_SORT: insertion sort; else fork sort(l, m),
 *               sort(m, r) with m = l + (r - l) / 2; join; fork merge of
 *               [l, m) and [m, r) into the other buffer; join.
 *   merge(A = [a0, a1) of the left run, B = [b0, b1) of the right run) writes
 *               dst[a0 + b0 - m ...): if |A| + |B| <= CUTOFF_MERGE: two-pointer
 *               merge (left first on ties); else split the longer run at its
 *               middle element s and binary-search the other run (left run
 *               split: B elements < A[s] go left; right run split: A elements
 *               <= B[s] go left), fork both halves, join.
 * Sorting happens in place in `data` (scratch holds the merged runs one level
 * up: the oracle copies back after each merge so every level reads `data`).
 * Counts: tasks and invocations (sort: 1 leaf / 3 internal; merge: 1 leaf /
 * 2 internal).
 */
typedef struct { int64_t tasks, invocations; } cs_stats;

static void cs_seq_merge(const int32_t *a, int64_t na, const int32_t *b, int64_t nb, int32_t *out)
{
    int64_t i = 0, j = 0, k = 0;
    while (i < na && j < nb) out[k++] = (b[j] < a[i]) ? b[j++] : a[i++];
    while (i < na) out[k++] = a[i++];
    while (j < nb) out[k++] = b[j++];
}

static int64_t lower_bound_i32(const int32_t *p, int64_t lo, int64_t hi, int32_t v)
{   /* first index in [lo, hi) with p[idx] >= v */
    while (lo < hi) {
        int64_t mid = lo + (hi - lo) / 2;
        if (p[mid] < v) lo = mid + 1; else hi = mid;
    }
    return lo;
}

static int64_t upper_bound_i32(const int32_t *p, int64_t lo, int64_t hi, int32_t v)
{   /* first index in [lo, hi) with p[idx] > v */
    while (lo < hi) {
        int64_t mid = lo + (hi - lo) / 2;
        if (p[mid] <= v) lo = mid + 1; else hi = mid;
    }
    return lo;
}

static void cs_merge(const int32_t *src, int32_t *dst, int64_t m, int64_t a0, int64_t a1, int64_t b0, int64_t b1,
                     int64_t cut_merge, cs_stats *st)
{
    st->tasks += 1;
    const int64_t na = a1 - a0, nb = b1 - b0;
    if (na + nb <= cut_merge) {
        cs_seq_merge(src + a0, na, src + b0, nb, dst + (a0 + b0 - m));
        st->invocations += 1;
        return;
    }
    int64_t sa, sb;
    if (na >= nb) {          /* split the left run at its middle */
        sa = a0 + na / 2;
        sb = lower_bound_i32(src, b0, b1, src[sa]);
    } else {                 /* split the right run at its middle */
        sb = b0 + nb / 2;
        sa = upper_bound_i32(src, a0, a1, src[sb]);
    }
    cs_merge(src, dst, m, a0, sa, b0, sb, cut_merge, st);
    cs_merge(src, dst, m, sa, a1, sb, b1, cut_merge, st);
    st->invocations += 2;
}

static void cs_sort(int32_t *data, int32_t *tmp, int64_t l, int64_t r, int64_t cut_sort, int64_t cut_merge,
                    cs_stats *st)
{
    st->tasks += 1;
    if (r - l <= cut_sort) {
        insertion_sort(data, l, r);
        st->invocations += 1;
        return;
    }
    const int64_t m = l + (r - l) / 2;
    cs_sort(data, tmp, l, m, cut_sort, cut_merge, st);
    cs_sort(data, tmp, m, r, cut_sort, cut_merge, st);
    cs_merge(data, tmp, m, l, m, m, r, cut_merge, st);   /* into tmp[l, r) */
    memcpy(data + l, tmp + l, (size_t)(r - l) * sizeof(int32_t));
    st->invocations += 3;
}

int oracle_cilksort(int32_t *data, int32_t *scratch, int64_t n, int64_t cut_sort, int64_t cut_merge,
                    int64_t *tasks, int64_t *invocations)
{
    if (n < 0 || cut_sort < 1 || cut_merge < 2) return -1;
    cs_stats st = {0, 0};
    cs_sort(data, scratch, 0, n, cut_sort, cut_merge, &st);
    *tasks = st.tasks;
    *invocations = st.invocations;
    return 0;
}

/* ----------------------------------------------------------------- SpMV */
/*
 * SpMV is only named by the paper as a block-cooperative workload (P:42,
 * §4.1); its definition is the standard CSR product
 *     y[i] = sum_{j = row_ptr[i]}^{row_ptr[i+1]-1} val[j] * x[col[j]],
 * accumulated here in fp64 and rounded once (R21).
 */
int oracle_spmv(const int32_t *row_ptr, const int32_t *col, const float *val,
                const float *x, int64_t nrows, double *y64, float *y32)
{
    for (int64_t i = 0; i < nrows; i++) {
        double s = 0.0;
        for (int64_t j = row_ptr[i]; j < row_ptr[i + 1]; j++)
            s += (double)val[j] * (double)x[col[j]];
        if (y64) y64[i] = s;
        if (y32) y32[i] = (float)s;
    }
    return 0;
}

/* ------------------------------------------------------------------ BFS */
/*
 * P:1053-1068 (Prog. graph traversal, §5.1.3) relaxes depth[u] with
 * atomicMin(depth[u], depth[v] + 1) and spawns bfs(u) on improvement, from
 * depth[src] = 0. At quiescence this is the unweighted shortest-path
 * distance (proof sketch in tests/test_oracle_bfs.py), so the oracle is the
 * textbook FIFO breadth-first search. Unreached vertices keep INT32_MAX.
 */
int oracle_bfs(const int32_t *row_ptr, const int32_t *col, int64_t nv, int32_t src,
               int32_t *depth)
{
    if (src < 0 || src >= nv) return -1;
    int32_t *queue = (int32_t *)malloc((size_t)(nv > 0 ? nv : 1) * sizeof(int32_t));
    if (!queue) return -2;
    for (int64_t v = 0; v < nv; v++) depth[v] = INT32_MAX;
    int64_t qh = 0, qt = 0;
    depth[src] = 0;
    queue[qt++] = src;
    while (qh < qt) {
        int32_t v = queue[qh++];
        for (int64_t e = row_ptr[v]; e < row_ptr[v + 1]; e++) {
            int32_t u = col[e];
            if (depth[u] == INT32_MAX) {
                depth[u] = depth[v] + 1;
                queue[qt++] = u;
            }
        }
    }
    free(queue);
    return 0;
}
