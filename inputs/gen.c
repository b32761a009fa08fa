/*
 * inputs/gen.c — seeded synthetic corpus generator (test and bench INPUTS only).
 *
 * This module holds none of the method's arithmetic (no subsampling, no negative sampler,
 * no SGD). It produces the token-id streams that stand in for the paper's One Billion Word
 * benchmark (Sec. "Experiments": dim=300, negative=5, window=5, sample=1e-4,
 * V=1,115,011) with the shapes BASELINE.json's configs name. Both the CPU oracle and the
 * CUDA path consume its output; neither imports the other.
 *
 * Recipe (DESIGN.md §"Input recipe", SURVEY.md §8(d) "Generator"):
 *   - Ids are frequency ranks: word w has weight (w+1)^-s, computed once in fp64 with libm
 *     pow() and quantised as zq[w] = floor(pow(w+1,-s) * 2^40). Id 0 is the most frequent.
 *   - Philox4x32-10 (own copy; C1), key = seed, counter =
 *     (ctr lo, ctr hi, 0, GEN<<24 | idx), GEN = 4. u64 = out[1]<<32 | out[0].
 *   - iid:     token i = invcdf_zipf(mulhi64(u64(GEN, i, 0), Z)).
 *   - planted: cluster(w) = w mod C. Sentence s = i / Lg draws its cluster
 *              c = invcdf(cluster weights, mulhi64(u64(GEN, s, 1), Zc_total)); token i then
 *              draws member m = invcdf(member weights of c, mulhi64(u64(GEN, i, 0), Z_c)),
 *              w = c + m*C. The marginal of w is exactly the quantised Zipf(s).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#include <pthread.h>

#define GEN_TAG 4u

static inline void gen_mulhilo(uint32_t a, uint32_t b, uint32_t* hi, uint32_t* lo) {
    uint64_t p = (uint64_t)a * (uint64_t)b;
    *hi = (uint32_t)(p >> 32);
    *lo = (uint32_t)p;
}

static void gen_philox(const uint32_t in[4], const uint32_t key[2], uint32_t out[4]) {
    uint32_t c0 = in[0], c1 = in[1], c2 = in[2], c3 = in[3];
    uint32_t k0 = key[0], k1 = key[1];
    for (int r = 0; r < 10; ++r) {
        uint32_t hi0, lo0, hi1, lo1;
        gen_mulhilo(0xD2511F53u, c0, &hi0, &lo0);
        gen_mulhilo(0xCD9E8D57u, c2, &hi1, &lo1);
        uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

static inline uint64_t gen_u64(uint64_t seed, uint64_t ctr, uint32_t idx) {
    uint32_t in[4] = {(uint32_t)ctr, (uint32_t)(ctr >> 32), 0u, (GEN_TAG << 24) | idx};
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t out[4];
    gen_philox(in, key, out);
    return ((uint64_t)out[1] << 32) | out[0];
}

static inline uint64_t gen_mulhi64(uint64_t a, uint64_t b) {
    return (uint64_t)(((unsigned __int128)a * b) >> 64);
}

/* smallest k in [0,n) with pre[k+1] > x, for x < pre[n] */
static inline int64_t gen_invcdf(const uint64_t* pre, int64_t n, uint64_t x) {
    int64_t lo = 0, hi = n - 1;
    while (lo < hi) {
        int64_t mid = lo + ((hi - lo) >> 1);
        if (pre[mid + 1] > x) hi = mid; else lo = mid + 1;
    }
    return lo;
}

/* exported: Philox block for the cross-implementation known-answer test */
void gen_philox4x32_10(const uint32_t in[4], const uint32_t key[2], uint32_t out[4]) {
    gen_philox(in, key, out);
}

/* zq[w] = floor(pow(w+1, -s) * 2^40); pre[0]=0, pre[w+1]=pre[w]+zq[w]. Returns 0. */
int gen_zipf_prefix(int64_t V, double s, uint64_t* pre) {
    pre[0] = 0;
    for (int64_t w = 0; w < V; ++w) {
        double wt = pow((double)(w + 1), -s);
        uint64_t q = (uint64_t)floor(wt * 1099511627776.0);
        if (q == 0) q = 1;
        pre[w + 1] = pre[w] + q;
    }
    return 0;
}

/* Planted tables. cl_pre[C+1]: prefix over cluster weights. mem_pre: per-cluster member
 * prefixes, cluster c occupying mem_pre[off[c] .. off[c]+M_c] (M_c+1 entries), where
 * off[c] = c + sum_{c'<c} M_{c'}; members of c are w = c + m*C, m < M_c. */
int gen_planted_tables(int64_t V, double s, int64_t C, uint64_t* cl_pre, uint64_t* mem_pre,
                       int64_t* off) {
    if (C < 1 || C > V) return -1;
    int64_t o = 0;
    cl_pre[0] = 0;
    for (int64_t c = 0; c < C; ++c) {
        off[c] = o;
        int64_t M = (V - 1 - c) / C + 1;
        mem_pre[o] = 0;
        for (int64_t m = 0; m < M; ++m) {
            int64_t w = c + m * C;
            double wt = pow((double)(w + 1), -s);
            uint64_t q = (uint64_t)floor(wt * 1099511627776.0);
            if (q == 0) q = 1;
            mem_pre[o + m + 1] = mem_pre[o + m] + q;
        }
        cl_pre[c + 1] = cl_pre[c] + mem_pre[o + M];
        o += M + 1;
    }
    off[C] = o;
    return 0;
}

typedef struct {
    int kind; /* 0 iid, 1 planted */
    uint64_t seed;
    int64_t V, C, Lg;
    const uint64_t *pre, *cl_pre, *mem_pre;
    const int64_t* off;
    int64_t i0, n;
    int32_t* out;
} gen_job;

static void gen_range(const gen_job* j, int64_t a, int64_t b) {
    if (j->kind == 0) {
        uint64_t Z = j->pre[j->V];
        for (int64_t k = a; k < b; ++k) {
            uint64_t i = (uint64_t)(j->i0 + k);
            j->out[k] = (int32_t)gen_invcdf(j->pre, j->V, gen_mulhi64(gen_u64(j->seed, i, 0), Z));
        }
    } else {
        uint64_t Zc = j->cl_pre[j->C];
        int64_t cur_s = -1, c = 0;
        for (int64_t k = a; k < b; ++k) {
            int64_t i = j->i0 + k;
            int64_t s = i / j->Lg;
            if (s != cur_s) {
                cur_s = s;
                c = gen_invcdf(j->cl_pre, j->C, gen_mulhi64(gen_u64(j->seed, (uint64_t)s, 1), Zc));
            }
            int64_t M = (j->V - 1 - c) / j->C + 1;
            const uint64_t* mp = j->mem_pre + j->off[c];
            int64_t m = gen_invcdf(mp, M, gen_mulhi64(gen_u64(j->seed, (uint64_t)i, 0), mp[M]));
            j->out[k] = (int32_t)(c + m * j->C);
        }
    }
}

typedef struct { const gen_job* j; int64_t a, b; } gen_slice;
static void* gen_thread(void* p) {
    gen_slice* s = (gen_slice*)p;
    gen_range(s->j, s->a, s->b);
    return NULL;
}

static void gen_run(const gen_job* j, int threads) {
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    if (threads == 1 || j->n < 65536) { gen_range(j, 0, j->n); return; }
    pthread_t th[256];
    gen_slice sl[256];
    for (int t = 0; t < threads; ++t) {
        sl[t].j = j;
        sl[t].a = j->n * t / threads;
        sl[t].b = j->n * (t + 1) / threads;
        pthread_create(&th[t], NULL, gen_thread, &sl[t]);
    }
    for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
}

/* tokens i0 .. i0+n-1 of the iid Zipf corpus */
void gen_iid(uint64_t seed, const uint64_t* pre, int64_t V, int64_t i0, int64_t n, int32_t* out,
             int threads) {
    gen_job j;
    memset(&j, 0, sizeof j);
    j.kind = 0; j.seed = seed; j.V = V; j.pre = pre; j.i0 = i0; j.n = n; j.out = out;
    gen_run(&j, threads);
}

/* tokens i0 .. i0+n-1 of the planted-cluster corpus with sentence length Lg */
void gen_planted(uint64_t seed, int64_t V, int64_t C, int64_t Lg, const uint64_t* cl_pre,
                 const uint64_t* mem_pre, const int64_t* off, int64_t i0, int64_t n, int32_t* out,
                 int threads) {
    gen_job j;
    memset(&j, 0, sizeof j);
    j.kind = 1; j.seed = seed; j.V = V; j.C = C; j.Lg = Lg;
    j.cl_pre = cl_pre; j.mem_pre = mem_pre; j.off = off; j.i0 = i0; j.n = n; j.out = out;
    gen_run(&j, threads);
}
