/*
 * oracle/w2v_oracle.c — TEST INFRASTRUCTURE ONLY. The plain, slow, sequential CPU oracle of
 * the HogBatch skip-gram negative-sampling SGD step (arXiv 1611.06172).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load this. It shares no code, header, table or constant generator with the CUDA path
 * (paper_1611_06172_b200/csrc); both follow the written contract in DESIGN.md §2 ("CONTRACT").
 *
 * Built twice: -DREAL=double (liboracle_f64.so, the parity reference) and -DREAL=float
 * (liboracle_f32.so, the fp32 error-budget twin). Model init, thresholds, sampler, window,
 * negatives and alpha are integer / fp32 / fp64 exactly as the contract fixes them, in both.
 *
 * Citations: PAPER.md:L is /root/reference/PAPER.md line L; "Alg.1 l.k" is PAPER.md:38+k.
 *   Alg.1 (word2vec Hogwild SGD, one thread)
 *   HogBatch GEMM formulation                 PAPER.md:116-126 (Sec. "Shared Memory
 *                                              Parallelization: HogBatch")
 *   data parallelism
 *   hyper-parameters
 * Readings of the paper's silences are DESIGN.md §3 R1..R18.
 *
 * Parity status of each function is listed in DESIGN.md §4 ("Oracle pins"); every function
 * here has at least one pin in tests/test_oracle_*.py. Parity unpinned: none at function
 * level; multi-replica *trained embeddings* are pinned only through invariants.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#include <pthread.h>

#ifndef REAL
#define REAL double
#endif

enum { TAG_POS = 1, TAG_NEG = 2, TAG_INIT = 3, TAG_GEN = 4, TAG_EVAL = 5, TAG_A1NEG = 6 };

/* ---------------------------------------------------------------- C1: Philox4x32-10 ---- */
/* Salmon, Moraes, Dror, Shaw, "Parallel random numbers: as easy as 1, 2, 3" (SC'11):
 * 10 rounds of  (hi0,lo0)=M0*c0, (hi1,lo1)=M1*c2, c = (hi1^c1^k0, lo1, hi0^c3^k1, lo0),
 * key schedule k0 += W0, k1 += W1 after each round. DESIGN.md C1. */
void orc_philox(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3], k0 = key[0], k1 = key[1];
    int round;
    for (round = 0; round < 10; ++round) {
        uint64_t p0 = (uint64_t)M0 * c0;
        uint64_t p1 = (uint64_t)M1 * c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        c0 = hi1 ^ c1 ^ k0;
        c1 = lo1;
        c2 = hi0 ^ c3 ^ k1;
        c3 = lo0;
        k0 += W0;
        k1 += W1;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* Philox(key = seed, counter = (p lo, p hi, e, tag<<24 | idx)) — DESIGN.md C1 */
void orc_rng_block(uint64_t seed, uint32_t tag, uint32_t e, uint64_t p, uint32_t idx, uint32_t out[4]) {
    uint32_t ctr[4], key[2];
    ctr[0] = (uint32_t)p;
    ctr[1] = (uint32_t)(p >> 32);
    ctr[2] = e;
    ctr[3] = (tag << 24) | (idx & 0xFFFFFFu);
    key[0] = (uint32_t)seed;
    key[1] = (uint32_t)(seed >> 32);
    orc_philox(ctr, key, out);
}

/* u64 number d of a (tag,e,p) stream: block idx = d>>1, half h = d&1 -> out[2h+1]<<32 | out[2h] */
uint64_t orc_rng_u64(uint64_t seed, uint32_t tag, uint32_t e, uint64_t p, uint32_t d) {
    uint32_t o[4];
    uint32_t h = d & 1u;
    orc_rng_block(seed, tag, e, p, d >> 1, o);
    return ((uint64_t)o[2 * h + 1] << 32) | o[2 * h];
}

static uint64_t mulhi64(uint64_t a, uint64_t b) {
    return (uint64_t)(((unsigned __int128)a * b) >> 64);
}

/* ---------------------------------------------------------------- a0: setup -------------- */
/* Counts c[w] = #{p : ids[p] = w}. Returns -1 if an id is outside [0,V) (SPEC.md:253 makes
 * id<V a precondition; we check it). */
int orc_counts(const int32_t* ids, int64_t n, int64_t V, int64_t* c) {
    int64_t p;
    memset(c, 0, sizeof(int64_t) * (size_t)V);
    for (p = 0; p < n; ++p) {
        if (ids[p] < 0 || ids[p] >= V) return -1;
        c[ids[p]] += 1;
    }
    return 0;
}

/* Keep thresholds (C2; reading R5 of PAPER.md:167 "sample=1e-4" via the reference
 * word2vec rule keep = (sqrt(z)+1)/z, z = c/(t*T)):
 *   thr[w] = 2^32 if t == 0 or c == 0 or k >= 1, else floor(k * 2^32). keep iff u32 < thr. */
void orc_thresholds(const int64_t* c, int64_t V, int64_t T, float t, uint64_t* thr) {
    int64_t w;
    double t64 = (double)t;
    for (w = 0; w < V; ++w) {
        if (t64 == 0.0 || c[w] == 0) { thr[w] = 4294967296ull; continue; }
        double z = (double)c[w] / (t64 * (double)T);
        double k = (sqrt(z) + 1.0) / z;
        thr[w] = (k >= 1.0) ? 4294967296ull : (uint64_t)floor(k * 4294967296.0);
    }
}

/* Unigram^0.75 sampler (reading R1 of Alg.1 l.10 "sample one word from V"):
 * q[w] = floor(sqrt(c)*sqrt(sqrt(c)) * 2^20), P[0]=0, P[w+1]=P[w]+q[w]. Returns -1 if P[V]=0.
 * DESIGN.md C3. */
int orc_sampler(const int64_t* c, int64_t V, uint64_t* P) {
    int64_t w;
    P[0] = 0;
    for (w = 0; w < V; ++w) {
        double x = (double)c[w];
        double wgt = sqrt(x) * sqrt(sqrt(x));
        P[w + 1] = P[w] + (uint64_t)floor(wgt * 1048576.0);
    }
    return P[V] == 0 ? -1 : 0;
}

/* invcdf(x) = smallest w with P[w+1] > x, x in [0, P[V]) — plain binary search (C3). */
int64_t orc_invcdf(const uint64_t* P, int64_t V, uint64_t x) {
    int64_t lo = 0, hi = V - 1;
    while (lo < hi) {
        int64_t mid = lo + (hi - lo) / 2;
        if (P[mid + 1] > x) hi = mid; else lo = mid + 1;
    }
    return lo;
}

/* Init (reading R10 of Alg.1 l.1 "Given model parameter Omega"):
 * M_in[r][d] = ((float)(u32>>8) * 2^-24 - 0.5f) / (float)D, u32 = word (r*D+d)&3 of
 * Philox(INIT, e=0, p=(r*D+d)>>2, idx=0); M_out = 0. fp32 arithmetic, IEEE division. */
void orc_init(int64_t V, int32_t D, uint64_t seed, float* M_in, float* M_out) {
    int64_t i, total = V * (int64_t)D;
    uint32_t o[4];
    for (i = 0; i < total; ++i) {
        if ((i & 3) == 0) orc_rng_block(seed, TAG_INIT, 0, (uint64_t)(i >> 2), 0, o);
        uint32_t u = o[i & 3];
        volatile float f = (float)(u >> 8) * 5.9604644775390625e-08f; /* 2^-24 */
        volatile float g = f - 0.5f;
        M_in[i] = g / (float)D;
        M_out[i] = 0.0f;
    }
}

/* Learning rate (reading R8): progress pi (rank-local words), W replicas,
 * E epochs over n_global words, quantum Q:
 *   alpha = (float)( (double)alpha0 * max(1 - (W*floor(pi/Q)*Q) / (E*n_global + 1), 1e-4) ) */
float orc_alpha(float alpha0, int64_t pi, int64_t Q, int32_t W, int32_t E, int64_t n_global) {
    int64_t num = (int64_t)W * (pi / Q) * Q;
    double frac = (double)num / (double)((int64_t)E * n_global + 1);
    double m = 1.0 - frac;
    if (m < 1e-4) m = 1e-4;
    return (float)((double)alpha0 * m);
}

/* sigma(x) = 1/(1+e^-x), exact (reading R9; Alg.1 l.14) */
static REAL sigmoid(REAL x) { return (REAL)1 / ((REAL)1 + exp(-x)); }

/* softplus(x) = log(1+e^x) = max(x,0) + log1p(e^-|x|), evaluated in fp64 */
static double softplus(double x) { return (x > 0 ? x : 0.0) + log1p(exp(-fabs(x))); }

/* ---------------------------------------------------------------- the steps ------------- */
/* O-HB: one HogBatch minibatch (Fig. 2 right).
 * A = M_in[ctx[0..N-1]] (N x D), B = M_out[out[0..K]] ((K+1) x D), both value snapshots
 * taken before any write (reading R11). C = A B^T; E = label - sigma(C) with label_j = [j=0];
 * dIn = (alpha E) B; dOut = (alpha E)^T A; then M_in[ctx_i] += dIn_i (i ascending) and
 * M_out[out_j] += dOut_j (j ascending); duplicates accumulate. Returns the
 * pre-update SGNS loss sum_i [softplus(-C_i0) + sum_{j>=1} softplus(C_ij)]. */
double orc_hogbatch_step(REAL* M_in, REAL* M_out, int32_t D, const int32_t* ctx, int32_t N,
                         const int32_t* out, int32_t K, float alpha_f) {
    int32_t i, j, d, KP1 = K + 1;
    REAL alpha = (REAL)alpha_f;
    REAL* A = (REAL*)malloc(sizeof(REAL) * (size_t)N * D);
    REAL* B = (REAL*)malloc(sizeof(REAL) * (size_t)KP1 * D);
    REAL* C = (REAL*)malloc(sizeof(REAL) * (size_t)N * KP1);
    REAL* G = (REAL*)malloc(sizeof(REAL) * (size_t)N * KP1);
    REAL* dIn = (REAL*)malloc(sizeof(REAL) * (size_t)N * D);
    REAL* dOut = (REAL*)malloc(sizeof(REAL) * (size_t)KP1 * D);
    double loss = 0.0;
    /* gather (snapshot) */
    for (i = 0; i < N; ++i) memcpy(A + (size_t)i * D, M_in + (size_t)ctx[i] * D, sizeof(REAL) * D);
    for (j = 0; j < KP1; ++j) memcpy(B + (size_t)j * D, M_out + (size_t)out[j] * D, sizeof(REAL) * D);
    /* C = A B^T ; E = label - sigma(C) ; G = alpha E */
    for (i = 0; i < N; ++i) {
        for (j = 0; j < KP1; ++j) {
            REAL s = 0;
            for (d = 0; d < D; ++d) s += A[(size_t)i * D + d] * B[(size_t)j * D + d];
            C[i * KP1 + j] = s;
            REAL label = (j == 0) ? (REAL)1 : (REAL)0;
            REAL err = label - sigmoid(s);
            G[i * KP1 + j] = alpha * err;
            loss += (j == 0) ? softplus(-(double)s) : softplus((double)s);
        }
    }
    /* dIn = G B  (N x D) */
    for (i = 0; i < N; ++i)
        for (d = 0; d < D; ++d) {
            REAL s = 0;
            for (j = 0; j < KP1; ++j) s += G[i * KP1 + j] * B[(size_t)j * D + d];
            dIn[(size_t)i * D + d] = s;
        }
    /* dOut = G^T A  ((K+1) x D) */
    for (j = 0; j < KP1; ++j)
        for (d = 0; d < D; ++d) {
            REAL s = 0;
            for (i = 0; i < N; ++i) s += G[i * KP1 + j] * A[(size_t)i * D + d];
            dOut[(size_t)j * D + d] = s;
        }
    /* write back */
    for (i = 0; i < N; ++i)
        for (d = 0; d < D; ++d) M_in[(size_t)ctx[i] * D + d] += dIn[(size_t)i * D + d];
    for (j = 0; j < KP1; ++j)
        for (d = 0; d < D; ++d) M_out[(size_t)out[j] * D + d] += dOut[(size_t)j * D + d];
    free(A); free(B); free(C); free(G); free(dIn); free(dOut);
    return loss;
}

/* O-A1: Algorithm 1 verbatim for one target word and N inputs; the K
 * negatives of input i are negs[i*K + (k-1)] (line 10, drawn by the caller). Returns the
 * SGNS loss of the (input, output) pairs at the moment each dot product is taken. */
double orc_alg1_step(REAL* M_in, REAL* M_out, int32_t D, const int32_t* ctx, int32_t N,
                     int32_t target, const int32_t* negs, int32_t K, float alpha_f) {
    int32_t i, j, k;
    REAL alpha = (REAL)alpha_f;
    REAL* temp = (REAL*)malloc(sizeof(REAL) * (size_t)D);
    double loss = 0.0;
    for (i = 0; i < N; ++i) {                                     /* line 2 */
        int32_t input_word = ctx[i];                              /* line 3 */
        for (j = 0; j < D; ++j) temp[j] = 0;                      /* line 4 */
        for (k = 0; k < K + 1; ++k) {                             /* line 6 */
            int32_t target_word;
            REAL label;
            if (k == 0) { target_word = target; label = 1; }      /* line 8 */
            else { target_word = negs[(size_t)i * K + (k - 1)]; label = 0; } /* line 10 */
            REAL inn = 0;                                         /* line 12 */
            for (j = 0; j < D; ++j)                               /* line 13 */
                inn += M_in[(size_t)input_word * D + j] * M_out[(size_t)target_word * D + j];
            REAL err = label - sigmoid(inn);                      /* line 14 */
            loss += (k == 0) ? softplus(-(double)inn) : softplus((double)inn);
            for (j = 0; j < D; ++j) temp[j] += err * M_out[(size_t)target_word * D + j]; /* line 15 */
            for (j = 0; j < D; ++j)                               /* line 17 */
                M_out[(size_t)target_word * D + j] += alpha * err * M_in[(size_t)input_word * D + j];
        }
        for (j = 0; j < D; ++j) M_in[(size_t)input_word * D + j] += alpha * temp[j]; /* line 20 */
    }
    free(temp);
    return loss;
}

/* ---------------------------------------------------------------- a1/a2: batches --------- */
/* Negative draw number k (1-based) of the target at global position p, continuing the draw
 * counter *d (C7; readings R1-R4): repeat x = invcdf(mulhi64(u64(NEG,e,p,d++), P[V]))
 * until x != tw, or allow_target_negative, or 100 tries; then x = (tw+1) mod V. */
int32_t orc_draw_negative(uint64_t seed, uint32_t e, uint64_t p, uint32_t* d, const uint64_t* P,
                          int64_t V, int32_t tw, int allow_target_negative) {
    int tries;
    for (tries = 0; tries < 100; ++tries) {
        uint64_t r = orc_rng_u64(seed, TAG_NEG, e, p, (*d)++);
        int32_t x = (int32_t)orc_invcdf(P, V, mulhi64(r, P[V]));
        if (x != tw || allow_target_negative) return x;
    }
    return (int32_t)((tw + 1) % V);
}

typedef struct {
    int64_t V;
    int32_t D, window, K;
    float alpha0, t;
    uint64_t seed;
    int32_t L;                      /* chunk length (reading R7) */
    int32_t allow_target_negative;  /* 1: literal Alg.1 l.10 */
    int64_t lr_quantum;             /* Q */
    int32_t epochs;                 /* E */
    int64_t n_global;               /* raw tokens over all replicas */
    int32_t world;                  /* W */
    int32_t algorithm;              /* 0 = HogBatch (O-HB), 1 = Alg.1 (O-A1) */
} orc_params;

typedef struct {
    int64_t words, targets, row_touches, loss_pairs;
    double loss_sum;
} orc_stats;

/* Debug stream for global positions [base, base+len): keep flag, half-window b (0 = not
 * kept), N (0 = not a trained target), ctx ids (2*window per position, -1 padded), and the
 * K shared negatives (-1 padded). Any pointer may be NULL. */
typedef struct {
    int64_t base, len;
    uint8_t* keep;
    uint8_t* b;
    uint8_t* N;
    int32_t* ctx;
    int32_t* neg;
    int32_t* a1neg;  /* O-A1 only: the K negatives of each input i, [len][2*window][K] (-1 padded) */
} orc_debug;

/* Train on global chunks [chunk_lo, chunk_hi) for epoch e (C5-C8, Sec. "Oracle
 * algorithm O-HB" steps 5.1-5.5). ids[k] is the token at global position ids_base+k; the
 * replica's shard is [shard_start, shard_start+n_local), chunk-aligned. thr and P come from
 * the GLOBAL counts. Returns 0, or -1 on bad arguments. */
int orc_train_range(const orc_params* prm, const uint64_t* thr, const uint64_t* P,
                    const int32_t* ids, int64_t ids_base, int64_t ids_len, int64_t shard_start,
                    int64_t n_local, int32_t e, int64_t chunk_lo, int64_t chunk_hi,
                    REAL* M_in, REAL* M_out, orc_stats* st, orc_debug* dbg) {
    const int64_t L = prm->L, V = prm->V;
    const int32_t D = prm->D, K = prm->K, W2 = 2 * prm->window;
    const int64_t shard_end = shard_start + n_local;
    int64_t s;
    int32_t *kept_pos_off, *ctx, *outs, *negs;
    if (L < 1 || D < 1 || prm->window < 1 || K < 0) return -1;
    kept_pos_off = (int32_t*)malloc(sizeof(int32_t) * (size_t)L);
    ctx = (int32_t*)malloc(sizeof(int32_t) * (size_t)W2);
    outs = (int32_t*)malloc(sizeof(int32_t) * (size_t)(K + 1));
    negs = (int32_t*)malloc(sizeof(int32_t) * (size_t)(W2 * (K > 0 ? K : 1) + 1));
    for (s = chunk_lo; s < chunk_hi; ++s) {
        int64_t c0 = s * L, c1 = (s + 1) * L;
        int64_t m, nk = 0;
        if (c1 > shard_end) c1 = shard_end;
        if (c0 < shard_start) c0 = shard_start;
        if (c0 >= c1) continue;
        /* 5.1 keep flags, compaction in order */
        for (int64_t p = c0; p < c1; ++p) {
            uint32_t o[4];
            int32_t w = ids[p - ids_base];
            orc_rng_block(prm->seed, TAG_POS, (uint32_t)e, (uint64_t)p, 0, o);
            int keep = (uint64_t)o[0] < thr[w];
            if (keep) kept_pos_off[nk++] = (int32_t)(p - c0);
            if (dbg && p >= dbg->base && p < dbg->base + dbg->len) {
                int64_t q = p - dbg->base;
                if (dbg->keep) dbg->keep[q] = (uint8_t)keep;
                if (dbg->b) dbg->b[q] = 0;
                if (dbg->N) dbg->N[q] = 0;
                if (dbg->ctx) for (int32_t u = 0; u < W2; ++u) dbg->ctx[q * W2 + u] = -1;
                if (dbg->neg) for (int32_t u = 0; u < K; ++u) dbg->neg[q * K + u] = -1;
                if (dbg->a1neg) for (int32_t u = 0; u < W2 * K; ++u) dbg->a1neg[q * W2 * K + u] = -1;
            }
        }
        st->words += c1 - c0;
        /* 5.2 - 5.5 per kept target, in order */
        for (m = 0; m < nk; ++m) {
            int64_t p = c0 + kept_pos_off[m];
            int32_t tw = ids[p - ids_base];
            uint32_t o[4];
            orc_rng_block(prm->seed, TAG_POS, (uint32_t)e, (uint64_t)p, 0, o);
            int32_t b = 1 + (int32_t)(((uint64_t)o[1] * (uint64_t)prm->window) >> 32);
            int32_t N = 0;
            for (int64_t mm = m - b; mm <= m + b; ++mm) {
                if (mm < 0 || mm >= nk || mm == m) continue;
                ctx[N++] = ids[c0 + kept_pos_off[mm] - ids_base];
            }
            int in_dbg = dbg && p >= dbg->base && p < dbg->base + dbg->len;
            if (in_dbg && dbg->b) dbg->b[p - dbg->base] = (uint8_t)b;
            if (N == 0) continue;
            float alpha = orc_alpha(prm->alpha0, (int64_t)e * n_local + (p - shard_start),
                                    prm->lr_quantum, prm->world, prm->epochs, prm->n_global);
            double loss;
            if (prm->algorithm == 0) {
                uint32_t d = 0;
                outs[0] = tw;
                for (int32_t k = 1; k <= K; ++k)
                    outs[k] = orc_draw_negative(prm->seed, (uint32_t)e, (uint64_t)p, &d, P, V, tw,
                                                prm->allow_target_negative);
                /* M_in == NULL: batch stream only (a1/a2 rows), no SGD step */
                loss = M_in ? orc_hogbatch_step(M_in, M_out, D, ctx, N, outs, K, alpha) : 0.0;
                st->row_touches += N + K + 1;
            } else {
                /* O-A1: per-input negatives on the A1NEG stream, idx = i<<12 | (d>>1) */
                for (int32_t i = 0; i < N; ++i) {
                    uint32_t d = 0;
                    for (int32_t k = 1; k <= K; ++k) {
                        int32_t x = -1;
                        int tries;
                        for (tries = 0; tries < 100; ++tries) {
                            uint32_t oo[4];
                            orc_rng_block(prm->seed, TAG_A1NEG, (uint32_t)e, (uint64_t)p,
                                          ((uint32_t)i << 12) | (d >> 1), oo);
                            uint64_t r = ((uint64_t)oo[2 * (d & 1) + 1] << 32) | oo[2 * (d & 1)];
                            d++;
                            x = (int32_t)orc_invcdf(P, V, mulhi64(r, P[V]));
                            if (x != tw || prm->allow_target_negative) break;
                        }
                        if (tries == 100) x = (int32_t)((tw + 1) % V);
                        negs[i * K + (k - 1)] = x;
                    }
                }
                loss = M_in ? orc_alg1_step(M_in, M_out, D, ctx, N, tw, negs, K, alpha) : 0.0;
                st->row_touches += (int64_t)N * (K + 1) + N;
            }
            st->loss_sum += loss;
            st->loss_pairs += (int64_t)N * (K + 1);
            st->targets += 1;
            if (in_dbg) {
                int64_t q = p - dbg->base;
                if (dbg->N) dbg->N[q] = (uint8_t)N;
                if (dbg->ctx) for (int32_t u = 0; u < N; ++u) dbg->ctx[q * W2 + u] = ctx[u];
                if (dbg->neg && prm->algorithm == 0)
                    for (int32_t u = 0; u < K; ++u) dbg->neg[q * K + u] = outs[u + 1];
                if (dbg->a1neg && prm->algorithm == 1)
                    for (int32_t u = 0; u < N * K; ++u) dbg->a1neg[q * W2 * K + u] = negs[u];
            }
        }
    }
    free(kept_pos_off); free(ctx); free(outs); free(negs);
    return 0;
}

/* CPU TIMING BASELINE ONLY (SURVEY.md §8(c) "--threads T Hogwild mode", §8(d)): T threads run
 * orc_train_range on contiguous slices of [chunk_lo, chunk_hi) concurrently on the SAME model,
 * with unsynchronised read-modify-writes — Hogwild as PAPER.md:34 describes it ("parallelized
 * over threads without any additional change"). Not used for parity: the result depends on the
 * interleaving. Statistics are summed over threads; no debug stream. */
typedef struct {
    const orc_params* prm;
    const uint64_t *thr, *P;
    const int32_t* ids;
    int64_t ids_base, ids_len, shard_start, n_local, chunk_lo, chunk_hi;
    int32_t e;
    REAL *M_in, *M_out;
    orc_stats st;
} orc_thread_job;

static void* orc_thread_main(void* arg) {
    orc_thread_job* j = (orc_thread_job*)arg;
    orc_train_range(j->prm, j->thr, j->P, j->ids, j->ids_base, j->ids_len, j->shard_start, j->n_local, j->e,
                    j->chunk_lo, j->chunk_hi, j->M_in, j->M_out, &j->st, NULL);
    return NULL;
}

int orc_train_range_hogwild(const orc_params* prm, const uint64_t* thr, const uint64_t* P, const int32_t* ids,
                            int64_t ids_base, int64_t ids_len, int64_t shard_start, int64_t n_local, int32_t e,
                            int64_t chunk_lo, int64_t chunk_hi, REAL* M_in, REAL* M_out, orc_stats* st,
                            int32_t threads) {
    orc_thread_job jobs[256];
    pthread_t th[256];
    int32_t t, T = threads < 1 ? 1 : threads > 256 ? 256 : threads;
    for (t = 0; t < T; ++t) {
        orc_thread_job* j = &jobs[t];
        j->prm = prm; j->thr = thr; j->P = P; j->ids = ids; j->ids_base = ids_base; j->ids_len = ids_len;
        j->shard_start = shard_start; j->n_local = n_local; j->e = e;
        j->chunk_lo = chunk_lo + (chunk_hi - chunk_lo) * t / T;
        j->chunk_hi = chunk_lo + (chunk_hi - chunk_lo) * (t + 1) / T;
        j->M_in = M_in; j->M_out = M_out;
        memset(&j->st, 0, sizeof j->st);
        pthread_create(&th[t], NULL, orc_thread_main, j);
    }
    for (t = 0; t < T; ++t) {
        pthread_join(th[t], NULL);
        st->words += jobs[t].st.words;
        st->targets += jobs[t].st.targets;
        st->row_touches += jobs[t].st.row_touches;
        st->loss_pairs += jobs[t].st.loss_pairs;
        st->loss_sum += jobs[t].st.loss_sum;
    }
    return 0;
}

/* Elementwise mean of W replicas, in place into every replica (reading R13).
 * The sum runs over replicas in rank order, then divides by W. */
void orc_average(REAL** reps, int32_t W, int64_t len) {
    int64_t i;
    for (i = 0; i < len; ++i) {
        REAL s = 0;
        for (int32_t r = 0; r < W; ++r) s += reps[r][i];
        s = s / (REAL)W;
        for (int32_t r = 0; r < W; ++r) reps[r][i] = s;
    }
}

int orc_real_size(void) { return (int)sizeof(REAL); }
