/*
 * exflow_oracle.c -- CPU restatement of the ExFlow reference path.
 * TEST INFRASTRUCTURE ONLY (see exflow_oracle.h). Citations are
 * /root/reference/proj paths.
 */
#include "exflow_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[512];
static int fail(const char* msg) {
    snprintf(g_err, sizeof(g_err), "%s", msg);
    return 2;
}
const char* orc_last_error(void) { return g_err; }

/* ------------------------------------------------------------------------
 * rng -- include/exflow/rng.hpp:17-66 (xoshiro256** seeded by splitmix64)
 * ---------------------------------------------------------------------- */
uint64_t orc_splitmix64(uint64_t* x) { /* rng.hpp:55-60 */
    uint64_t z = (*x += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

void orc_rng_init(orc_rng* r, uint64_t seed) { /* rng.hpp:19-24 */
    uint64_t x = seed;
    for (int i = 0; i < 4; ++i) r->s[i] = orc_splitmix64(&x);
}

static inline uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

uint64_t orc_rng_next(orc_rng* r) { /* rng.hpp:26-36 */
    uint64_t* s = r->s;
    const uint64_t result = rotl64(s[1] * 5, 7) * 9;
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl64(s[3], 45);
    return result;
}

uint64_t orc_rng_below(orc_rng* r, uint64_t bound) { /* rng.hpp:40-48 */
    const uint64_t threshold = (0 - bound) % bound;
    for (;;) {
        const uint64_t v = orc_rng_next(r);
        if (v >= threshold) return v % bound;
    }
}

double orc_rng_uniform01(orc_rng* r) { /* rng.hpp:53 */
    return (double)(orc_rng_next(r) >> 11) * 0x1.0p-53;
}

uint64_t orc_seed_stream(uint64_t seed, uint64_t stream) { /* rng.hpp:70-73 */
    uint64_t x = seed ^ (0xA0761D6478BD642FULL * (stream + 1));
    return orc_splitmix64(&x);
}

void orc_shuffle_int(int32_t* v, int64_t n, orc_rng* r) { /* rng.hpp:76-82 */
    for (int64_t i = n; i > 1; --i) {
        const int64_t j = (int64_t)orc_rng_below(r, (uint64_t)i);
        int32_t tmp = v[i - 1];
        v[i - 1] = v[j];
        v[j] = tmp;
    }
}

/* ------------------------------------------------------------------------
 * synth -- src/synth.cpp:11-58
 * ---------------------------------------------------------------------- */
int orc_generate_markov_trace(int32_t E, int32_t L, int64_t T, double alpha,
                              int32_t groups, uint64_t seed, int32_t* paths) {
    /* validate: synth.cpp:11-28 */
    if (E < 1) return fail("num_experts must be >= 1");
    if (L < 2) return fail("num_layers must be >= 2");
    if (T < 1) return fail("num_tokens must be >= 1");
    if (alpha < 0.0 || alpha > 1.0) return fail("affinity_strength must be in [0,1]");
    if (groups < 1 || E % groups != 0) return fail("planted_groups must divide num_experts");
    const int32_t block = E / groups;
    orc_rng r;
    orc_rng_init(&r, seed);
    /* draw order: synth.cpp:40-51 */
    for (int64_t t = 0; t < T; ++t) {
        int32_t current = (int32_t)orc_rng_below(&r, (uint64_t)E);
        paths[t * L] = current;
        for (int32_t j = 1; j < L; ++j) {
            if (orc_rng_uniform01(&r) < alpha) {
                current = (current / block) * block + (int32_t)orc_rng_below(&r, (uint64_t)block);
            } else {
                current = (int32_t)orc_rng_below(&r, (uint64_t)E);
            }
            paths[t * L + j] = current;
        }
    }
    return 0;
}

double orc_expected_planted_locality(double alpha, int32_t groups) { /* synth.cpp:55-58 */
    return alpha + (1.0 - alpha) / groups;
}

/* ------------------------------------------------------------------------
 * trace -- src/trace.cpp:53-70 (validate), :191-260, :285-304
 * ---------------------------------------------------------------------- */
int orc_validate_trace(const int32_t* paths, int64_t T, int32_t L, int32_t E) {
    if (E < 1) return fail("num_experts must be >= 1");
    if (L < 2) return fail("num_layers must be >= 2");
    if (T < 1) return fail("trace contains no token paths");
    for (int64_t i = 0; i < T * (int64_t)L; ++i) {
        if (paths[i] < 0 || paths[i] >= E) return fail("expert id out of range");
    }
    return 0;
}

int orc_count_transitions(const int32_t* paths, int64_t T, int32_t L, int32_t E,
                          int32_t gap, int64_t* counts, int64_t* row_totals) {
    int rc = orc_validate_trace(paths, T, L, E);
    if (rc) return rc;
    if (gap < 1 || gap > L - 1) return fail("gap out of range"); /* trace.cpp:193-196 */
    const int32_t pairs = L - gap;
    memset(counts, 0, sizeof(int64_t) * (size_t)pairs * E * E);
    /* HOT LOOP trace.cpp:205-209 */
    for (int64_t t = 0; t < T; ++t) {
        const int32_t* p = paths + t * L;
        for (int32_t j = 0; j < pairs; ++j) {
            counts[((int64_t)j * E + p[j]) * E + p[j + gap]] += 1;
        }
    }
    /* row totals trace.cpp:210-213 */
    if (row_totals) {
        for (int32_t j = 0; j < pairs; ++j)
            for (int32_t a = 0; a < E; ++a) {
                int64_t s = 0;
                for (int32_t b = 0; b < E; ++b) s += counts[((int64_t)j * E + a) * E + b];
                row_totals[(int64_t)j * E + a] = s;
            }
    }
    return 0;
}

/* Integer-sum-parallel variant allowed by SPEC.md:102 / :339 (result equals
 * the sequential sum exactly: per-thread partial integer counts are summed). */
typedef struct {
    const int32_t* paths;
    int64_t t0, t1;
    int32_t L, E, gap;
    int64_t* counts;
} hist_job;

static void* hist_worker(void* arg) {
    hist_job* job = (hist_job*)arg;
    const int32_t pairs = job->L - job->gap;
    for (int64_t t = job->t0; t < job->t1; ++t) {
        const int32_t* p = job->paths + t * job->L;
        for (int32_t j = 0; j < pairs; ++j)
            job->counts[((int64_t)j * job->E + p[j]) * job->E + p[j + job->gap]] += 1;
    }
    return NULL;
}

int orc_count_transitions_mt(const int32_t* paths, int64_t T, int32_t L, int32_t E,
                             int32_t gap, int64_t* counts, int64_t* row_totals,
                             int32_t threads) {
    if (threads <= 1) return orc_count_transitions(paths, T, L, E, gap, counts, row_totals);
    int rc = orc_validate_trace(paths, T, L, E);
    if (rc) return rc;
    if (gap < 1 || gap > L - 1) return fail("gap out of range");
    const int32_t pairs = L - gap;
    const size_t n = (size_t)pairs * E * E;
    pthread_t* tid = (pthread_t*)malloc(sizeof(pthread_t) * threads);
    hist_job* jobs = (hist_job*)malloc(sizeof(hist_job) * threads);
    for (int i = 0; i < threads; ++i) {
        jobs[i].paths = paths;
        jobs[i].t0 = T * i / threads;
        jobs[i].t1 = T * (i + 1) / threads;
        jobs[i].L = L;
        jobs[i].E = E;
        jobs[i].gap = gap;
        jobs[i].counts = (int64_t*)calloc(n, sizeof(int64_t));
        pthread_create(&tid[i], NULL, hist_worker, &jobs[i]);
    }
    memset(counts, 0, sizeof(int64_t) * n);
    for (int i = 0; i < threads; ++i) {
        pthread_join(tid[i], NULL);
        for (size_t k = 0; k < n; ++k) counts[k] += jobs[i].counts[k];
        free(jobs[i].counts);
    }
    free(jobs);
    free(tid);
    if (row_totals) {
        for (int32_t j = 0; j < pairs; ++j)
            for (int32_t a = 0; a < E; ++a) {
                int64_t s = 0;
                for (int32_t b = 0; b < E; ++b) s += counts[((int64_t)j * E + a) * E + b];
                row_totals[(int64_t)j * E + a] = s;
            }
    }
    return 0;
}

void orc_conditional_probabilities(const int64_t* counts, const int64_t* row_totals,
                                   int32_t pairs, int32_t E, double* probs,
                                   uint8_t* seen) { /* trace.cpp:217-240 */
    for (int32_t j = 0; j < pairs; ++j)
        for (int32_t a = 0; a < E; ++a) {
            const int64_t tot = row_totals[(int64_t)j * E + a];
            seen[(int64_t)j * E + a] = tot > 0;
            for (int32_t b = 0; b < E; ++b) {
                const int64_t idx = ((int64_t)j * E + a) * E + b;
                probs[idx] = tot > 0 ? (double)counts[idx] / (double)tot : 0.0;
            }
        }
}

int orc_most_affiliated(const double* probs, const uint8_t* seen, int32_t pairs,
                        int32_t E, int32_t source_layer, int32_t expert) { /* trace.cpp:242-260 */
    if (source_layer < 0 || source_layer >= pairs) return -fail("source layer out of range");
    if (expert < 0 || expert >= E) return -fail("expert out of range");
    if (!seen[(int64_t)source_layer * E + expert]) return -fail("no observations");
    const double* row = probs + ((int64_t)source_layer * E + expert) * E;
    int32_t best = 0; /* first maximum wins: lowest-index tie-break */
    for (int32_t b = 1; b < E; ++b)
        if (row[b] > row[best]) best = b;
    return best;
}

int orc_permute_experts(const int32_t* paths, int64_t T, int32_t L, int32_t E,
                        const int32_t* perm, int32_t* out) { /* trace.cpp:285-304 */
    int rc = orc_validate_trace(paths, T, L, E);
    if (rc) return rc;
    uint8_t* hit = (uint8_t*)calloc((size_t)E, 1);
    for (int32_t e = 0; e < E; ++e) {
        if (perm[e] < 0 || perm[e] >= E || hit[perm[e]]) {
            free(hit);
            return fail("not a permutation of [0,E)");
        }
        hit[perm[e]] = 1;
    }
    free(hit);
    for (int64_t i = 0; i < T * (int64_t)L; ++i) out[i] = perm[paths[i]];
    return 0;
}

/* ------------------------------------------------------------------------
 * placement -- src/placement.cpp:434-526, 618-667
 * ---------------------------------------------------------------------- */
int orc_validate_placement(const int32_t* assign, int32_t L, int32_t E, int32_t gpus) {
    /* placement.cpp:434-470 */
    if (E < 1 || L < 1) return fail("placement must cover at least one expert and layer");
    if (E % gpus != 0) return fail("num_experts not divisible by total GPUs");
    const int32_t cap = E / gpus;
    int32_t* load = (int32_t*)malloc(sizeof(int32_t) * gpus);
    for (int32_t j = 0; j < L; ++j) {
        memset(load, 0, sizeof(int32_t) * gpus);
        for (int32_t i = 0; i < E; ++i) {
            const int32_t g = assign[j * E + i];
            if (g < 0 || g >= gpus) {
                free(load);
                return fail("gpu id out of range");
            }
            load[g]++;
        }
        for (int32_t g = 0; g < gpus; ++g)
            if (load[g] != cap) {
                free(load);
                return fail("placement imbalance");
            }
    }
    free(load);
    return 0;
}

int orc_contiguous_placement(int32_t E, int32_t L, int32_t gpus, int32_t* assign) {
    /* placement.cpp:482-502: expert i -> gpu i / (E/G) on every layer */
    if (gpus < 1 || E % gpus != 0) return fail("num_experts not divisible by total GPUs");
    const int32_t cap = E / gpus;
    for (int32_t j = 0; j < L; ++j)
        for (int32_t i = 0; i < E; ++i) assign[j * E + i] = i / cap;
    return 0;
}

int orc_random_placement(int32_t E, int32_t L, int32_t gpus, uint64_t seed,
                         int32_t* assign) {
    /* placement.cpp:504-526 with random_balanced :222-226 */
    if (gpus < 1 || E % gpus != 0) return fail("num_experts not divisible by total GPUs");
    const int32_t cap = E / gpus;
    orc_rng r;
    orc_rng_init(&r, seed);
    for (int32_t j = 0; j < L; ++j) {
        int32_t* row = assign + (int64_t)j * E;
        for (int32_t i = 0; i < E; ++i) row[i] = i / cap;
        orc_shuffle_int(row, E, &r);
    }
    return 0;
}

double orc_objective_crossings(const int64_t* counts, int32_t pairs, int32_t E,
                               int32_t gap, const int32_t* assign,
                               int32_t gpus_per_node, int32_t level_node) {
    /* placement.cpp:618-643 */
    double total = 0.0;
    for (int32_t j = 0; j < pairs; ++j)
        for (int32_t a = 0; a < E; ++a)
            for (int32_t b = 0; b < E; ++b) {
                const int64_t w = counts[((int64_t)j * E + a) * E + b];
                if (w == 0) continue;
                int32_t from = assign[j * E + a];
                int32_t to = assign[(j + gap) * E + b];
                if (level_node) {
                    from /= gpus_per_node;
                    to /= gpus_per_node;
                }
                if (from != to) total += (double)w;
            }
    return total;
}

int64_t orc_balanced_assignment_count(int32_t items, int32_t parts, int64_t cap) {
    /* placement.cpp:645-667 */
    if (parts < 1 || items < 1 || items % parts != 0) return -1;
    const int32_t k = items / parts;
    unsigned __int128 product = 1;
    int32_t remaining = items;
    for (int32_t p = 0; p < parts; ++p) {
        unsigned __int128 binom = 1;
        for (int32_t i = 1; i <= k; ++i) {
            binom = binom * (unsigned)(remaining - k + i) / (unsigned)i;
            if (binom > (unsigned __int128)cap * 2 + 2) return cap + 1;
        }
        product *= binom;
        if (product > (unsigned __int128)cap) return cap + 1;
        remaining -= k;
    }
    return (int64_t)product;
}

/* next_permutation over a sorted int pattern (lexicographic), as used by
 * tests/oracle_util.hpp:18-28 */
static int next_perm(int32_t* a, int32_t n) {
    int32_t i = n - 2;
    while (i >= 0 && a[i] >= a[i + 1]) --i;
    if (i < 0) return 0;
    int32_t j = n - 1;
    while (a[j] <= a[i]) --j;
    int32_t t = a[i]; a[i] = a[j]; a[j] = t;
    for (int32_t l = i + 1, r = n - 1; l < r; ++l, --r) {
        t = a[l]; a[l] = a[r]; a[r] = t;
    }
    return 1;
}

double orc_brute_force_optimum(const int64_t* counts, int32_t L, int32_t E,
                               int32_t parts) {
    /* tests/oracle_util.hpp:18-65: all S^L labeled balanced placements */
    int32_t pattern[64];
    if (E > 64 || E % parts != 0) return -1.0;
    for (int32_t i = 0; i < E; ++i) pattern[i] = i / (E / parts);
    int64_t S = 0, capS = 4096;
    int32_t* all = (int32_t*)malloc(sizeof(int32_t) * E * capS);
    do {
        if (S == capS) {
            capS *= 2;
            all = (int32_t*)realloc(all, sizeof(int32_t) * E * capS);
        }
        memcpy(all + S * E, pattern, sizeof(int32_t) * E);
        ++S;
    } while (next_perm(pattern, E));
    int64_t* odo = (int64_t*)calloc((size_t)L, sizeof(int64_t));
    double best = INFINITY;
    for (;;) {
        double cost = 0.0;
        for (int32_t j = 0; j + 1 < L; ++j) {
            const int32_t* s = all + odo[j] * E;
            const int32_t* t = all + odo[j + 1] * E;
            for (int32_t a = 0; a < E; ++a)
                for (int32_t b = 0; b < E; ++b) {
                    const int64_t w = counts[((int64_t)j * E + a) * E + b];
                    if (w > 0 && s[a] != t[b]) cost += (double)w;
                }
        }
        if (cost < best) best = cost;
        int32_t j = L - 1;
        while (j >= 0 && ++odo[j] == S) odo[j--] = 0;
        if (j < 0) break;
    }
    free(odo);
    free(all);
    return best;
}

/* ------------------------------------------------------------------------
 * comm simulator -- src/sim.cpp:34-191
 * ---------------------------------------------------------------------- */
static int tier_between(int32_t a, int32_t b, int32_t gpn) { /* sim.cpp:15-20 */
    if (a == b) return 0;
    return (a / gpn) == (b / gpn) ? 1 : 2;
}

int orc_token_hops(const int32_t* path, int32_t L, int32_t home,
                   const int32_t* assign, int32_t E, int32_t num_nodes,
                   int32_t gpus_per_node, int32_t mode, int32_t* hops_out,
                   int32_t* crossed_out, int32_t* tier_out) {
    /* sim.cpp:34-76 */
    const int32_t gpus = num_nodes * gpus_per_node;
    if (home < 0 || home >= gpus) return fail("home gpu out of range");
    int32_t location = home;
    for (int32_t j = 0; j < L; ++j) {
        const int32_t expert = path[j];
        if (expert < 0 || expert >= E) return fail("expert id out of range in path");
        const int32_t eg = assign[j * E + expert];
        int32_t crossed, tier, hops;
        if (mode == ORC_VANILLA) { /* sim.cpp:60-64 */
            crossed = eg != home;
            tier = tier_between(home, eg, gpus_per_node);
            hops = crossed ? 2 : 0;
        } else { /* sim.cpp:65-71 */
            crossed = eg != location;
            tier = tier_between(location, eg, gpus_per_node);
            hops = crossed ? 1 : 0;
            location = eg;
        }
        hops_out[j] = hops;
        if (crossed_out) crossed_out[j] = crossed;
        if (tier_out) tier_out[j] = tier;
    }
    return 0;
}

typedef struct {
    const int32_t* paths;
    const int32_t* homes;
    const int32_t* assign;
    int64_t t0, t1;
    int32_t L, E, gpn, gpus, mode;
    int64_t c[6]; /* gpu_local node_local away moves hops_intra hops_inter */
} sim_job;

static void sim_range(sim_job* job) {
    const int32_t L = job->L, E = job->E, gpn = job->gpn;
    int64_t gl = 0, nl = 0, away = 0, moves = 0, hi = 0, he = 0;
    /* HOT LOOP sim.cpp:110-145 */
    for (int64_t t = job->t0; t < job->t1; ++t) {
        const int32_t home = job->homes ? job->homes[t] : (int32_t)(t % job->gpus);
        int32_t location = home;
        const int32_t* p = job->paths + t * L;
        for (int32_t j = 0; j < L; ++j) {
            const int32_t eg = job->assign[j * E + p[j]];
            if (eg == location) ++gl;
            if (eg / gpn == location / gpn) ++nl;
            if (eg != home) ++away;
            if (eg != location) {
                ++moves;
                if (job->mode == ORC_COHERENT) {
                    if (tier_between(location, eg, gpn) == 2) ++he; else ++hi;
                }
            }
            if (job->mode == ORC_VANILLA && eg != home) {
                if (tier_between(home, eg, gpn) == 2) he += 2; else hi += 2;
            }
            location = eg;
        }
    }
    job->c[0] = gl; job->c[1] = nl; job->c[2] = away;
    job->c[3] = moves; job->c[4] = hi; job->c[5] = he;
}

static void* sim_worker(void* arg) {
    sim_range((sim_job*)arg);
    return NULL;
}

double orc_volume_table1(int32_t gpus, int32_t tokens_per_gpu, int32_t layers,
                         double ratio, int32_t gating, int32_t method) {
    /* sim.cpp:171-191 */
    if (gpus < 1 || tokens_per_gpu < 1 || layers < 1) return NAN;
    if (!(ratio >= 0.0 && ratio <= 1.0)) return NAN;
    const double g = gpus, n = tokens_per_gpu, l = layers;
    if (method != 3) return (gating == 0 ? 2.0 : 4.0) * g * n * l * ratio;
    return gating == 0 ? g * n * (l * ratio + g) : g * n * (2.0 * l * ratio + g);
}

int orc_simulate_mt(const int32_t* paths, int64_t T, int32_t L, int32_t E,
                    const int32_t* assign, int32_t num_nodes, int32_t gpus_per_node,
                    double intra_cost, double inter_cost, int32_t tokens_per_gpu,
                    int32_t mode, const int32_t* homes, orc_sim_report* out,
                    int32_t threads) {
    int rc = orc_validate_trace(paths, T, L, E);
    if (rc) return rc;
    const int32_t gpus = num_nodes * gpus_per_node;
    if (num_nodes < 1 || gpus_per_node < 1) return fail("topology must have at least one node and one GPU per node");
    if (intra_cost < 0.0 || inter_cost < intra_cost) return fail("hop costs must satisfy inter >= intra >= 0");
    if (tokens_per_gpu < 1) return fail("tokens_per_gpu must be >= 1");
    rc = orc_validate_placement(assign, L, E, gpus);
    if (rc) return rc;
    if (homes)
        for (int64_t t = 0; t < T; ++t)
            if (homes[t] < 0 || homes[t] >= gpus) return fail("home gpu out of range");
    if (threads < 1) threads = 1;
    sim_job* jobs = (sim_job*)calloc((size_t)threads, sizeof(sim_job));
    pthread_t* tid = (pthread_t*)malloc(sizeof(pthread_t) * threads);
    for (int i = 0; i < threads; ++i) {
        jobs[i].paths = paths; jobs[i].homes = homes; jobs[i].assign = assign;
        jobs[i].t0 = T * i / threads; jobs[i].t1 = T * (i + 1) / threads;
        jobs[i].L = L; jobs[i].E = E; jobs[i].gpn = gpus_per_node;
        jobs[i].gpus = gpus; jobs[i].mode = mode;
        if (threads > 1) pthread_create(&tid[i], NULL, sim_worker, &jobs[i]);
    }
    if (threads == 1) sim_range(&jobs[0]);
    int64_t c[6] = {0, 0, 0, 0, 0, 0};
    for (int i = 0; i < threads; ++i) {
        if (threads > 1) pthread_join(tid[i], NULL);
        for (int k = 0; k < 6; ++k) c[k] += jobs[i].c[k];
    }
    free(jobs);
    free(tid);
    memset(out, 0, sizeof(*out));
    out->gpu_local_events = c[0];
    out->node_local_events = c[1];
    out->away_from_home_events = c[2];
    out->coherent_moves = c[3];
    out->hops_intra_node = c[4];
    out->hops_inter_node = c[5];
    const double events = (double)T * L; /* sim.cpp:147-151 */
    out->locality_gpu = c[0] / events;
    out->locality_node = c[1] / events;
    out->p = c[2] / events;
    out->p_star = c[3] / events;
    if (mode == ORC_VANILLA) { /* sim.cpp:153-157 */
        out->alltoall_count = 2L * L;
        out->volume_units = orc_volume_table1(gpus, tokens_per_gpu, L, out->p, 0, 0);
    } else { /* sim.cpp:158-165 */
        out->alltoall_count = L;
        out->allgather_count = 1;
        out->setup_allgather_count = 1;
        out->volume_units = orc_volume_table1(gpus, tokens_per_gpu, L, out->p_star, 0, 3);
    }
    out->estimated_latency = c[4] * intra_cost + c[5] * inter_cost; /* sim.cpp:166-167 */
    return 0;
}

int orc_simulate(const int32_t* paths, int64_t T, int32_t L, int32_t E,
                 const int32_t* assign, int32_t num_nodes, int32_t gpus_per_node,
                 double intra_cost, double inter_cost, int32_t tokens_per_gpu,
                 int32_t mode, const int32_t* homes, orc_sim_report* out) {
    return orc_simulate_mt(paths, T, L, E, assign, num_nodes, gpus_per_node, intra_cost,
                           inter_cost, tokens_per_gpu, mode, homes, out, 1);
}
