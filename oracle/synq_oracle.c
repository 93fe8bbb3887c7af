/* synq_oracle.c — plain-C restatement of the reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see synq_oracle.h).  Every function names the
 * reference lines it restates.  Paths are relative to /root/reference/proj.
 * Compiled with -ffp-contract=off: the reference library carries no FMA
 * (built without -march), so neither may its checker.
 */
#include "synq_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ RNG */

/* include/synq/random.hpp:10-15 */
uint64_t so_splitmix64(uint64_t* state) {
    uint64_t z = (*state += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

/* include/synq/random.hpp:17-20 */
uint64_t so_derive_seed(uint64_t master, uint64_t index) {
    uint64_t s = master ^ (0xd1b54a32d192ed03ull * (index + 1));
    return so_splitmix64(&s);
}

/* include/synq/random.hpp:32-41 */
void so_xs_seed(so_xorshift* r, uint64_t seed) {
    uint64_t s = seed;
    uint64_t a = so_splitmix64(&s);
    uint64_t b = so_splitmix64(&s);
    r->x = (uint32_t)a;
    r->y = (uint32_t)(a >> 32);
    r->z = (uint32_t)b;
    r->w = (uint32_t)(b >> 32);
    if ((r->x | r->y | r->z | r->w) == 0) r->w = 0x6b43a9b5u;
}

/* include/synq/random.hpp:43-50 (Marsaglia xor128) */
uint32_t so_xs_next(so_xorshift* r) {
    uint32_t t = r->x ^ (r->x << 11);
    r->x = r->y;
    r->y = r->z;
    r->z = r->w;
    r->w = r->w ^ (r->w >> 19) ^ (t ^ (t >> 8));
    return r->w;
}

/* include/synq/random.hpp:53-55: (u + 1) * 2^-32, in (0, 1] */
double so_xs_uniform01(so_xorshift* r) { return ((double)so_xs_next(r) + 1.0) * 0x1p-32; }

/* include/synq/random.hpp:65-68 */
static uint64_t so_geometric(double p, so_xorshift* r) {
    double denom = log1p(-p);
    return (uint64_t)floor(log(so_xs_uniform01(r)) / denom);
}

/* include/synq/random.hpp:72-82 */
uint32_t so_binomial(uint32_t m, double p, so_xorshift* r) {
    if (p <= 0.0 || m == 0) return 0;
    if (p >= 1.0) return m;
    uint32_t count = 0;
    uint64_t pos = so_geometric(p, r);
    while (pos < m) {
        ++count;
        pos += 1 + so_geometric(p, r);
    }
    return count;
}

void so_xs_fill(uint64_t seed, uint32_t* out, size_t n) {
    so_xorshift r;
    so_xs_seed(&r, seed);
    for (size_t i = 0; i < n; ++i) out[i] = so_xs_next(&r);
}

void so_binomial_fill(uint64_t seed, uint32_t m, double p, uint32_t* out, size_t n) {
    so_xorshift r;
    so_xs_seed(&r, seed);
    for (size_t i = 0; i < n; ++i) out[i] = so_binomial(m, p, &r);
}

/* --------------------------------------------------------- construction */

/* include/synq/adjacency.hpp:112-163, with the uniform source abstracted:
 * draws[i] for i < n+2 are the uniforms the generator consumes in order. */
static void sorted_random_core(uint32_t n, uint32_t a, uint32_t b, double* pos, uint32_t* out,
                               double* trace) {
    const uint32_t span = b - a;
    double sum = 0.0;
    /* exclusive running sum of -ln(u) (adjacency.hpp:138-143) */
    for (uint32_t i = 0; i < n + 2; ++i) {
        double e = -log(pos[i]);
        if (trace) trace[i] = e;
        pos[i] = sum;
        sum += e;
    }
    double total = pos[n + 1];
    if (total <= 0.0) total = 1.0; /* adjacency.hpp:147 */
    const double scale = (double)(span - n);
    if (trace) {
        for (uint32_t i = 0; i < n + 2; ++i) {
            trace[(n + 2) + i] = pos[i];
            trace[2 * (n + 2) + i] = pos[i] / total;
            trace[3 * (n + 2) + i] = floor(pos[i] / total * scale + 0.5);
        }
    }
    /* adjacency.hpp:158-161: round half up, then add the rank offset */
    for (uint32_t i = 0; i < n; ++i) {
        double v = pos[i + 1] / total * scale;
        out[i] = a + (uint32_t)floor(v + 0.5) + i;
    }
}

int so_sorted_random(uint32_t n, uint32_t a, uint32_t b, so_xorshift* rng, uint32_t* out) {
    if (b <= a || n > b - a) return -1; /* adjacency.hpp:115-117 */
    double* pos = (double*)malloc(sizeof(double) * (n + 2));
    for (uint32_t i = 0; i < n + 2; ++i) pos[i] = so_xs_uniform01(rng);
    sorted_random_core(n, a, b, pos, out, NULL);
    free(pos);
    return 0;
}

int so_sorted_random_replay(uint32_t n, uint32_t a, uint32_t b, const double* draws,
                            uint32_t* out, double* trace) {
    if (b <= a || n > b - a) return -1;
    double* pos = (double*)malloc(sizeof(double) * (n + 2));
    memcpy(pos, draws, sizeof(double) * (n + 2));
    sorted_random_core(n, a, b, pos, out, trace);
    free(pos);
    return 0;
}

static uint32_t desc_neurons(const so_desc* d) {
    uint64_t t = 0;
    for (uint32_t i = 0; i < d->npops; ++i) t += d->pop[i];
    return (uint32_t)t;
}

/* src/network_desc.cpp:15-22 */
static void id_range(const so_desc* d, uint32_t pop, uint32_t* lo, uint32_t* hi) {
    uint32_t first = 0;
    for (uint32_t i = 0; i < pop; ++i) first += d->pop[i];
    *lo = first;
    *hi = first + d->pop[pop];
}

/* src/adjacency.cpp:29-71 plan_jobs: one binomial per (connection, source)
 * on a single master stream derive_seed(seed, 0); jobs grouped per source in
 * connection order; offsets tile each source's row. */
static so_graph* plan(const so_desc* d, uint64_t seed, uint32_t pitch_align) {
    so_graph* g = (so_graph*)calloc(1, sizeof(so_graph));
    const uint32_t n = desc_neurons(d);
    g->neurons = n;
    g->degree = (uint32_t*)calloc(n ? n : 1, sizeof(uint32_t));
    so_xorshift rng;
    so_xs_seed(&rng, so_derive_seed(seed, 0));

    /* per-source job counts, to lay out source-major order */
    uint32_t* njob_src = (uint32_t*)calloc(n ? n : 1, sizeof(uint32_t));
    for (uint32_t ci = 0; ci < d->nconn; ++ci) {
        uint32_t sa, sb;
        id_range(d, d->csrc[ci], &sa, &sb);
        for (uint32_t s = sa; s < sb; ++s) njob_src[s]++;
    }
    uint64_t* first = (uint64_t*)calloc((size_t)n + 1, sizeof(uint64_t));
    for (uint32_t s = 0; s < n; ++s) first[s + 1] = first[s] + njob_src[s];
    g->njobs = first[n];
    g->jobs = (so_job*)calloc(g->njobs ? g->njobs : 1, sizeof(so_job));
    uint32_t* fill = (uint32_t*)calloc(n ? n : 1, sizeof(uint32_t));

    for (uint32_t ci = 0; ci < d->nconn; ++ci) {
        uint32_t sa, sb, ta, tb;
        id_range(d, d->csrc[ci], &sa, &sb);
        id_range(d, d->cdst[ci], &ta, &tb);
        const uint32_t span = tb - ta;
        for (uint32_t s = sa; s < sb; ++s) {
            uint32_t k = so_binomial(span, d->cp[ci], &rng);
            g->degree[s] += k;
            so_job* j = &g->jobs[first[s] + fill[s]++];
            j->n = k;
            j->a = ta;
            j->b = tb;
        }
    }
    for (uint32_t i = 0; i < n; ++i)
        if (g->degree[i] > g->deg_max) g->deg_max = g->degree[i];
    if (pitch_align == 0) pitch_align = 1;
    g->pitch = (g->deg_max + pitch_align - 1) / pitch_align * pitch_align;
    for (uint32_t s = 0; s < n; ++s) {
        uint64_t o = (uint64_t)s * g->pitch;
        for (uint64_t q = first[s]; q < first[s + 1]; ++q) {
            g->jobs[q].o = o;
            o += g->jobs[q].n;
            g->edges += g->jobs[q].n;
        }
    }
    free(njob_src);
    free(first);
    free(fill);
    return g;
}

so_graph* so_plan_graph(const so_desc* d, uint64_t seed, uint32_t pitch_align) {
    return plan(d, seed, pitch_align);
}

static int cmp_u32(const void* a, const void* b) {
    uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
    return x < y ? -1 : x > y;
}

/* src/adjacency.cpp:73-103 expand_jobs: job j reseeds derive_seed(seed, j+1),
 * writes sorted_random at its offset; then every row is sorted. */
so_graph* so_build_graph(const so_desc* d, uint64_t seed, uint32_t pitch_align) {
    so_graph* g = plan(d, seed, pitch_align);
    size_t cells = (size_t)g->neurons * g->pitch;
    g->cells = (uint32_t*)malloc(sizeof(uint32_t) * (cells ? cells : 1));
    memset(g->cells, 0xff, sizeof(uint32_t) * cells);
    for (uint64_t j = 0; j < g->njobs; ++j) {
        const so_job* job = &g->jobs[j];
        if (job->n == 0) continue;
        so_xorshift r;
        so_xs_seed(&r, so_derive_seed(seed, j + 1));
        so_sorted_random(job->n, job->a, job->b, &r, g->cells + job->o);
    }
    for (uint32_t s = 0; s < g->neurons; ++s)
        qsort(g->cells + (size_t)s * g->pitch, g->degree[s], sizeof(uint32_t), cmp_u32);
    return g;
}

void so_graph_free(so_graph* g) {
    if (!g) return;
    free(g->jobs);
    free(g->degree);
    free(g->cells);
    free(g);
}

/* ------------------------------------------------------------ models */

/* include/synq/models/lif.hpp:13-20 */
typedef struct lif_p {
    float tau_m, v_rest, v_reset, v_threshold, refractory, background;
} lif_p;

/* include/synq/models/lif.hpp:66-76 */
typedef struct stdp_p {
    float a_plus, a_minus, tau_plus, tau_minus, w_min, w_max, decay_plus, decay_minus;
} stdp_p;

struct so_sim {
    int model;
    so_desc desc;
    so_graph* g;
    uint32_t n, delay, history, bframes, words;
    float dt;
    uint64_t seed;
    /* model constants (include/synq/models/benchmarks.hpp) */
    lif_p lif;
    float w_exc, w_inh, scale_c, p_spike, v_init_lo, v_init_hi;
    uint32_t n_exc, n_recurrent, first_pop;
    stdp_p stdp;
    /* state */
    float *V, *ACC, *REF;
    uint8_t* flag;
    so_xorshift* rng;
    float *W, *PT, *QT;
    uint32_t* ages;
    uint32_t* expiring;
    uint32_t expiring_count;
    uint32_t* qentries; /* delay frames x n */
    uint32_t* qcount;
    uint64_t* bits; /* bframes x words */
    int64_t t;
    uint64_t counters[6];
    /* frame log */
    uint32_t* log;
    uint64_t log_words, log_cap;
};

static int has_syn(const so_sim* s) { return s->model == SO_BRUNEL_PLUS; }
static int uses_rng(const so_sim* s) { return s->model != SO_PINGPONG; }

/* include/synq/spike_ring.hpp:85-89 */
static int bit(const so_sim* s, int64_t u, uint32_t id) {
    if (u < 0 || s->bframes == 0) return 0;
    const uint64_t* w = s->bits + (size_t)(u % s->bframes) * s->words;
    return (int)((w[id >> 6] >> (id & 63)) & 1u);
}

static uint32_t rounded(double x) { return (uint32_t)llround(x); }

/* src/benchmarks.cpp:140-158 brunel_desc */
static void brunel_desc(uint32_t neurons, so_desc* d) {
    uint32_t ne = rounded(0.4 * neurons), ni = rounded(0.1 * neurons);
    memset(d, 0, sizeof *d);
    d->npops = 3;
    d->pop[0] = ne;
    d->pop[1] = ni;
    d->pop[2] = neurons - ne - ni;
    const uint32_t cs[6] = {0, 0, 1, 1, 2, 2}, cd[6] = {0, 1, 0, 1, 0, 1};
    d->nconn = 6;
    for (int i = 0; i < 6; ++i) {
        d->csrc[i] = cs[i];
        d->cdst[i] = cd[i];
        d->cp[i] = 0.1;
    }
    d->dt = 0.1;
    d->delay = rounded(15.0);
}

/* src/benchmarks.cpp:82-96 build_vogels */
static void vogels_desc(uint32_t neurons, so_desc* d) {
    uint32_t ne = rounded(0.8 * neurons);
    memset(d, 0, sizeof *d);
    d->npops = 2;
    d->pop[0] = ne;
    d->pop[1] = neurons - ne;
    const uint32_t cs[4] = {0, 0, 1, 1}, cd[4] = {0, 1, 0, 1};
    d->nconn = 4;
    for (int i = 0; i < 4; ++i) {
        d->csrc[i] = cs[i];
        d->cdst[i] = cd[i];
        d->cp[i] = 0.02;
    }
    d->dt = 0.1;
    d->delay = rounded(8.0);
}

/* src/benchmarks.cpp:52-61 build_pingpong */
static void pingpong_desc(so_desc* d) {
    memset(d, 0, sizeof *d);
    d->npops = 2;
    d->pop[0] = d->pop[1] = rounded(100.0);
    d->nconn = 2;
    d->csrc[0] = 0;
    d->cdst[0] = 1;
    d->cp[0] = 0.01;
    d->csrc[1] = 1;
    d->cdst[1] = 0;
    d->cp[1] = 0.01;
    d->dt = 1.0;
    d->delay = rounded(1.0);
}

static double conn_p(const so_desc* d, uint32_t src, uint32_t dst) {
    for (uint32_t i = 0; i < d->nconn; ++i)
        if (d->csrc[i] == src && d->cdst[i] == dst) return d->cp[i];
    return 0.0;
}

/* model parameterisation from desc (src/benchmarks.cpp:40-199, defaults
 * src/params.cpp:8-56) */
static void parameterise(so_sim* s) {
    const so_desc* d = &s->desc;
    double n = (double)s->n;
    if (s->model == SO_PINGPONG) {
        s->first_pop = d->pop[0]; /* benchmarks.cpp:44 */
        return;
    }
    if (s->model == SO_VOGELS) {
        s->lif = (lif_p){20.0f, -49.0f, -60.0f, -50.0f, 5.0f, 0.0f};
        s->w_exc = 0.4f;
        s->w_inh = -2.2f;
        s->n_exc = d->pop[0];
        s->v_init_lo = -60.0f;
        s->v_init_hi = -50.0f;
        s->scale_c = (float)(16000000.0 / (n * n)); /* analysis.cpp:32 */
        return;
    }
    /* brunel / brunel+: fill_brunel_common (benchmarks.cpp:105-138) */
    s->lif = (lif_p){20.0f, 0.0f, 10.0f, 20.0f, 2.0f, 0.0f};
    const double j = 0.1, g = 5.0, eta = 2.0;
    uint32_t ne = d->pop[0], ni = d->pop[1], ns = d->pop[2];
    s->w_exc = (float)j;
    s->w_inh = (float)(-g * j);
    s->n_exc = ne;
    s->n_recurrent = ne + ni;
    s->v_init_hi = s->lif.v_threshold;
    double scale = 20000.0 / n; /* analysis.cpp:34 */
    s->scale_c = (float)scale;
    double c_e = conn_p(d, 0, 0) * ne;
    double c_p = conn_p(d, 2, 0) * ns;
    double theta = s->lif.v_threshold - s->lif.v_rest;
    double tau_s = s->lif.tau_m / 1000.0;
    double rate_thr_hz = theta / (j * scale * c_e * tau_s);
    double rate_p_hz = eta * rate_thr_hz * c_e / c_p;
    double p_spike = rate_p_hz / 1000.0 * d->dt;
    s->p_spike = (float)p_spike;
    if (s->model == SO_BRUNEL_PLUS) {
        /* benchmarks.cpp:183-191, lif.hpp:72-75 bind(dt) uses float exp */
        s->stdp = (stdp_p){0.01f, 0.0105f, 20.0f, 20.0f, 0.0f, 0.3f, 1.0f, 1.0f};
        float dtf = (float)d->dt;
        s->stdp.decay_plus = expf(-dtf / s->stdp.tau_plus);
        s->stdp.decay_minus = expf(-dtf / s->stdp.tau_minus);
    }
}

static float weight_of(const so_sim* s, uint32_t src) {
    if (s->model == SO_VOGELS) return src < s->n_exc ? s->w_exc : s->w_inh;
    /* benchmarks.hpp:90-92 */
    return src < s->n_exc ? s->w_exc : (src < s->n_recurrent ? s->w_inh : s->w_exc);
}

/* engine.hpp:154-186 init() */
static void sim_init(so_sim* s) {
    s->t = 0;
    memset(s->counters, 0, sizeof s->counters);
    memset(s->qcount, 0, sizeof(uint32_t) * s->delay);
    if (s->bits) memset(s->bits, 0, sizeof(uint64_t) * (size_t)s->bframes * s->words);
    s->expiring_count = 0;
    if (uses_rng(s))
        for (uint32_t i = 0; i < s->n; ++i)
            so_xs_seed(&s->rng[i], so_derive_seed(s->seed, (1ull << 32) + i));
    for (uint32_t i = 0; i < s->n; ++i) {
        switch (s->model) {
            case SO_PINGPONG: /* benchmarks.hpp:22-25 */
                s->flag[i] = i < s->first_pop ? 1 : 0;
                break;
            case SO_VOGELS: /* benchmarks.hpp:53-59 */
                s->V[i] = s->v_init_lo +
                          (float)so_xs_uniform01(&s->rng[i]) * (s->v_init_hi - s->v_init_lo);
                s->ACC[i] = 0.0f;
                s->REF[i] = 0.0f;
                break;
            default: /* benchmarks.hpp:94-99 */
                s->V[i] = (float)so_xs_uniform01(&s->rng[i]) * s->v_init_hi;
                s->ACC[i] = 0.0f;
                s->REF[i] = 0.0f;
        }
    }
    if (has_syn(s)) {
        /* engine.hpp:172-185 + benchmarks.hpp:122-127 */
        memset(s->ages, 0, sizeof(uint32_t) * s->n);
        for (uint32_t i = 0; i < s->n; ++i) {
            size_t base = (size_t)i * s->g->deg_max;
            for (uint32_t k = 0; k < s->g->degree[i]; ++k) {
                s->W[base + k] = weight_of(s, i);
                s->PT[base + k] = 0.0f;
                s->QT[base + k] = 0.0f;
            }
        }
    }
}

/* d_param parameterises the model (benchmarks.cpp runs on the descriptor
 * before sim_runtime.cpp:22-23 applies dt/delay overrides); d is the
 * descriptor the engine actually runs. */
static so_sim* sim_alloc(int model, const so_desc* d_param, const so_desc* d, uint64_t seed,
                         uint32_t history_frames) {
    so_sim* s = (so_sim*)calloc(1, sizeof(so_sim));
    s->model = model;
    s->desc = *d_param;
    s->seed = seed;
    s->n = desc_neurons(d);
    parameterise(s);
    s->desc = *d;
    s->dt = (float)d->dt; /* engine.hpp:123 */
    s->delay = d->delay;
    s->g = so_build_graph(d, seed, 32);
    if (has_syn(s)) { /* engine.hpp:135-139 */
        uint32_t floor_ = s->delay + 1;
        s->history = history_frames ? (history_frames > floor_ ? history_frames : floor_)
                                    : (floor_ > 50 ? floor_ : 50);
    }
    s->bframes = has_syn(s) ? s->history : 0;
    s->words = (s->n + 63) / 64;
    s->qentries = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)s->delay * (s->n ? s->n : 1));
    s->qcount = (uint32_t*)calloc(s->delay, sizeof(uint32_t));
    if (s->bframes) s->bits = (uint64_t*)calloc((size_t)s->bframes * s->words, sizeof(uint64_t));
    size_t n1 = s->n ? s->n : 1;
    if (model == SO_PINGPONG) {
        s->flag = (uint8_t*)calloc(n1, 1);
    } else {
        s->V = (float*)calloc(n1, sizeof(float));
        s->ACC = (float*)calloc(n1, sizeof(float));
        s->REF = (float*)calloc(n1, sizeof(float));
        s->rng = (so_xorshift*)calloc(n1, sizeof(so_xorshift));
    }
    if (has_syn(s)) {
        size_t cap = (size_t)s->n * s->g->deg_max;
        s->W = (float*)calloc(cap ? cap : 1, sizeof(float));
        s->PT = (float*)calloc(cap ? cap : 1, sizeof(float));
        s->QT = (float*)calloc(cap ? cap : 1, sizeof(float));
        s->ages = (uint32_t*)calloc(n1, sizeof(uint32_t));
        s->expiring = (uint32_t*)calloc(n1, sizeof(uint32_t));
    }
    sim_init(s);
    return s;
}

so_sim* so_sim_new_desc(int model, const so_desc* d, uint64_t seed, uint32_t history_frames) {
    return sim_alloc(model, d, d, seed, history_frames);
}

so_sim* so_sim_new(int model, uint32_t neurons, uint64_t seed, uint32_t history_frames,
                   double dt_override, uint32_t delay_override) {
    so_desc d;
    switch (model) {
        case SO_PINGPONG: pingpong_desc(&d); break;
        case SO_VOGELS: vogels_desc(neurons, &d); break;
        case SO_BRUNEL:
        case SO_BRUNEL_PLUS: brunel_desc(neurons, &d); break;
        default: return NULL;
    }
    so_desc run = d;
    if (dt_override > 0) run.dt = dt_override;
    if (delay_override > 0) run.delay = delay_override;
    return sim_alloc(model, &d, &run, seed, history_frames);
}

void so_sim_free(so_sim* s) {
    if (!s) return;
    so_graph_free(s->g);
    free(s->V);
    free(s->ACC);
    free(s->REF);
    free(s->flag);
    free(s->rng);
    free(s->W);
    free(s->PT);
    free(s->QT);
    free(s->ages);
    free(s->expiring);
    free(s->qentries);
    free(s->qcount);
    free(s->bits);
    free(s->log);
    free(s);
}

/* include/synq/models/lif.hpp:23-42 */
static int lif_update(float* v, float* acc, float* refrac, const lif_p* p, float dt) {
    if (*refrac > 0.0f) {
        *refrac -= dt;
        *v = p->v_reset;
        *acc = 0.0f;
        return 0;
    }
    *v += dt * (-(*v - p->v_rest) / p->tau_m) + *acc + dt * p->background;
    *acc = 0.0f;
    if (*v >= p->v_threshold) {
        *v = p->v_reset;
        *refrac = p->refractory;
        return 1;
    }
    return 0;
}

static float clampf_(float x, float lo, float hi) { return x < lo ? lo : (hi < x ? hi : x); }

/* include/synq/models/lif.hpp:78-89 stdp_step, gated by
 * benchmarks.hpp:120,129-131 plastic(src, dst) */
static void update_synapse(const so_sim* s, uint32_t src, uint32_t dst, float* w, float* pt,
                           float* qt, int pre, int post) {
    if (!(src < s->n_exc && dst < s->n_exc)) return;
    const stdp_p* p = &s->stdp;
    *pt *= p->decay_plus;
    *qt *= p->decay_minus;
    if (pre) *w = clampf_(*w - p->a_minus * *qt, p->w_min, p->w_max);
    if (post) *w = clampf_(*w + p->a_plus * *pt, p->w_min, p->w_max);
    if (pre) *pt += 1.0f;
    if (post) *qt += 1.0f;
}

/* engine.hpp:414-436 catch_up */
static void catch_up(so_sim* s, uint32_t n, int64_t through) {
    const int64_t a0 = s->ages[n];
    if (a0 > through) return;
    const uint32_t* row = s->g->cells + (size_t)n * s->g->pitch;
    const uint32_t deg = s->g->degree[n];
    const size_t base = (size_t)n * s->g->deg_max;
    for (uint32_t k = 0; k < deg; ++k) {
        float w = s->W[base + k], pt = s->PT[base + k], qt = s->QT[base + k];
        for (int64_t u = a0; u <= through; ++u)
            update_synapse(s, n, row[k], &w, &pt, &qt, bit(s, u - (int64_t)s->delay, n),
                           bit(s, u, row[k]));
        s->W[base + k] = w;
        s->PT[base + k] = pt;
        s->QT[base + k] = qt;
    }
    s->counters[3] += (uint64_t)deg * (uint64_t)(through - a0 + 1);
    s->ages[n] = (uint32_t)(through + 1);
}

static void log_frame(so_sim* s, const uint32_t* ids, uint32_t count) {
    if (s->log_words + count + 1 > s->log_cap) {
        uint64_t cap = s->log_cap ? s->log_cap * 2 : 4096;
        while (cap < s->log_words + count + 1) cap *= 2;
        s->log = (uint32_t*)realloc(s->log, sizeof(uint32_t) * cap);
        s->log_cap = cap;
    }
    s->log[s->log_words++] = count;
    memcpy(s->log + s->log_words, ids, sizeof(uint32_t) * count);
    s->log_words += count;
}

/* engine.hpp:188-218 step(), deterministic order */
static void sim_step(so_sim* s) {
    const int64_t t = s->t;
    const uint32_t qs = (uint32_t)(t % s->delay);
    /* spike_ring.hpp:47-55 begin_step */
    s->qcount[qs] = 0;
    if (s->bframes) memset(s->bits + (size_t)(t % s->bframes) * s->words, 0, 8 * s->words);
    s->expiring_count = 0;
    uint32_t* q = s->qentries + (size_t)qs * s->n;

    /* engine.hpp:308-341 stage_update (ascending ids) */
    for (uint32_t i = 0; i < s->n; ++i) {
        int spk;
        if (s->model == SO_PINGPONG) { /* benchmarks.hpp:27-31 */
            spk = s->flag[i] != 0;
            s->flag[i] = 0;
        } else if (s->model != SO_VOGELS && i >= s->n_recurrent) {
            /* benchmarks.hpp:101-104 -> lif.hpp:52-54 */
            spk = so_xs_uniform01(&s->rng[i]) <= (double)s->p_spike;
        } else {
            spk = lif_update(&s->V[i], &s->ACC[i], &s->REF[i], &s->lif, s->dt);
        }
        if (spk) {
            q[s->qcount[qs]++] = i;
            if (s->bframes) s->bits[(size_t)(t % s->bframes) * s->words + (i >> 6)] |= 1ull << (i & 63);
        }
        if (has_syn(s)) { /* engine.hpp:318-330 */
            int transmits = (s->delay == 1) ? spk : bit(s, t - (int64_t)s->delay + 1, i);
            if (!transmits && (int64_t)s->ages[i] + s->history <= t + s->delay + 1)
                s->expiring[s->expiring_count++] = i;
        }
    }
    s->counters[1] += s->qcount[qs];
    log_frame(s, q, s->qcount[qs]);

    const int64_t due = t - (int64_t)s->delay + 1;
    /* engine.hpp:343-367 stage_synapses */
    if (has_syn(s)) {
        s->counters[4] += s->expiring_count;
        if (due >= 0) {
            const uint32_t* f = s->qentries + (size_t)(due % s->delay) * s->n;
            uint32_t c = s->qcount[due % s->delay];
            for (uint32_t k = 0; k < c; ++k) catch_up(s, f[k], t);
        }
        for (uint32_t k = 0; k < s->expiring_count; ++k) catch_up(s, s->expiring[k], t);
    }
    /* engine.hpp:369-409 stage_receive */
    if (due >= 0) {
        s->counters[5]++;
        const uint32_t* f = s->qentries + (size_t)(due % s->delay) * s->n;
        uint32_t c = s->qcount[due % s->delay];
        for (uint32_t k = 0; k < c; ++k) {
            uint32_t src = f[k];
            const uint32_t* row = s->g->cells + (size_t)src * s->g->pitch;
            uint32_t deg = s->g->degree[src];
            s->counters[2] += deg;
            size_t base = (size_t)src * s->g->deg_max;
            for (uint32_t j = 0; j < deg; ++j) {
                uint32_t to = row[j];
                switch (s->model) {
                    case SO_PINGPONG: s->flag[to] = 1; break; /* benchmarks.hpp:32-35 */
                    case SO_BRUNEL_PLUS: /* benchmarks.hpp:132-135 */
                        s->ACC[to] += s->scale_c * s->W[base + j];
                        break;
                    default: /* lif.hpp:46-49 */
                        s->ACC[to] += s->scale_c * weight_of(s, src);
                }
            }
        }
    }
    s->t++;
    s->counters[0]++;
}

void so_sim_run(so_sim* s, int64_t steps) {
    for (int64_t i = 0; i < steps; ++i) sim_step(s);
}

/* engine.hpp:226-234 */
void so_sim_flush(so_sim* s) {
    if (!has_syn(s)) return;
    for (uint32_t i = 0; i < s->n; ++i) catch_up(s, i, s->t - 1);
}

const so_graph* so_sim_graph(const so_sim* s) { return s->g; }
int64_t so_sim_now(const so_sim* s) { return s->t; }
uint32_t so_sim_neurons(const so_sim* s) { return s->n; }
uint32_t so_sim_delay(const so_sim* s) { return s->delay; }
uint32_t so_sim_history(const so_sim* s) { return s->history; }
void so_sim_counters(const so_sim* s, uint64_t out[6]) { memcpy(out, s->counters, sizeof s->counters); }

void so_sim_field(const so_sim* s, int f, uint32_t* out) {
    if (s->model == SO_PINGPONG) {
        for (uint32_t i = 0; i < s->n; ++i) out[i] = s->flag[i];
        return;
    }
    const float* src = f == 0 ? s->V : (f == 1 ? s->ACC : s->REF);
    memcpy(out, src, sizeof(float) * s->n);
}

void so_sim_syn_field(const so_sim* s, int f, float* out) {
    if (!has_syn(s)) return;
    const float* src = f == 0 ? s->W : (f == 1 ? s->PT : s->QT);
    memcpy(out, src, sizeof(float) * (size_t)s->n * s->g->deg_max);
}

void so_sim_ages(const so_sim* s, uint32_t* out) {
    if (has_syn(s)) memcpy(out, s->ages, sizeof(uint32_t) * s->n);
}

uint64_t so_sim_frame_words(const so_sim* s) { return s->log_words; }
void so_sim_frames(const so_sim* s, uint32_t* out) {
    memcpy(out, s->log, sizeof(uint32_t) * s->log_words);
}

void so_sim_constants(const so_sim* s, double out[6]) {
    out[0] = s->scale_c;
    out[1] = s->p_spike;
    out[2] = s->w_exc;
    out[3] = s->w_inh;
    out[4] = s->stdp.decay_plus;
    out[5] = s->stdp.decay_minus;
}
