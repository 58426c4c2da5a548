/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle. Never linked into, loaded by or
 * called from the product path (paper_2308_14129_b200/); only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg use it, as the
 * checker.
 *
 * A plain-C restatement of the reference's algorithms on the SPEED hot path,
 * written from the reference's specification (each function cites the
 * reference file:line it follows, paths under /root/reference/proj). It is
 * pinned (tests/test_oracle.py) against the reference library itself compiled
 * into oracle/_ref/ and against the reference tests' golden vectors.
 *
 * Deliberately naive: dense per-partition membership arrays, linear scans,
 * sequential loops in the reference's order.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct { uint32_t src, dst; double ts; } o_edge; /* types.hpp:15-21 */

/* ---------------------------------------------------------- mt19937_64
 * The 64-bit Mersenne Twister as specified by C++11 [rand.eng.mers] (the
 * engine behind rng.hpp's draws). */
typedef struct { uint64_t mt[312]; int i; } o_mt;

static void mt_seed(o_mt* m, uint64_t s) {
    m->mt[0] = s;
    for (int i = 1; i < 312; ++i)
        m->mt[i] = 6364136223846793005ULL * (m->mt[i - 1] ^ (m->mt[i - 1] >> 62)) + (uint64_t)i;
    m->i = 312;
}

static uint64_t mt_next(o_mt* m) {
    if (m->i >= 312) {
        for (int k = 0; k < 312; ++k) {
            uint64_t y = (m->mt[k] & 0xFFFFFFFF80000000ULL) | (m->mt[(k + 1) % 312] & 0x7FFFFFFFULL);
            uint64_t v = m->mt[(k + 156) % 312] ^ (y >> 1);
            if (y & 1ULL) v ^= 0xB5026F5AA96619E9ULL;
            m->mt[k] = v;
        }
        m->i = 0;
    }
    uint64_t x = m->mt[m->i++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= x >> 43;
    return x;
}

/* rng.hpp:13-41 */
static double draw_unit(o_mt* m) { return (double)(mt_next(m) >> 11) * 0x1.0p-53; }
static uint64_t draw_below(o_mt* m, uint64_t n) { return mt_next(m) % n; }

uint64_t oracle_mt_first(uint64_t seed) { o_mt m; mt_seed(&m, seed); return mt_next(&m); }

/* ------------------------------------------------------ gen_powerlaw
 * graph_io.cpp:175-250. Returns 0 ok, 2 on invalid parameters. */
int oracle_gen_powerlaw(uint32_t nodes, uint64_t edges, double alpha, uint64_t seed, o_edge* out) {
    if (nodes < 2 || edges < 1 || !(alpha > 1.0)) return 2;
    uint64_t m_per = edges / nodes;
    if (m_per < 1) m_per = 1;
    double a = (alpha - 3.0) * (double)m_per;
    double a_min = -0.95 * (double)m_per;
    if (a < a_min) a = a_min;
    double ceil_ = a > 0.0 ? 1.0 + a / (double)m_per : 1.0;
    o_mt m;
    mt_seed(&m, seed);
    uint64_t* deg = calloc(nodes, sizeof(uint64_t));
    uint32_t* pool = malloc(sizeof(uint32_t) * 2 * edges);
    uint64_t np = 0, cnt = 0;
#define PUSH(u_, v_) do { out[cnt].src = (u_); out[cnt].dst = (v_); out[cnt].ts = (double)(cnt + 1); \
        ++cnt; ++deg[(u_)]; ++deg[(v_)]; pool[np++] = (u_); pool[np++] = (v_); } while (0)
#define DRAW_PREF(res) do { int ok_ = 0; for (int t_ = 0; t_ < 64; ++t_) { \
        uint32_t u_ = pool[draw_below(&m, np)]; \
        double r_ = (1.0 + a / (double)deg[u_]) / ceil_; \
        if (draw_unit(&m) < r_) { res = u_; ok_ = 1; break; } } \
        if (!ok_) res = pool[draw_below(&m, np)]; } while (0)
    for (uint64_t r = 0; r < m_per && cnt < edges; ++r) PUSH(0u, 1u);
    for (uint32_t v = 2; v < nodes && cnt < edges; ++v)
        for (uint64_t r = 0; r < m_per && cnt < edges; ++r) {
            uint32_t u;
            DRAW_PREF(u);
            for (int t = 0; u == v && t < 64; ++t) DRAW_PREF(u);
            if (u == v) u = (v + 1) % 2;
            PUSH(v, u);
        }
    while (cnt < edges) {
        uint32_t u, v;
        DRAW_PREF(u);
        DRAW_PREF(v);
        for (int t = 0; v == u && t < 64; ++t) DRAW_PREF(v);
        if (v == u) v = (u + 1) % nodes;
        PUSH(u, v);
    }
#undef PUSH
#undef DRAW_PREF
    for (uint64_t i = edges; i > 1; --i) { /* fisher_yates rng.hpp:36-41 */
        uint64_t j = draw_below(&m, i);
        o_edge t = out[i - 1]; out[i - 1] = out[j]; out[j] = t;
    }
    for (uint64_t t = 0; t < edges; ++t) out[t].ts = (double)(t + 1);
    free(deg);
    free(pool);
    return 0;
}

/* --------------------------------------------------------- centrality
 * centrality.cpp:27-52 */
int oracle_compute_centrality(const o_edge* e, uint64_t n, uint32_t node_count, double t_max,
                              double beta, int normalize, double* cent) {
    if (!(beta > 0.0 && beta < 1.0)) return 2;
    for (uint32_t i = 0; i < node_count; ++i) cent[i] = 0.0;
    if (n == 0) return 0;
    double t_min = e[0].ts, span = t_max - t_min;
    int sc = normalize && span > 0.0;
    double top = sc ? (t_max - t_min) / span : t_max;
    for (uint64_t k = 0; k < n; ++k) {
        double t = sc ? (e[k].ts - t_min) / span : e[k].ts;
        double w = exp(beta * (t - top));
        cent[e[k].src] += w;
        cent[e[k].dst] += w;
    }
    return 0;
}

/* centrality.cpp:66-88: selection by repeated max scan (O(k*N), fine for tests). */
int oracle_select_hubs(const double* cent, uint32_t node_count, double k, int base_all,
                       uint32_t* hubs, uint64_t* n_hubs) {
    if (!(k >= 0.0 && k <= 1.0)) return 2;
    uint64_t active = 0;
    for (uint32_t i = 0; i < node_count; ++i) active += cent[i] > 0.0;
    uint64_t base = base_all ? node_count : active;
    uint64_t want = (uint64_t)floor(k * (double)base);
    uint64_t take = want < active ? want : active;
    unsigned char* used = calloc(node_count ? node_count : 1, 1);
    for (uint64_t s = 0; s < take; ++s) {
        int64_t best = -1;
        for (uint32_t i = 0; i < node_count; ++i) {
            if (used[i] || !(cent[i] > 0.0)) continue;
            if (best < 0 || cent[i] > cent[best]) best = i; /* ties: first (smaller) id */
        }
        used[best] = 1;
    }
    uint64_t c = 0;
    for (uint32_t i = 0; i < node_count; ++i)
        if (used[i]) hubs[c++] = i;
    *n_hubs = c;
    free(used);
    return 0;
}

/* --------------------------------------------------------------- SEP
 * partitioner.cpp:11-148, Cases 1-5 with A-sets as dense membership rows
 * in[i*P + p] plus insertion-ordered lists. Outputs: edge_part[n],
 * node_parts as parts_flat[node_count*P] with counts[node_count] (shared
 * nodes hold 0..P-1), shared[] ascending. Returns 0 / 2 / 3. */
int oracle_partition_stream(const o_edge* e, uint64_t n, uint32_t node_count, int P, double lambda,
                            double eps, const double* cent, uint32_t cent_n, const unsigned char* is_hub,
                            int32_t* edge_part, int32_t* parts_flat, uint32_t* counts,
                            uint32_t* shared, uint64_t* n_shared, uint64_t* discards) {
    if (P < 1 || !(lambda > 0.0) || !(eps > 0.0)) return 2;
    for (uint64_t k = 1; k < n; ++k)
        if (e[k].ts < e[k - 1].ts) return 2;
    unsigned char* in = calloc((size_t)node_count * P + 1, 1);
    int32_t* order = malloc(sizeof(int32_t) * ((size_t)node_count * P + 1)); /* insertion order */
    uint32_t* na = calloc(node_count + 1, sizeof(uint32_t));
    uint64_t* sizes = calloc(P, sizeof(uint64_t));
    uint64_t mx = 0, mn = 0;
    *discards = 0;
#define CENT(x) ((x) < cent_n ? cent[(x)] : 0.0)
    for (uint64_t k = 0; k < n; ++k) {
        uint32_t i = e[k].src, j = e[k].dst;
        int ai = na[i] > 0, aj = na[j] > 0, hi = is_hub[i], hj = is_hub[j];
        int32_t target = -1, greedy = 0;
        if (!ai || !aj) {
            if (ai && !hi) target = order[(size_t)i * P];
            else if (aj && !hj) target = order[(size_t)j * P];
            else greedy = 1;
        } else if (hi != hj) {
            target = hi ? order[(size_t)j * P] : order[(size_t)i * P];
        } else if (hi) {
            greedy = 1;
        } else {
            if (order[(size_t)i * P] != order[(size_t)j * P]) { edge_part[k] = -1; ++*discards; continue; }
            target = order[(size_t)i * P];
        }
        if (greedy) { /* argmax of score (partitioner.cpp:27-68), strict > */
            double ci = CENT(i), cj = CENT(j), sum = ci + cj;
            double ti = sum > 0.0 ? ci / sum : 0.5, tj = sum > 0.0 ? cj / sum : 0.5;
            double best = 0.0;
            for (int p = 0; p < P; ++p) {
                double h = 0.0;
                if (in[(size_t)i * P + p]) h += 1.0 + (1.0 - ti);
                if (in[(size_t)j * P + p]) h += 1.0 + (1.0 - tj);
                double s = h + lambda * (double)(mx - sizes[p]) / (eps + (double)(mx - mn));
                if (p == 0 || s > best) { best = s; target = p; }
            }
        }
        edge_part[k] = target;
        uint32_t ends[2] = {i, j};
        for (int q = 0; q < 2; ++q) {
            uint32_t x = ends[q];
            if (!in[(size_t)x * P + target]) { in[(size_t)x * P + target] = 1; order[(size_t)x * P + na[x]++] = target; }
        }
        if ((!hi && na[i] > 1) || (!hj && na[j] > 1)) {
            free(in); free(order); free(na); free(sizes);
            return 3; /* ResidencyViolation */
        }
        ++sizes[target];
        mx = sizes[0]; mn = sizes[0];
        for (int p = 1; p < P; ++p) { if (sizes[p] > mx) mx = sizes[p]; if (sizes[p] < mn) mn = sizes[p]; }
    }
#undef CENT
    uint64_t ns = 0;
    for (uint32_t i = 0; i < node_count; ++i) {
        if (na[i] > 1) {
            shared[ns++] = i;
            counts[i] = (uint32_t)P;
            for (int p = 0; p < P; ++p) parts_flat[(size_t)i * P + p] = p;
        } else {
            counts[i] = na[i];
            if (na[i]) parts_flat[(size_t)i * P] = order[(size_t)i * P];
        }
    }
    *n_shared = ns;
    free(in); free(order); free(na); free(sizes);
    return 0;
}

/* --------------------------------------------------- induce_subgraphs
 * pac_sim.cpp:106-132. member[p*N + i]; writes, for partition p, the stream
 * positions of its edges into idx (capacity n) and returns their count. */
uint64_t oracle_induce_one(const o_edge* e, uint64_t n, const unsigned char* member, uint64_t* idx) {
    uint64_t c = 0;
    for (uint64_t k = 0; k < n; ++k)
        if (member[e[k].src] && member[e[k].dst]) idx[c++] = k;
    return c;
}

/* ------------------------------------------------- surrogate MSG / UPD
 * pac_sim.cpp:28-104. state row-major [N*d], w_m [d*3d], omega [d]. */
void oracle_model_seeded(int d, uint64_t seed, double* w_m, double* omega) {
    o_mt m;
    mt_seed(&m, seed);
    size_t cols = 3 * (size_t)d;
    double scale = 1.0 / sqrt((double)cols);
    for (size_t k = 0; k < (size_t)d * cols; ++k) { /* draw_normal rng.hpp:28-34 */
        double u1 = draw_unit(&m), u2 = draw_unit(&m);
        while (u1 <= 0.0) u1 = draw_unit(&m);
        w_m[k] = sqrt(-2.0 * log(u1)) * cos(2.0 * M_PI * u2) * scale;
    }
    double f = 0.5 + (1.5 - 0.5) * draw_unit(&m);
    double steps = d > 1 ? (double)(d - 1) : 1.0;
    for (int r = 0; r < d; ++r) omega[r] = f * pow(10.0, -3.0 * (double)r / steps);
}

static void o_message(int d, const double* w, const double* om, const double* sx, const double* sy,
                      double dt, double* out) {
    for (int r = 0; r < d; ++r) {
        const double* wr = w + (size_t)r * 3 * d;
        double acc = 0.0;
        for (int c = 0; c < d; ++c) acc += wr[c] * sx[c];
        for (int c = 0; c < d; ++c) acc += wr[d + c] * sy[c];
        for (int c = 0; c < d; ++c) acc += wr[2 * d + c] * cos(om[c] * dt);
        out[r] = tanh(acc);
    }
}

/* Returns 0 ok, 2 NonChronological (state untouched for that edge). */
int oracle_model_update(double* state, double* last_ts, int d, const o_edge* ed, const double* w,
                        const double* om, double g) {
    uint32_t i = ed->src, j = ed->dst;
    if (ed->ts < last_ts[i] || ed->ts < last_ts[j]) return 2;
    double* si = state + (size_t)i * d;
    double* sj = state + (size_t)j * d;
    double* buf = malloc(sizeof(double) * 4 * d);
    double *a = buf, *b = buf + d, *mi = buf + 2 * d, *mj = buf + 3 * d;
    memcpy(a, si, sizeof(double) * d);
    memcpy(b, sj, sizeof(double) * d);
    if (i == j) {
        o_message(d, w, om, a, a, ed->ts - last_ts[i], mi);
        for (int r = 0; r < d; ++r) si[r] = (1.0 - g) * a[r] + g * mi[r];
        last_ts[i] = ed->ts;
    } else {
        o_message(d, w, om, a, b, ed->ts - last_ts[i], mi);
        o_message(d, w, om, b, a, ed->ts - last_ts[j], mj);
        for (int r = 0; r < d; ++r) {
            si[r] = (1.0 - g) * a[r] + g * mi[r];
            sj[r] = (1.0 - g) * b[r] + g * mj[r];
        }
        last_ts[i] = ed->ts;
        last_ts[j] = ed->ts;
    }
    free(buf);
    return 0;
}

/* pac_sim.cpp:162-203; states are W separate [N*d] blocks laid out back to back. */
void oracle_sync_shared(int W, uint32_t N, int d, double* states, double* clocks,
                        const uint32_t* shared, uint64_t n_shared, int average) {
    if (W < 2 || n_shared == 0) return;
    size_t S = (size_t)N * d;
    for (uint64_t s = 0; s < n_shared; ++s) {
        uint32_t n = shared[s];
        if (!average) {
            int best = 0;
            for (int w = 1; w < W; ++w)
                if (clocks[(size_t)w * N + n] > clocks[(size_t)best * N + n]) best = w;
            for (int w = 0; w < W; ++w) {
                if (w == best) continue;
                memcpy(states + w * S + (size_t)n * d, states + best * S + (size_t)n * d, sizeof(double) * d);
                clocks[(size_t)w * N + n] = clocks[(size_t)best * N + n];
            }
        } else {
            int agree = 1;
            for (int w = 1; w < W && agree; ++w) {
                agree = clocks[(size_t)w * N + n] == clocks[n];
                for (int c = 0; c < d && agree; ++c)
                    agree = states[w * S + (size_t)n * d + c] == states[(size_t)n * d + c];
            }
            if (agree) continue;
            double ts = 0.0;
            for (int w = 0; w < W; ++w)
                if (clocks[(size_t)w * N + n] > ts) ts = clocks[(size_t)w * N + n];
            for (int c = 0; c < d; ++c) {
                double m = 0.0;
                for (int w = 0; w < W; ++w) m += states[w * S + (size_t)n * d + c];
                m /= (double)W;
                for (int w = 0; w < W; ++w) states[w * S + (size_t)n * d + c] = m;
            }
            for (int w = 0; w < W; ++w) clocks[(size_t)w * N + n] = ts;
        }
    }
}

/* Alg. 2 lockstep epoch (pac_sim.cpp:205-264) over W workers whose edges are
 * CSR e_off[W+1]. loops_out[W], batches_out[W]. Returns 0 / 2. */
int oracle_run_epoch(int W, uint32_t N, int d, const uint64_t* e_off, const o_edge* edges,
                     double* states, double* clocks, const double* w, const double* om, double g,
                     const uint32_t* shared, uint64_t n_shared, int average, uint64_t B,
                     uint64_t* batches_out, uint64_t* loops_out) {
    size_t S = (size_t)N * d;
    double* snap = malloc(sizeof(double) * (S + N) * (W ? W : 1));
    uint64_t* pos = calloc(W ? W : 1, sizeof(uint64_t));
    unsigned char* done = calloc(W ? W : 1, 1);
    int rc = 0;
    for (int k = 0; k < W; ++k) {
        uint64_t ne = e_off[k + 1] - e_off[k];
        batches_out[k] = (ne + B - 1) / B;
        loops_out[k] = 0;
        if (batches_out[k] == 0) {
            loops_out[k] = 1;
            done[k] = 1;
            memcpy(snap + k * (S + N), states + k * S, sizeof(double) * S);
            memcpy(snap + k * (S + N) + S, clocks + (size_t)k * N, sizeof(double) * N);
        }
    }
    for (;;) {
        int all = 1;
        for (int k = 0; k < W; ++k) all &= done[k];
        if (all) break;
        for (int k = 0; k < W; ++k) {
            if (batches_out[k] == 0) continue;
            if (pos[k] == 0) {
                memset(states + k * S, 0, sizeof(double) * S);
                memset(clocks + (size_t)k * N, 0, sizeof(double) * N);
            }
            uint64_t ne = e_off[k + 1] - e_off[k];
            uint64_t lo = pos[k] * B, hi = (pos[k] + 1) * B < ne ? (pos[k] + 1) * B : ne;
            for (uint64_t q = lo; q < hi; ++q)
                if (oracle_model_update(states + k * S, clocks + (size_t)k * N, d, edges + e_off[k] + q, w, om, g)) {
                    rc = 2;
                    goto out;
                }
            if (++pos[k] == batches_out[k]) {
                ++loops_out[k];
                done[k] = 1;
                pos[k] = 0;
                memcpy(snap + k * (S + N), states + k * S, sizeof(double) * S);
                memcpy(snap + k * (S + N) + S, clocks + (size_t)k * N, sizeof(double) * N);
            }
        }
    }
    for (int k = 0; k < W; ++k) {
        memcpy(states + k * S, snap + k * (S + N), sizeof(double) * S);
        memcpy(clocks + (size_t)k * N, snap + k * (S + N) + S, sizeof(double) * N);
    }
    oracle_sync_shared(W, N, d, states, clocks, shared, n_shared, average);
out:
    free(snap);
    free(pos);
    free(done);
    return rc;
}

/* digest.hpp:12-37 / pac_sim.cpp:18-26 */
uint64_t oracle_digest(const double* state, const double* clocks, uint32_t N, int d) {
    uint64_t h = 14695981039346656037ULL;
    for (uint32_t i = 0; i < N; ++i)
        for (int r = 0; r <= d; ++r) {
            double v = r < d ? state[(size_t)i * d + r] : clocks[i];
            uint64_t b;
            memcpy(&b, &v, 8);
            for (int k = 0; k < 8; ++k) { h ^= (uint8_t)(b >> (8 * k)); h *= 1099511628211ULL; }
        }
    return h;
}
