/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * Plain-C restatement of the reference algorithm on the INSPIRIT hot path.
 * Every function cites the reference lines it restates; paths are relative to
 * /root/reference/proj.  Compiled with -ffp-contract=off and without
 * -ffast-math so FP64 sums round exactly like the reference build (x86-64
 * SSE2, no FMA).  See oracle.h for who may call it.
 */
#include "oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- errors */

static _Thread_local char g_err[1024];
const char* orc_last_error(void) { return g_err; }

static int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}

#define XALLOC(T, n) ((T*)calloc((size_t)((n) > 0 ? (n) : 1), sizeof(T)))

/* ------------------------------------------------------------ graph view */

typedef struct {
    int64_t g, n, nh;
    const int32_t *doff, *dep, *ioff, *in, *ooff, *out, *type;
    const int64_t *hbytes, *tid;
    const tbsim_batch_desc* b;
    /* index (build_index, src/taskgraph.cpp:11-43): succ/pred sorted
     * ascending, multi-edges kept */
    int32_t *soff, *succ, *poff, *pred;
} view_t;

static const char* type_name(const view_t* v, int32_t ty, char* buf) {
    if (v->b->type_names && ty >= 0 && ty < v->b->n_type_names) return v->b->type_names[ty];
    sprintf(buf, "type%d", ty);
    return buf;
}

static int64_t task_ident(const view_t* v, int64_t pos) { return v->tid ? v->tid[pos] : pos; }

static int cmp_i32(const void* a, const void* b) {
    int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
    return (x > y) - (x < y);
}

static void view_open(view_t* v, const tbsim_batch_desc* b, int64_t g) {
    memset(v, 0, sizeof *v);
    v->b = b;
    v->g = g;
    int64_t t0 = b->task_base[g];
    v->n = b->task_base[g + 1] - t0;
    v->nh = b->handle_base[g + 1] - b->handle_base[g];
    v->doff = b->dep_off + t0 + g;
    v->dep = b->dep + b->edge_base[g];
    v->ioff = b->in_off + t0 + g;
    v->in = b->in + b->in_base[g];
    v->ooff = b->out_off + t0 + g;
    v->out = b->out + b->out_base[g];
    v->type = b->type + t0;
    v->hbytes = b->handle_bytes + b->handle_base[g];
    v->tid = b->task_id ? b->task_id + t0 : NULL;
    /* succ: iterate dependents in position order, so lists come out sorted
     * (taskgraph.cpp:21-34,35-38); pred: copy then sort each list. */
    int64_t n = v->n, E = v->doff[n];
    v->soff = XALLOC(int32_t, n + 1);
    v->succ = XALLOC(int32_t, E);
    v->poff = XALLOC(int32_t, n + 1);
    v->pred = XALLOC(int32_t, E);
    for (int64_t i = 0; i < n; ++i)
        for (int32_t k = v->doff[i]; k < v->doff[i + 1]; ++k) v->soff[v->dep[k] + 1]++;
    for (int64_t i = 0; i < n; ++i) v->soff[i + 1] += v->soff[i];
    int32_t* cur = XALLOC(int32_t, n);
    for (int64_t i = 0; i < n; ++i) cur[i] = v->soff[i];
    for (int64_t i = 0; i < n; ++i)
        for (int32_t k = v->doff[i]; k < v->doff[i + 1]; ++k) v->succ[cur[v->dep[k]]++] = (int32_t)i;
    free(cur);
    for (int64_t i = 0; i <= n; ++i) v->poff[i] = v->doff[i];
    memcpy(v->pred, v->dep, sizeof(int32_t) * (size_t)E);
    for (int64_t i = 0; i < n; ++i)
        qsort(v->pred + v->poff[i], (size_t)(v->poff[i + 1] - v->poff[i]), sizeof(int32_t), cmp_i32);
}

static void view_close(view_t* v) {
    free(v->soff); free(v->succ); free(v->poff); free(v->pred);
}

/* ---------------------------------------------------- orders and levels */

/* topological_layers: FIFO Kahn, layer = longest path from an entry
 * (src/taskgraph.cpp:197-219). */
static int layers_of(const view_t* v, int32_t* layer) {
    int64_t n = v->n, done = 0, head = 0, tail = 0;
    int32_t* unmet = XALLOC(int32_t, n);
    int32_t* q = XALLOC(int32_t, n);
    for (int64_t i = 0; i < n; ++i) {
        layer[i] = 0;
        unmet[i] = v->poff[i + 1] - v->poff[i];
        if (unmet[i] == 0) q[tail++] = (int32_t)i;
    }
    while (head < tail) {
        int32_t u = q[head++];
        done++;
        for (int32_t k = v->soff[u]; k < v->soff[u + 1]; ++k) {
            int32_t s = v->succ[k];
            if (layer[s] < layer[u] + 1) layer[s] = layer[u] + 1;
            if (--unmet[s] == 0) q[tail++] = s;
        }
    }
    free(unmet); free(q);
    if (done != n) return fail(TBSIM_E_RUNTIME, "graph has a dependency cycle");
    return 0;
}

/* topological_order: Kahn with a min-heap of positions
 * (src/taskgraph.cpp:221-241). */
static void heap_push(int32_t* h, int64_t* sz, int32_t x) {
    int64_t i = (*sz)++;
    h[i] = x;
    while (i > 0) {
        int64_t p = (i - 1) / 2;
        if (h[p] <= h[i]) break;
        int32_t t = h[p]; h[p] = h[i]; h[i] = t;
        i = p;
    }
}
static int32_t heap_pop(int32_t* h, int64_t* sz) {
    int32_t top = h[0];
    h[0] = h[--(*sz)];
    int64_t i = 0;
    for (;;) {
        int64_t l = 2 * i + 1, r = l + 1, m = i;
        if (l < *sz && h[l] < h[m]) m = l;
        if (r < *sz && h[r] < h[m]) m = r;
        if (m == i) break;
        int32_t t = h[m]; h[m] = h[i]; h[i] = t;
        i = m;
    }
    return top;
}
static int topo_order(const view_t* v, int32_t* order) {
    int64_t n = v->n, sz = 0, cnt = 0;
    int32_t* unmet = XALLOC(int32_t, n);
    int32_t* h = XALLOC(int32_t, n);
    for (int64_t i = 0; i < n; ++i) {
        unmet[i] = v->poff[i + 1] - v->poff[i];
        if (unmet[i] == 0) heap_push(h, &sz, (int32_t)i);
    }
    while (sz > 0) {
        int32_t u = heap_pop(h, &sz);
        order[cnt++] = u;
        for (int32_t k = v->soff[u]; k < v->soff[u + 1]; ++k)
            if (--unmet[v->succ[k]] == 0) heap_push(h, &sz, v->succ[k]);
    }
    free(unmet); free(h);
    if (cnt != n) return fail(TBSIM_E_RUNTIME, "graph has a dependency cycle");
    return 0;
}

/* ------------------------------------------------------------- ability */

/* height_groups (src/attributes.cpp:33-55) + ability_impl (:57-92): sets of
 * descendants OR-ed over successors, processed by increasing height. */
static void ability_of(const view_t* v, int64_t* ability) {
    int64_t n = v->n;
    if (n == 0) return;
    int64_t nw = (n + 63) / 64;
    int32_t* height = XALLOC(int32_t, n);
    int32_t* unproc = XALLOC(int32_t, n);
    int32_t* stack = XALLOC(int32_t, n);
    int64_t sp = 0, max_h = 0;
    for (int64_t i = 0; i < n; ++i) {
        unproc[i] = v->soff[i + 1] - v->soff[i];
        if (unproc[i] == 0) stack[sp++] = (int32_t)i;
    }
    while (sp > 0) {
        int32_t u = stack[--sp];
        if (height[u] > max_h) max_h = height[u];
        for (int32_t k = v->poff[u]; k < v->poff[u + 1]; ++k) {
            int32_t p = v->pred[k];
            if (height[p] < height[u] + 1) height[p] = height[u] + 1;
            if (--unproc[p] == 0) stack[sp++] = p;
        }
    }
    uint64_t** desc = XALLOC(uint64_t*, n);
    int32_t* remaining = XALLOC(int32_t, n);
    for (int64_t i = 0; i < n; ++i) remaining[i] = v->poff[i + 1] - v->poff[i];
    for (int64_t h = 0; h <= max_h; ++h) {
        for (int64_t u = 0; u < n; ++u) {
            if (height[u] != h) continue;
            uint64_t* set = XALLOC(uint64_t, nw);
            for (int32_t k = v->soff[u]; k < v->soff[u + 1]; ++k) {
                int32_t s = v->succ[k];
                set[s >> 6] |= 1ull << (s & 63);
                if (desc[s])
                    for (int64_t w = 0; w < nw; ++w) set[w] |= desc[s][w];
            }
            int64_t c = 0;
            for (int64_t w = 0; w < nw; ++w) c += __builtin_popcountll(set[w]);
            ability[u] = c;
            desc[u] = set;
        }
        for (int64_t u = 0; u < n; ++u) {
            if (height[u] != h) continue;
            for (int32_t k = v->soff[u]; k < v->soff[u + 1]; ++k) {
                int32_t s = v->succ[k];
                if (--remaining[s] == 0) { free(desc[s]); desc[s] = NULL; }
            }
        }
    }
    for (int64_t i = 0; i < n; ++i) free(desc[i]);
    free(desc); free(remaining); free(height); free(unproc); free(stack);
}

/* ----------------------------------------------------------- efficiency */

/* gpu_times_or_throw (src/attributes.cpp:94-99) over CostTable::gpu_ms
 * (src/platform.cpp:27-37). */
static int gpu_times(const view_t* v, const tbsim_costs* c, double* gpu) {
    char buf[32];
    for (int64_t i = 0; i < v->n; ++i) {
        int32_t ty = v->type[i];
        double ms = (ty < c->n_types && c->gpu_ms) ? c->gpu_ms[ty] : 0.0;
        if (!(ms > 0.0))
            return fail(TBSIM_E_RUNTIME, "no gpu cost entry for task type %s", type_name(v, ty, buf));
        gpu[i] = ms;
    }
    return 0;
}

/* efficiency_of (src/attributes.cpp:110-137): forward max-plus relaxation
 * from src in topological order; counts v != src with dist <= w.  Returns
 * counts for several windows at once (dist does not depend on w). */
static void efficiency_multi(const view_t* v, const int32_t* topo, const int32_t* topo_pos,
                             const double* gpu, const double* ws, int nw, int64_t* counts /*[n*nw]*/) {
    int64_t n = v->n;
    double* dist = XALLOC(double, n);
    uint32_t* stamp = XALLOC(uint32_t, n);
    uint32_t cur = 0;
    for (int64_t src = 0; src < n; ++src) {
        cur += 1;
        dist[src] = 0.0;
        stamp[src] = cur;
        int64_t live = 1;
        for (int k = 0; k < nw; ++k) counts[src * nw + k] = 0;
        for (int64_t p = topo_pos[src]; p < n && live > 0; ++p) {
            int32_t u = topo[p];
            if (stamp[u] != cur) continue;
            live -= 1;
            if (u != src)
                for (int k = 0; k < nw; ++k)
                    if (dist[u] <= ws[k]) counts[src * nw + k] += 1;
            for (int32_t e = v->soff[u]; e < v->soff[u + 1]; ++e) {
                int32_t s = v->succ[e];
                double cand = dist[u] + gpu[s];
                if (stamp[s] != cur) {
                    stamp[s] = cur;
                    dist[s] = cand;
                    live += 1;
                } else if (cand > dist[s]) {
                    dist[s] = cand;
                }
            }
        }
    }
    free(dist); free(stamp);
}

static int64_t gcd64(int64_t a, int64_t b) {
    if (a < 0) a = -a;
    if (b < 0) b = -b;
    while (b) { int64_t t = a % b; a = b; b = t; }
    return a;
}

static int cmp_f64(const void* a, const void* b) {
    double x = *(const double*)a, y = *(const double*)b;
    return (x > y) - (x < y);
}

/* median_gpu_time_ms: lower median (src/platform.cpp:233-240). */
static int median_gpu(const view_t* v, const tbsim_costs* c, double* med) {
    if (v->n == 0) return fail(TBSIM_E_RUNTIME, "empty graph has no median time");
    double* t = XALLOC(double, v->n);
    int rc = gpu_times(v, c, t);
    if (!rc) {
        qsort(t, (size_t)v->n, sizeof(double), cmp_f64);
        *med = t[(v->n - 1) / 2];
    }
    free(t);
    return rc;
}

/* mean_ms (src/platform.cpp:39-50): ((0 + cpu) + gpu) / count. */
static int mean_ms(const view_t* v, const tbsim_costs* c, int32_t ty, double* out) {
    double sum = 0.0;
    int n = 0;
    if (ty < c->n_types && c->cpu_ms && c->cpu_ms[ty] > 0.0) { sum += c->cpu_ms[ty]; n++; }
    if (ty < c->n_types && c->gpu_ms && c->gpu_ms[ty] > 0.0) { sum += c->gpu_ms[ty]; n++; }
    if (n == 0) {
        char buf[32];
        return fail(TBSIM_E_RUNTIME, "no cost entry for task type %s", type_name(v, ty, buf));
    }
    *out = sum / n;
    return 0;
}

typedef struct { int64_t s, c; } frac_t;

/* Score of one efficiency vector: distinct reduced per-class means
 * (src/attributes.cpp:205-217). */
static int64_t class_score(const int64_t* eff, int64_t stride, const int32_t* cls, int64_t n,
                           int64_t n_cls) {
    int64_t* sum = XALLOC(int64_t, n_cls);
    int64_t* cnt = XALLOC(int64_t, n_cls);
    for (int64_t i = 0; i < n; ++i) { sum[cls[i]] += eff[i * stride]; cnt[cls[i]] += 1; }
    frac_t* f = XALLOC(frac_t, n_cls);
    int64_t distinct = 0;
    for (int64_t c = 0; c < n_cls; ++c) {
        int64_t d = gcd64(sum[c] == 0 ? cnt[c] : sum[c], cnt[c]);
        frac_t x = {sum[c] / d, cnt[c] / d};
        int seen = 0;
        for (int64_t j = 0; j < distinct; ++j)
            if (f[j].s == x.s && f[j].c == x.c) { seen = 1; break; }
        if (!seen) f[distinct++] = x;
    }
    free(sum); free(cnt); free(f);
    return distinct;
}

int orc_attributes(const tbsim_batch_desc* b, const tbsim_costs* costs, int request,
                   int priority_kind, tbsim_attr_out* o) {
    for (int64_t g = 0; g < b->n_graphs; ++g) {
        view_t v;
        view_open(&v, b, g);
        int64_t n = v.n, t0 = b->task_base[g];
        int rc = 0;
        int want_all = (request & TBSIM_ATTR_ALL) != 0;
        int32_t* layer = XALLOC(int32_t, n);
        int32_t* topo = XALLOC(int32_t, n);
        int32_t* topo_pos = XALLOC(int32_t, n);
        double* gpu = XALLOC(double, n);
        int64_t* tmp = XALLOC(int64_t, n);
        int64_t* counts = XALLOC(int64_t, n * 11);
        double unit = o->unit_time_ms ? o->unit_time_ms[g] : 0.0;

        if ((request & TBSIM_ATTR_ABILITY) || want_all) {
            ability_of(&v, tmp);
            if (o->ability) memcpy(o->ability + t0, tmp, sizeof(int64_t) * (size_t)n);
        }
        if (!rc && ((request & TBSIM_ATTR_CALIBRATE) || want_all)) {
            /* calibrate_unit_time (src/attributes.cpp:189-232) */
            double med = 0.0, w0, ws[11];
            rc = layers_of(&v, layer);
            if (!rc) rc = median_gpu(&v, costs, &med);
            if (!rc) rc = gpu_times(&v, costs, gpu);
            if (!rc) rc = topo_order(&v, topo);
            if (!rc) {
                for (int64_t p = 0; p < n; ++p) topo_pos[topo[p]] = (int32_t)p;
                /* class ids: distinct (layer, type) pairs in first-seen order */
                int32_t* cls = XALLOC(int32_t, n);
                int64_t n_cls = 0;
                int32_t* cl_layer = XALLOC(int32_t, n);
                int32_t* cl_type = XALLOC(int32_t, n);
                for (int64_t i = 0; i < n; ++i) {
                    int64_t c = 0;
                    for (; c < n_cls; ++c)
                        if (cl_layer[c] == layer[i] && cl_type[c] == v.type[i]) break;
                    if (c == n_cls) { cl_layer[c] = layer[i]; cl_type[c] = v.type[i]; n_cls++; }
                    cls[i] = (int32_t)c;
                }
                w0 = 2.0 * med;
                for (int k = -4; k <= 6; ++k) ws[k + 4] = ldexp(w0, k);
                efficiency_multi(&v, topo, topo_pos, gpu, ws, 11, counts);
                int64_t best = -1, w0s = 0;
                double best_w = 0.0;
                for (int k = 0; k < 11; ++k) {
                    int64_t s = class_score(counts + k, 11, cls, n, n_cls);
                    if (k == 4) w0s = s;
                    if (s > best) { best = s; best_w = ws[k]; }
                }
                unit = best_w;
                if (o->unit_time_ms) o->unit_time_ms[g] = best_w;
                if (o->w0_ms) o->w0_ms[g] = w0;
                if (o->best_score) o->best_score[g] = best;
                if (o->w0_score) o->w0_score[g] = w0s;
                if (o->evaluations) o->evaluations[g] = 11;
                free(cls); free(cl_layer); free(cl_type);
            }
        }
        if (!rc && ((request & TBSIM_ATTR_EFFICIENCY) || want_all)) {
            /* efficiency_impl (src/attributes.cpp:139-165) */
            if (!(unit >= 0.0)) rc = fail(TBSIM_E_INVALID_ARGUMENT, "unit time must be non-negative");
            if (!rc && n > 0) {
                rc = gpu_times(&v, costs, gpu);
                if (!rc) rc = topo_order(&v, topo);
                if (!rc) {
                    for (int64_t p = 0; p < n; ++p) topo_pos[topo[p]] = (int32_t)p;
                    efficiency_multi(&v, topo, topo_pos, gpu, &unit, 1, tmp);
                    if (o->efficiency) memcpy(o->efficiency + t0, tmp, sizeof(int64_t) * (size_t)n);
                }
            }
        }
        int want_rank = (request & TBSIM_ATTR_RANK) || (want_all && priority_kind == TBSIM_PRIO_UPWARD_RANK);
        int want_depth = (request & TBSIM_ATTR_DEPTH) || (want_all && priority_kind == TBSIM_PRIO_DEPTH);
        if (!rc && want_rank) {
            /* upward_rank_priority (src/attributes.cpp:234-253) */
            double* mean = XALLOC(double, n);
            double* rank = XALLOC(double, n);
            for (int64_t i = 0; i < n && !rc; ++i) rc = mean_ms(&v, costs, v.type[i], &mean[i]);
            if (!rc) rc = topo_order(&v, topo);
            if (!rc) {
                for (int64_t p = n - 1; p >= 0; --p) {
                    int32_t u = topo[p];
                    double best = 0.0;
                    for (int32_t k = v.soff[u]; k < v.soff[u + 1]; ++k)
                        if (rank[v.succ[k]] > best) best = rank[v.succ[k]];
                    rank[u] = mean[u] + best;
                }
                if (o->static_priority)
                    for (int64_t i = 0; i < n; ++i) o->static_priority[t0 + i] = (int64_t)(rank[i] * 1000.0);
            }
            free(mean); free(rank);
        }
        if (!rc && want_depth) {
            /* depth_priority (src/attributes.cpp:255-265) */
            rc = topo_order(&v, topo);
            if (!rc) {
                for (int64_t i = 0; i < n; ++i) tmp[i] = 0;
                for (int64_t p = n - 1; p >= 0; --p) {
                    int32_t u = topo[p];
                    for (int32_t k = v.soff[u]; k < v.soff[u + 1]; ++k)
                        if (tmp[v.succ[k]] + 1 > tmp[u]) tmp[u] = tmp[v.succ[k]] + 1;
                }
                int64_t* dst = (request & TBSIM_ATTR_DEPTH) ? o->depth : NULL;
                if (dst) memcpy(dst + t0, tmp, sizeof(int64_t) * (size_t)n);
                if (want_all && priority_kind == TBSIM_PRIO_DEPTH && o->static_priority)
                    memcpy(o->static_priority + t0, tmp, sizeof(int64_t) * (size_t)n);
            }
        }
        if (!rc && want_all && priority_kind == TBSIM_PRIO_ZERO && o->static_priority)
            memset(o->static_priority + t0, 0, sizeof(int64_t) * (size_t)n);
        if (!rc && (request & TBSIM_ATTR_LAYERS)) {
            rc = layers_of(&v, layer);
            if (!rc && o->layer) memcpy(o->layer + t0, layer, sizeof(int32_t) * (size_t)n);
        }
        free(layer); free(topo); free(topo_pos); free(gpu); free(tmp); free(counts);
        view_close(&v);
        if (rc) return rc;
    }
    return 0;
}

/* ------------------------------------------------------------ regulator */

/* calculate_k (src/policies.cpp:153-169) */
double orc_calculate_k(const double* t, const int64_t* y, int n) {
    if (n < 2) return 0.0;
    double sx = 0.0, sy = 0.0;
    for (int i = 0; i < n; ++i) { sx += t[i]; sy += (double)y[i]; }
    const double dn = (double)n;
    const double mx = sx / dn, my = sy / dn;
    double sxx = 0.0, sxy = 0.0;
    for (int i = 0; i < n; ++i) {
        sxx += (t[i] - mx) * (t[i] - mx);
        sxy += (t[i] - mx) * ((double)y[i] - my);
    }
    if (sxx == 0.0) return 0.0;
    return sxy / sxx;
}

/* regulator_step (src/policies.cpp:171-203) */
void orc_regulator_step(tbsim_regulator_state* st, const tbsim_regulator_cfg* cfg,
                        int64_t cur, double now) {
    if (st->n_samples < TBSIM_MAX_SLOPE_SAMPLES) {
        st->sample_time[st->n_samples] = now;
        st->sample_nready[st->n_samples] = cur;
        st->n_samples++;
    } else { /* ring full: only reachable when slope_samples >= capacity */
        memmove(st->sample_time, st->sample_time + 1, sizeof(double) * (TBSIM_MAX_SLOPE_SAMPLES - 1));
        memmove(st->sample_nready, st->sample_nready + 1, sizeof(int64_t) * (TBSIM_MAX_SLOPE_SAMPLES - 1));
        st->sample_time[TBSIM_MAX_SLOPE_SAMPLES - 1] = now;
        st->sample_nready[TBSIM_MAX_SLOPE_SAMPLES - 1] = cur;
    }
    while (st->n_samples > cfg->slope_samples) {
        memmove(st->sample_time, st->sample_time + 1, sizeof(double) * (size_t)(st->n_samples - 1));
        memmove(st->sample_nready, st->sample_nready + 1, sizeof(int64_t) * (size_t)(st->n_samples - 1));
        st->n_samples--;
    }
    int64_t d = cur - st->last_trigger_nready;
    if ((d < 0 ? -d : d) < cfg->task_window) return;
    st->last_trigger_nready = cur;
    if (cur > st->peak) st->peak = cur;
    st->phase = cur >= st->peak - cfg->dec_step ? TBSIM_PHASE_INC : TBSIM_PHASE_DEC;
    if (st->phase == TBSIM_PHASE_INC) {
        if (cur - st->prev_nready >= cfg->s_inc) {
            st->cur_k = orc_calculate_k(st->sample_time, st->sample_nready, st->n_samples);
            if (st->cur_k < cfg->k_inc) st->mode = TBSIM_MODE_EFFICIENCY;
            else if (st->cur_k > cfg->k_inc) st->mode = TBSIM_MODE_ABILITY;
        }
    } else {
        if (cur > st->peak - cfg->s_dec * st->s_dec_count) {
            st->mode = TBSIM_MODE_ABILITY;
        } else if (cur <= st->peak - cfg->s_dec * (st->s_dec_count + 1) + cfg->c) {
            st->mode = TBSIM_MODE_LOCALITY;
            if (cur <= st->peak - cfg->s_dec * (st->s_dec_count + 1)) st->s_dec_count += 1;
        }
    }
    st->prev_nready = cur;
}

int orc_default_regulator_config(const tbsim_batch_desc* b, int64_t g,
                                 const tbsim_platform_desc* p, tbsim_regulator_cfg* cfg) {
    /* default_regulator_config (src/policies.cpp:139-151) */
    view_t v;
    view_open(&v, b, g);
    double med = 0.0;
    int rc = median_gpu(&v, &p->costs, &med);
    view_close(&v);
    if (rc) return rc;
    int64_t n = p->n_workers;
    memset(cfg, 0, sizeof *cfg);
    cfg->task_window = (n + 3) / 4 > 2 ? (n + 3) / 4 : 2;
    cfg->s_inc = n;
    cfg->k_inc = (double)n / med;
    cfg->s_dec = (n + 3) / 4 > 2 ? (n + 3) / 4 : 2;
    cfg->c = (cfg->s_dec + 1) / 2;
    cfg->dec_step = cfg->s_dec;
    cfg->slope_samples = 8;
    return 0;
}

/* ------------------------------------------------------------ simulation */

enum { EV_READY = 0, EV_PUSHDONE = 1, EV_XFER = 2, EV_DONE = 3 };
typedef struct { double time; uint64_t seq; int32_t kind, task, worker; } event_t;

static int ev_less(const event_t* a, const event_t* b) { /* EventAfter, engine.cpp:26-31 */
    if (a->time != b->time) return a->time < b->time;
    return a->seq < b->seq;
}

typedef struct {
    const view_t* v;
    const tbsim_platform_desc* p;
    int policy;
    const tbsim_regulator_cfg* cfg;
    tbsim_regulator_state* st;
    const int64_t *ability, *efficiency, *prio;
    event_t* heap; int64_t hsz;
    uint64_t next_seq, next_qseq;
    double now;
    int64_t nready, completed;
    int32_t* unmet;
    /* per worker queue: task, seq in insertion order */
    int32_t** qtask; uint64_t** qseq; int64_t* qlen;
    char* busy; double* busy_until;
    char* resid; /* [nh * nodes] */
    int32_t* pw; double *ps, *pe;
    double makespan;
    int64_t n_push, n_pop, n_samp;
    tbsim_sim_out* o; int64_t t0;
    int64_t pop_counts[3];
} sim_t;

static void ev_push(sim_t* s, double time, int kind, int task, int worker) {
    event_t e = {time, s->next_seq++, kind, task, worker};
    int64_t i = s->hsz++;
    s->heap[i] = e;
    while (i > 0) {
        int64_t p = (i - 1) / 2;
        if (!ev_less(&s->heap[i], &s->heap[p])) break;
        event_t t = s->heap[p]; s->heap[p] = s->heap[i]; s->heap[i] = t;
        i = p;
    }
}
static event_t ev_pop(sim_t* s) {
    event_t top = s->heap[0];
    s->heap[0] = s->heap[--s->hsz];
    int64_t i = 0;
    for (;;) {
        int64_t l = 2 * i + 1, r = l + 1, m = i;
        if (l < s->hsz && ev_less(&s->heap[l], &s->heap[m])) m = l;
        if (r < s->hsz && ev_less(&s->heap[r], &s->heap[m])) m = r;
        if (m == i) break;
        event_t t = s->heap[m]; s->heap[m] = s->heap[i]; s->heap[i] = t;
        i = m;
    }
    return top;
}

static double cost_of(const sim_t* s, int32_t ty, int kind) {
    const tbsim_costs* c = &s->p->costs;
    if (ty >= c->n_types) return 0.0;
    const double* a = kind ? c->gpu_ms : c->cpu_ms;
    return a ? a[ty] : 0.0;
}
static int can_run(const sim_t* s, int32_t ty, int w) { return cost_of(s, ty, s->p->kind[w]) > 0.0; }
static double exec_ms(const sim_t* s, int32_t task, int w) { return cost_of(s, s->v->type[task], s->p->kind[w]); }

/* transfer_one_ms (src/engine.cpp:86-103) + Platform::transfer_time_ms
 * (src/platform.cpp:56-63) */
static double transfer_one(const sim_t* s, int32_t h, int to) {
    int nn = s->p->n_nodes;
    if (s->resid[(int64_t)h * nn + to]) return 0.0;
    int best = -1;
    double best_bw = -1.0;
    for (int node = 0; node < nn; ++node) {
        if (!s->resid[(int64_t)h * nn + node]) continue;
        double bw = s->p->bandwidth[node * nn + to];
        if (bw > best_bw) { best_bw = bw; best = node; }
    }
    /* best >= 0 always: handles start on node 0 and never lose residency */
    return s->p->latency_ms + (double)s->v->hbytes[h] / s->p->bandwidth[best * nn + to];
}
static double transfer_total(const sim_t* s, int32_t task, int node) { /* engine.cpp:105-110 */
    double total = 0.0;
    for (int32_t k = s->v->ioff[task]; k < s->v->ioff[task + 1]; ++k)
        total += transfer_one(s, s->v->in[k], node);
    return total;
}
static double free_at(const sim_t* s, int w) { /* engine.cpp:53-59 */
    double t = s->busy[w] ? s->busy_until[w] : s->now;
    for (int64_t i = 0; i < s->qlen[w]; ++i) t += exec_ms(s, s->qtask[w][i], w);
    return t;
}
static double resident_fraction(const sim_t* s, int32_t task, int node) { /* engine.cpp:63-74 */
    const view_t* v = s->v;
    if (v->ioff[task] == v->ioff[task + 1]) return 1.0;
    int64_t total = 0, local = 0;
    for (int32_t k = v->ioff[task]; k < v->ioff[task + 1]; ++k) {
        int32_t h = v->in[k];
        total += v->hbytes[h];
        if (s->resid[(int64_t)h * s->p->n_nodes + node]) local += v->hbytes[h];
    }
    return (double)local / (double)total;
}

/* push rules (src/policies.cpp:13-72) */
static int select_worker(sim_t* s, int32_t task, int* out) {
    int best = -1;
    double best_key = 0.0;
    for (int w = 0; w < s->p->n_workers; ++w) {
        if (!can_run(s, s->v->type[task], w)) continue;
        double key;
        if (s->policy == TBSIM_POLICY_FIFO) {
            key = (double)s->qlen[w] + (s->busy[w] ? 1.0 : 0.0);
        } else {
            double fa = free_at(s, w);
            double start = s->now > fa ? s->now : fa;
            if (s->policy == TBSIM_POLICY_DM)
                key = start + exec_ms(s, task, w);
            else
                key = start + transfer_total(s, task, s->p->memory_node[w]) + exec_ms(s, task, w);
        }
        if (best < 0 || key < best_key) { best = w; best_key = key; }
    }
    if (best < 0) {
        char buf[32];
        return fail(TBSIM_E_RUNTIME, "no worker can run task type %s",
                    type_name(s->v, s->v->type[task], buf));
    }
    *out = best;
    return 0;
}

/* pop rules (src/policies.cpp:74-137) */
static int64_t select_entry(sim_t* s, int w) {
    int64_t len = s->qlen[w];
    int32_t* qt = s->qtask[w];
    uint64_t* qs = s->qseq[w];
    int64_t best = 0;
    if (s->policy <= TBSIM_POLICY_DMDA) {
        for (int64_t i = 1; i < len; ++i) if (qs[i] < qs[best]) best = i;
        return best;
    }
    if (s->policy == TBSIM_POLICY_DMDAP) {
        for (int64_t i = 1; i < len; ++i) {
            int64_t p = s->prio[qt[i]], bp = s->prio[qt[best]];
            if (p > bp || (p == bp && qs[i] < qs[best])) best = i;
        }
        return best;
    }
    int mode = s->st->mode;
    s->pop_counts[mode] += 1;
    int node = s->p->memory_node[w];
    double bk0, bk1;
#define KEY(i, k0, k1)                                                           \
    do {                                                                         \
        int32_t t_ = qt[i];                                                      \
        if (mode == TBSIM_MODE_ABILITY) { k0 = (double)s->ability[t_]; k1 = 0.0; } \
        else if (mode == TBSIM_MODE_EFFICIENCY) { k0 = (double)s->efficiency[t_]; k1 = 0.0; } \
        else { k0 = resident_fraction(s, t_, node); k1 = (double)s->efficiency[t_]; } \
    } while (0)
    KEY(0, bk0, bk1);
    for (int64_t i = 1; i < len; ++i) {
        double k0, k1;
        KEY(i, k0, k1);
        if (k0 > bk0 || (k0 == bk0 && k1 > bk1)) {
            best = i; bk0 = k0; bk1 = k1;
        } else if (k0 == bk0 && k1 == bk1) {
            int64_t p = s->prio[qt[i]], bp = s->prio[qt[best]];
            if (p > bp || (p == bp && qs[i] < qs[best])) best = i;
        }
    }
#undef KEY
    return best;
}

static void record_sample(sim_t* s) {
    if (s->o->sample_time) {
        s->o->sample_time[2 * s->t0 + s->n_samp] = s->now;
        s->o->sample_nready[2 * s->t0 + s->n_samp] = s->nready;
    }
    s->n_samp++;
}

static void queue_event(sim_t* s) {
    if (s->policy == TBSIM_POLICY_INSPIRIT) orc_regulator_step(s->st, s->cfg, s->nready, s->now);
}

static void maybe_dispatch(sim_t* s, int w) { /* engine.cpp:143-166 */
    if (s->busy[w] || s->qlen[w] == 0) return;
    int64_t pick = select_entry(s, w);
    int32_t task = s->qtask[w][pick];
    for (int64_t i = pick; i + 1 < s->qlen[w]; ++i) {
        s->qtask[w][i] = s->qtask[w][i + 1];
        s->qseq[w][i] = s->qseq[w][i + 1];
    }
    s->qlen[w]--;
    s->nready -= 1;
    if (s->o->pop_time) {
        s->o->pop_time[s->t0 + s->n_pop] = s->now;
        s->o->pop_task[s->t0 + s->n_pop] = task;
        s->o->pop_worker[s->t0 + s->n_pop] = w;
    }
    s->n_pop++;
    record_sample(s);
    queue_event(s);
    double transfer = transfer_total(s, task, s->p->memory_node[w]);
    double exec = exec_ms(s, task, w);
    double start = s->now + transfer;
    double end = start + exec;
    s->pw[task] = w; s->ps[task] = start; s->pe[task] = end;
    s->busy[w] = 1;
    s->busy_until[w] = end;
    if (transfer > 0.0) ev_push(s, start, EV_XFER, task, w);
    ev_push(s, end, EV_DONE, task, w);
}

static int on_push(sim_t* s, int32_t task) { /* engine.cpp:124-141 */
    int w;
    int rc = select_worker(s, task, &w);
    if (rc) return rc;
    s->qtask[w][s->qlen[w]] = task;
    s->qseq[w][s->qlen[w]] = s->next_qseq++;
    s->qlen[w]++;
    s->nready += 1;
    if (s->o->push_time) {
        s->o->push_time[s->t0 + s->n_push] = s->now;
        s->o->push_task[s->t0 + s->n_push] = task;
    }
    s->n_push++;
    record_sample(s);
    queue_event(s);
    maybe_dispatch(s, w);
    return 0;
}

int orc_simulate(const tbsim_batch_desc* b, const tbsim_platform_desc* platforms,
                 const int32_t* platform_of, int policy, const tbsim_regulator_cfg* reg,
                 const tbsim_attr_in* attrs, tbsim_sim_out* o) {
    for (int64_t g = 0; g < b->n_graphs; ++g) {
        view_t v;
        view_open(&v, b, g);
        sim_t s;
        memset(&s, 0, sizeof s);
        s.v = &v;
        s.p = &platforms[platform_of ? platform_of[g] : 0];
        s.policy = policy;
        s.o = o;
        s.t0 = b->task_base[g];
        int64_t n = v.n, W = s.p->n_workers, nn = s.p->n_nodes;
        tbsim_regulator_cfg cfg;
        int rc = 0;
        if (reg) cfg = reg[g];
        else rc = orc_default_regulator_config(b, g, s.p, &cfg);
        if (rc) { view_close(&v); return rc; }
        s.cfg = &cfg;
        tbsim_regulator_state st0;
        memset(&st0, 0, sizeof st0);
        st0.mode = TBSIM_MODE_EFFICIENCY;
        st0.phase = TBSIM_PHASE_INC;
        st0.s_dec_count = 1;
        s.st = o->reg_state ? &o->reg_state[g] : &st0;
        int64_t* zeros = XALLOC(int64_t, n);
        s.ability = attrs && attrs->ability ? attrs->ability + s.t0 : zeros;
        s.efficiency = attrs && attrs->efficiency ? attrs->efficiency + s.t0 : zeros;
        s.prio = attrs && attrs->static_priority ? attrs->static_priority + s.t0 : zeros;
        s.heap = XALLOC(event_t, 4 * n + 8);
        s.unmet = XALLOC(int32_t, n);
        s.qtask = XALLOC(int32_t*, W);
        s.qseq = XALLOC(uint64_t*, W);
        for (int64_t w = 0; w < W; ++w) { s.qtask[w] = XALLOC(int32_t, n); s.qseq[w] = XALLOC(uint64_t, n); }
        s.qlen = XALLOC(int64_t, W);
        s.busy = XALLOC(char, W);
        s.busy_until = XALLOC(double, W);
        s.resid = XALLOC(char, v.nh * nn);
        s.pw = XALLOC(int32_t, n); s.ps = XALLOC(double, n); s.pe = XALLOC(double, n);
        for (int64_t i = 0; i < n; ++i) s.pw[i] = -1;
        for (int64_t h = 0; h < v.nh; ++h) s.resid[h * nn] = 1; /* engine.cpp:215-216 */
        for (int64_t i = 0; i < n; ++i) {                       /* engine.cpp:218-221 */
            s.unmet[i] = v.poff[i + 1] - v.poff[i];
            if (s.unmet[i] == 0) ev_push(&s, 0.0, EV_READY, (int)i, -1);
        }
        while (!rc && s.hsz > 0) { /* engine.cpp:223-233 */
            event_t e = ev_pop(&s);
            s.now = e.time;
            switch (e.kind) {
            case EV_READY: ev_push(&s, s.now, EV_PUSHDONE, e.task, -1); break;
            case EV_PUSHDONE: rc = on_push(&s, e.task); break;
            case EV_XFER: { /* engine.cpp:168-172 */
                int node = s.p->memory_node[e.worker];
                for (int32_t k = v.ioff[e.task]; k < v.ioff[e.task + 1]; ++k)
                    s.resid[(int64_t)v.in[k] * nn + node] = 1;
                break;
            }
            case EV_DONE: { /* engine.cpp:174-185 */
                int node = s.p->memory_node[e.worker];
                for (int32_t k = v.ooff[e.task]; k < v.ooff[e.task + 1]; ++k)
                    s.resid[(int64_t)v.out[k] * nn + node] = 1;
                s.busy[e.worker] = 0;
                s.completed++;
                if (s.now > s.makespan) s.makespan = s.now;
                for (int32_t k = v.soff[e.task]; k < v.soff[e.task + 1]; ++k)
                    if (--s.unmet[v.succ[k]] == 0) ev_push(&s, s.now, EV_READY, v.succ[k], -1);
                maybe_dispatch(&s, e.worker);
                break;
            }
            }
        }
        if (!rc) {
            for (int64_t i = 0; i < n; ++i) {
                if (o->worker) o->worker[s.t0 + i] = s.pw[i];
                if (o->start_ms) o->start_ms[s.t0 + i] = s.ps[i];
                if (o->end_ms) o->end_ms[s.t0 + i] = s.pe[i];
            }
            if (o->makespan_ms) o->makespan_ms[g] = s.makespan;
            if (o->completed) o->completed[g] = s.completed;
            if (o->pop_mode_counts)
                for (int m = 0; m < 3; ++m) o->pop_mode_counts[3 * g + m] = s.pop_counts[m];
            if (s.completed != n) { /* engine.cpp:235-246 */
                char msg[1024];
                int len = snprintf(msg, sizeof msg, "simulation stuck with %lld tasks unfinished:",
                                   (long long)(n - s.completed));
                int listed = 0;
                for (int64_t i = 0; i < n && listed < 20; ++i)
                    if (s.pw[i] < 0) {
                        len += snprintf(msg + len, sizeof msg - (size_t)len, " %lld",
                                        (long long)task_ident(&v, i));
                        listed++;
                    }
                if (listed < n - s.completed) snprintf(msg + len, sizeof msg - (size_t)len, " ...");
                rc = fail(TBSIM_E_RUNTIME, "%s", msg);
            }
        }
        for (int64_t w = 0; w < W; ++w) { free(s.qtask[w]); free(s.qseq[w]); }
        free(s.qtask); free(s.qseq); free(s.qlen); free(s.busy); free(s.busy_until);
        free(s.resid); free(s.pw); free(s.ps); free(s.pe); free(s.heap); free(s.unmet); free(zeros);
        view_close(&v);
        if (rc) return rc;
    }
    return 0;
}

/* ------------------------------------------------------------ generators */

/* MT19937-64 (the engine std::mt19937_64 specifies: w=64, n=312, m=156,
 * r=31, a=0xB5026F5AA96619E9, u=29 d=0x5555555555555555, s=17
 * b=0x71D67FFFEDA60000, t=37 c=0xFFF7EEE000000000, l=43, f=6364136223846793005). */
typedef struct { uint64_t mt[312]; int idx; } mt64_t;

static void mt_seed(mt64_t* m, uint64_t seed) {
    m->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        m->mt[i] = 6364136223846793005ull * (m->mt[i - 1] ^ (m->mt[i - 1] >> 62)) + (uint64_t)i;
    m->idx = 312;
}
static uint64_t mt_next(mt64_t* m) {
    if (m->idx >= 312) {
        const uint64_t UM = 0xFFFFFFFF80000000ull, LM = 0x7FFFFFFFull;
        for (int i = 0; i < 312; ++i) {
            uint64_t x = (m->mt[i] & UM) | (m->mt[(i + 1) % 312] & LM);
            uint64_t xa = x >> 1;
            if (x & 1) xa ^= 0xB5026F5AA96619E9ull;
            m->mt[i] = m->mt[(i + 156) % 312] ^ xa;
        }
        m->idx = 0;
    }
    uint64_t x = m->mt[m->idx++];
    x ^= (x >> 29) & 0x5555555555555555ull;
    x ^= (x << 17) & 0x71D67FFFEDA60000ull;
    x ^= (x << 37) & 0xFFF7EEE000000000ull;
    x ^= x >> 43;
    return x;
}
static double uniform01(mt64_t* m) { return (double)(mt_next(m) >> 11) * 0x1.0p-53; } /* generators.cpp:20-22 */
static uint64_t uniform_below(mt64_t* m, uint64_t n) { return mt_next(m) % n; }      /* generators.cpp:24-26 */

enum { TY_GEMM = 0, TY_SYRK, TY_TRSM, TY_POTRF, TY_GETRF, TY_STENCIL,
       TY_L0, TY_L1, TY_L2, TY_L3, TY_UNIT };

typedef struct {
    int32_t *dep_off, *dep, *in_off, *in, *out_off, *out, *type;
    int64_t n, n_dep, n_in, n_out, cap_t, cap_d, cap_i, cap_o;
} gbuild_t;

static void gb_init(gbuild_t* b, int64_t cap_t) {
    memset(b, 0, sizeof *b);
    b->cap_t = cap_t; b->cap_d = b->cap_i = b->cap_o = 4 * cap_t + 16;
    b->dep_off = XALLOC(int32_t, cap_t + 1); b->in_off = XALLOC(int32_t, cap_t + 1);
    b->out_off = XALLOC(int32_t, cap_t + 1); b->type = XALLOC(int32_t, cap_t);
    b->dep = XALLOC(int32_t, b->cap_d); b->in = XALLOC(int32_t, b->cap_i); b->out = XALLOC(int32_t, b->cap_o);
}
static void gb_grow(int32_t** a, int64_t* cap, int64_t need) {
    if (need <= *cap) return;
    while (*cap < need) *cap *= 2;
    *a = (int32_t*)realloc(*a, sizeof(int32_t) * (size_t)*cap);
}
static int32_t gb_add(gbuild_t* b, int32_t type, const int32_t* deps, int nd, const int32_t* in,
                      int ni, const int32_t* out, int no) {
    gb_grow(&b->dep, &b->cap_d, b->n_dep + nd);
    gb_grow(&b->in, &b->cap_i, b->n_in + ni);
    gb_grow(&b->out, &b->cap_o, b->n_out + no);
    for (int k = 0; k < nd; ++k) b->dep[b->n_dep++] = deps[k];
    for (int k = 0; k < ni; ++k) b->in[b->n_in++] = in[k];
    for (int k = 0; k < no; ++k) b->out[b->n_out++] = out[k];
    b->type[b->n] = type;
    b->n++;
    b->dep_off[b->n] = (int32_t)b->n_dep;
    b->in_off[b->n] = (int32_t)b->n_in;
    b->out_off[b->n] = (int32_t)b->n_out;
    return (int32_t)(b->n - 1);
}
static void gb_finish(gbuild_t* b, orc_graph* g, int64_t nh, int64_t bytes_each) {
    g->n = (int32_t)b->n; g->n_dep = (int32_t)b->n_dep; g->n_in = (int32_t)b->n_in;
    g->n_out = (int32_t)b->n_out; g->n_handles = (int32_t)nh;
    g->dep_off = b->dep_off; g->dep = b->dep; g->in_off = b->in_off; g->in = b->in;
    g->out_off = b->out_off; g->out = b->out; g->type = b->type;
    g->handle_bytes = XALLOC(int64_t, nh);
    for (int64_t h = 0; h < nh; ++h) g->handle_bytes[h] = bytes_each;
}

void orc_graph_free(orc_graph* g) {
    free(g->dep_off); free(g->dep); free(g->in_off); free(g->in);
    free(g->out_off); free(g->out); free(g->type); free(g->handle_bytes);
    memset(g, 0, sizeof *g);
}

static int cmp_int(const void* a, const void* b) {
    int x = *(const int*)a, y = *(const int*)b;
    return (x > y) - (x < y);
}

/* generate_layered_dag (src/generators.cpp:184-244) */
int orc_gen_layered(int32_t n_tasks, int32_t n_layers, double p, uint64_t seed, orc_graph* out) {
    if (n_layers < 1) return fail(TBSIM_E_INVALID_ARGUMENT, "autogen: n_layers must be >= 1");
    if (n_tasks < n_layers) return fail(TBSIM_E_INVALID_ARGUMENT, "autogen: n_tasks must be >= n_layers");
    if (!(p >= 0.0 && p <= 1.0)) return fail(TBSIM_E_INVALID_ARGUMENT, "autogen: edge_prob must be in [0,1]");
    mt64_t rng;
    mt_seed(&rng, seed);
    int64_t n = n_tasks;
    /* deps per task: collected into one growing array */
    int32_t* doff = XALLOC(int32_t, n + 1);
    int64_t cap = 4 * n + 16, nd = 0;
    int32_t* dep = XALLOC(int32_t, cap);
    for (int64_t i = 0; i < n; ++i) {
        int32_t layer = (int32_t)(i % n_layers);
        doff[i] = (int32_t)nd;
        if (layer == 0) continue;
        /* members of layer-1 are j = layer-1, layer-1+L, ... < n */
        int64_t first = nd, cnt = 0;
        for (int64_t j = layer - 1; j < n; j += n_layers) {
            cnt++;
            if (uniform01(&rng) < p) {
                gb_grow(&dep, &cap, nd + 1);
                dep[nd++] = (int32_t)j;
            }
        }
        if (nd == first) {
            gb_grow(&dep, &cap, nd + 1);
            dep[nd++] = (int32_t)(layer - 1 + (int64_t)uniform_below(&rng, (uint64_t)cnt) * n_layers);
        }
    }
    doff[n] = (int32_t)nd;
    int* degree = XALLOC(int, n);
    for (int64_t i = 0; i < n; ++i) {
        degree[i] += doff[i + 1] - doff[i];
        for (int32_t k = doff[i]; k < doff[i + 1]; ++k) degree[dep[k]] += 1;
    }
    int* sorted = XALLOC(int, n);
    memcpy(sorted, degree, sizeof(int) * (size_t)n);
    qsort(sorted, (size_t)n, sizeof(int), cmp_int);
    int q1 = sorted[(size_t)((double)(n - 1) * 0.25)];
    int q2 = sorted[(size_t)((double)(n - 1) * 0.5)];
    int q3 = sorted[(size_t)((double)(n - 1) * 0.75)];
    static const int64_t tiles[4] = {160 * 160 * 4, 320 * 320 * 4, 640 * 640 * 4, 960 * 960 * 4};
    out->n = (int32_t)n; out->n_dep = (int32_t)nd; out->n_in = (int32_t)nd;
    out->n_out = (int32_t)n; out->n_handles = (int32_t)n;
    out->handle_bytes = XALLOC(int64_t, n);
    for (int64_t i = 0; i < n; ++i) out->handle_bytes[i] = tiles[uniform_below(&rng, 4)];
    out->dep_off = doff; out->dep = dep;
    out->in_off = XALLOC(int32_t, n + 1); out->in = XALLOC(int32_t, nd);
    memcpy(out->in_off, doff, sizeof(int32_t) * (size_t)(n + 1));
    memcpy(out->in, dep, sizeof(int32_t) * (size_t)nd);
    out->out_off = XALLOC(int32_t, n + 1); out->out = XALLOC(int32_t, n);
    out->type = XALLOC(int32_t, n);
    for (int64_t i = 0; i < n; ++i) {
        out->out_off[i + 1] = (int32_t)(i + 1);
        out->out[i] = (int32_t)i;
        int d = degree[i];
        out->type[i] = TY_L0 + (d <= q1 ? 0 : d <= q2 ? 1 : d <= q3 ? 2 : 3);
    }
    free(degree); free(sorted);
    return 0;
}

/* build_cholesky_dag (src/generators.cpp:30-87): lower-triangular tiles. */
int orc_gen_cholesky(int32_t nb, int64_t bytes, orc_graph* out) {
    if (nb < 1) return fail(TBSIM_E_INVALID_ARGUMENT, "cholesky: nblocks must be >= 1");
    if (bytes <= 0) return fail(TBSIM_E_INVALID_ARGUMENT, "cholesky: block_bytes must be > 0");
    int64_t n = nb;
    int32_t* tile = XALLOC(int32_t, n * n);
    int32_t nh = 0;
    for (int64_t i = 0; i < n; ++i)
        for (int64_t j = 0; j <= i; ++j) tile[i * n + j] = nh++;
    int32_t* potrf = XALLOC(int32_t, n);
    int32_t* trsm = XALLOC(int32_t, n * n);
    int32_t* syrk = XALLOC(int32_t, n * n);
    int32_t* gemm = XALLOC(int32_t, n * n);
    gbuild_t b;
    gb_init(&b, n * n * n / 3 + 4 * n + 8);
    for (int64_t k = 0; k < n; ++k) {
        int32_t d[3], in[3], o[1];
        int nd = 0;
        if (k > 0) d[nd++] = syrk[k * n + k - 1];
        in[0] = tile[k * n + k]; o[0] = tile[k * n + k];
        potrf[k] = gb_add(&b, TY_POTRF, d, nd, in, 1, o, 1);
        for (int64_t i = k + 1; i < n; ++i) {
            nd = 0;
            d[nd++] = potrf[k];
            if (k > 0) d[nd++] = gemm[i * n + k];
            in[0] = tile[k * n + k]; in[1] = tile[i * n + k]; o[0] = tile[i * n + k];
            trsm[i * n + k] = gb_add(&b, TY_TRSM, d, nd, in, 2, o, 1);
        }
        for (int64_t i = k + 1; i < n; ++i) {
            nd = 0;
            d[nd++] = trsm[i * n + k];
            if (k > 0) d[nd++] = syrk[i * n + k - 1];
            in[0] = tile[i * n + k]; in[1] = tile[i * n + i]; o[0] = tile[i * n + i];
            syrk[i * n + k] = gb_add(&b, TY_SYRK, d, nd, in, 2, o, 1);
            for (int64_t j = k + 1; j < i; ++j) {
                nd = 0;
                d[nd++] = trsm[i * n + k];
                d[nd++] = trsm[j * n + k];
                if (k > 0) d[nd++] = gemm[i * n + j];
                in[0] = tile[i * n + k]; in[1] = tile[j * n + k]; in[2] = tile[i * n + j];
                o[0] = tile[i * n + j];
                gemm[i * n + j] = gb_add(&b, TY_GEMM, d, nd, in, 3, o, 1);
            }
        }
    }
    gb_finish(&b, out, nh, bytes);
    free(tile); free(potrf); free(trsm); free(syrk); free(gemm);
    return 0;
}

/* build_lu_dag (src/generators.cpp:89-142): full tile grid, no pivoting. */
int orc_gen_lu(int32_t nb, int64_t bytes, orc_graph* out) {
    if (nb < 1) return fail(TBSIM_E_INVALID_ARGUMENT, "lu: nblocks must be >= 1");
    if (bytes <= 0) return fail(TBSIM_E_INVALID_ARGUMENT, "lu: block_bytes must be > 0");
    int64_t n = nb;
    int32_t* getrf = XALLOC(int32_t, n);
    int32_t* trow = XALLOC(int32_t, n * n);
    int32_t* tcol = XALLOC(int32_t, n * n);
    int32_t* gemm = XALLOC(int32_t, n * n);
#define TILE(i, j) ((int32_t)((i) * n + (j)))
    gbuild_t b;
    gb_init(&b, n * n * n / 3 + 2 * n * n + 8);
    for (int64_t k = 0; k < n; ++k) {
        int32_t d[3], in[3], o[1];
        int nd = 0;
        if (k > 0) d[nd++] = gemm[k * n + k];
        in[0] = TILE(k, k); o[0] = TILE(k, k);
        getrf[k] = gb_add(&b, TY_GETRF, d, nd, in, 1, o, 1);
        for (int64_t j = k + 1; j < n; ++j) {
            nd = 0;
            d[nd++] = getrf[k];
            if (k > 0) d[nd++] = gemm[k * n + j];
            in[0] = TILE(k, k); in[1] = TILE(k, j); o[0] = TILE(k, j);
            trow[k * n + j] = gb_add(&b, TY_TRSM, d, nd, in, 2, o, 1);
        }
        for (int64_t i = k + 1; i < n; ++i) {
            nd = 0;
            d[nd++] = getrf[k];
            if (k > 0) d[nd++] = gemm[i * n + k];
            in[0] = TILE(k, k); in[1] = TILE(i, k); o[0] = TILE(i, k);
            tcol[i * n + k] = gb_add(&b, TY_TRSM, d, nd, in, 2, o, 1);
        }
        for (int64_t i = k + 1; i < n; ++i)
            for (int64_t j = k + 1; j < n; ++j) {
                nd = 0;
                d[nd++] = tcol[i * n + k];
                d[nd++] = trow[k * n + j];
                if (k > 0) d[nd++] = gemm[i * n + j];
                in[0] = TILE(i, k); in[1] = TILE(k, j); in[2] = TILE(i, j);
                o[0] = TILE(i, j);
                gemm[i * n + j] = gb_add(&b, TY_GEMM, d, nd, in, 3, o, 1);
            }
    }
#undef TILE
    gb_finish(&b, out, n * n, bytes);
    free(getrf); free(trow); free(tcol); free(gemm);
    return 0;
}
