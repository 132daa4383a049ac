/*
 * radial_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the CPU reference's hot path, used solely as the
 * parity checker by tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg.  Nothing in paper_2506_19852_b200/ links or calls this
 * file; the product path is the CUDA library and fails loudly without it.
 *
 * Every function cites the reference file:line it restates
 * (/root/reference/proj/include/radial/...).  Parity of this restatement is
 * pinned against the reference itself (oracle/_ref, built from the
 * reference headers by oracle/Makefile) and against the golden sha256
 * vectors of SURVEY.md section 8c (tests/golden/layouts.json).
 *
 * The backward restatement (ro_attention_bwd) has no reference counterpart (the
 * reference has no gradient code): its parity is unpinned by the
 * reference and is cross-checked only against torch float64 autograd and
 * finite differences (tests/test_oracle.py).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

#define RO_KIND_RADIAL 0
#define RO_KIND_DENSE 1
#define RO_KIND_SPATIAL 2
#define RO_KIND_TEMPORAL 3
#define RO_KIND_STA 4
#define RO_KIND_POWER 5
#define RO_KIND_HARMONIC 6

typedef struct {
    int kind;
    int sink;
    int has_tw, has_sw;
    uint32_t tw, sw;
} ro_pattern;

/* ------------------------------------------------------------------------ */
/* mask.hpp:22-35  floor_log2 / band_exponent                                */
/* ------------------------------------------------------------------------ */
static uint32_t ro_floor_log2(uint64_t x) {
    uint32_t e = 0;
    while (x >= 2) {
        x >>= 1;
        ++e;
    }
    return e;
}
static uint32_t ro_band_exponent(uint64_t d) { return ro_floor_log2(d < 1 ? 1 : d); }

/* ------------------------------------------------------------------------ */
/* mask.hpp:105-154  detail::kept_span (all frame-structured kinds)          */
/* returns 1 and [*lo,*hi] when frame j keeps an interval, 0 otherwise,      */
/* -1 for the power kind (no per-frame span) or a missing window.            */
/* ------------------------------------------------------------------------ */
int ro_kept_span(int kind, int sink, uint32_t tw, uint32_t sw, uint32_t s, uint32_t i,
                 uint32_t k_lo, uint32_t k_hi, uint32_t j, uint32_t* lo, uint32_t* hi) {
    const uint64_t d = i < j ? (uint64_t)(j - i) : (uint64_t)(i - j);
#define RO_BAND(sigma_)                                                        \
    do {                                                                       \
        uint32_t sg_ = (sigma_);                                               \
        *lo = k_lo > sg_ ? k_lo - sg_ : 0;                                     \
        uint64_t h64_ = (uint64_t)k_hi + sg_;                                  \
        *hi = h64_ >= s ? s - 1 : (uint32_t)h64_;                              \
        return 1;                                                              \
    } while (0)
    if (sink && j == 0) { /* mask.hpp:120 */
        *lo = 0;
        *hi = s - 1;
        return 1;
    }
    switch (kind) {
        case RO_KIND_DENSE:
            *lo = 0;
            *hi = s - 1;
            return 1;
        case RO_KIND_RADIAL: { /* mask.hpp:125-131 */
            uint64_t pw = (uint64_t)1 << ro_band_exponent(d);
            if (pw <= s) RO_BAND((uint32_t)(s / pw) - 1);
            uint64_t period = (pw + s - 1) / s;
            if (d % period == 0) {
                *lo = k_lo;
                *hi = k_hi;
                return 1;
            }
            return 0;
        }
        case RO_KIND_SPATIAL:
            if (d <= tw) {
                *lo = 0;
                *hi = s - 1;
                return 1;
            }
            return 0;
        case RO_KIND_TEMPORAL:
            RO_BAND(sw < s - 1 ? sw : s - 1);
        case RO_KIND_STA:
            if (d <= tw) RO_BAND(sw < s - 1 ? sw : s - 1);
            return 0;
        case RO_KIND_HARMONIC: {
            uint64_t dist = d < 1 ? 1 : d;
            uint64_t width = s / dist;
            if (width >= 1) RO_BAND((uint32_t)width - 1);
            uint64_t period = (dist + s - 1) / s;
            if (d % period == 0) {
                *lo = k_lo;
                *hi = k_hi;
                return 1;
            }
            return 0;
        }
        default:
            return -1;
    }
#undef RO_BAND
}

/* mask.hpp:165-176  radial_keep (token predicate, exact integer width test) */
int ro_radial_keep(uint32_t i, uint32_t j, uint32_t k, uint32_t l, uint32_t s, int sink) {
    if (sink && j == 0) return 1;
    const uint64_t d = i < j ? (uint64_t)(j - i) : (uint64_t)(i - j);
    const uint64_t pw = (uint64_t)1 << ro_band_exponent(d);
    const uint64_t dk = k < l ? (uint64_t)(l - k) : (uint64_t)(k - l);
    if (pw <= s && dk + 1 <= s / pw) return 1;
    const uint64_t period = (pw + s - 1) / s;
    return d % period == 0 && k == l;
}

/* block.hpp:47-54 grid_rows_for */
uint64_t ro_grid_rows(uint32_t f, uint32_t s, uint32_t B) {
    uint64_t n = (uint64_t)f * s;
    return (n + B - 1) / B;
}

/* ------------------------------------------------------------------------ */
/* block.hpp:59-120  blockify, row by row (painting restatement).            */
/* hit: scratch of R bytes. Emits the row's kept J ascending into out        */
/* (may be NULL) and returns the count.                                      */
/* ------------------------------------------------------------------------ */
static uint64_t ro_block_row(uint32_t f, uint32_t s, uint32_t B, const ro_pattern* p,
                             uint64_t R, uint64_t I, uint8_t* hit, uint32_t* out) {
    const uint64_t n = (uint64_t)f * s;
    memset(hit, 0, R);
    if (p->kind == RO_KIND_POWER) { /* block.hpp:71-80 */
        for (uint64_t t = 0; t < R; t = t == 0 ? 1 : t << 1) {
            if (I >= t) hit[I - t] = 1;
            if (I + t < R) hit[I + t] = 1;
        }
        if (p->sink) {
            uint64_t last = (s - 1) / B;
            for (uint64_t J = 0; J <= last && J < R; ++J) hit[J] = 1;
        }
    } else { /* block.hpp:81-97 */
        const uint64_t u0 = I * B;
        const uint64_t u1 = ((I + 1) * B < n ? (I + 1) * B : n) - 1;
        for (uint64_t i = u0 / s; i * s <= u1; ++i) {
            uint64_t k_lo = (u0 > i * s ? u0 : i * s) - i * s;
            uint64_t k_hi = (u1 < i * s + s - 1 ? u1 : i * s + s - 1) - i * s;
            for (uint32_t j = 0; j < f; ++j) {
                uint32_t lo, hi;
                int r = ro_kept_span(p->kind, p->sink, p->tw, p->sw, s, (uint32_t)i,
                                     (uint32_t)k_lo, (uint32_t)k_hi, j, &lo, &hi);
                if (r != 1) continue;
                uint64_t v_lo = (uint64_t)j * s + lo, v_hi = (uint64_t)j * s + hi;
                for (uint64_t J = v_lo / B; J <= v_hi / B; ++J) hit[J] = 1;
            }
        }
    }
    uint64_t c = 0;
    for (uint64_t J = 0; J < R; ++J)
        if (hit[J]) {
            if (out) out[c] = (uint32_t)J;
            ++c;
        }
    return c;
}

/* Fills row_ptr[R+1] (u64). Returns nnz, or -1 on bad arguments. */
int64_t ro_blockify_rowptr(uint32_t f, uint32_t s, uint32_t B, int kind, int sink, uint32_t tw,
                           uint32_t sw, uint64_t* row_ptr) {
    if (f < 1 || s < 1 || B < 1) return -1;
    ro_pattern p = {kind, sink, 1, 1, tw, sw};
    uint64_t R = ro_grid_rows(f, s, B);
    uint8_t* hit = (uint8_t*)malloc(R ? R : 1);
    row_ptr[0] = 0;
    for (uint64_t I = 0; I < R; ++I) row_ptr[I + 1] = row_ptr[I] + ro_block_row(f, s, B, &p, R, I, hit, NULL);
    free(hit);
    return (int64_t)row_ptr[R];
}

/* Fills col_idx for a row_ptr produced by ro_blockify_rowptr. */
int ro_blockify_colidx(uint32_t f, uint32_t s, uint32_t B, int kind, int sink, uint32_t tw,
                       uint32_t sw, const uint64_t* row_ptr, uint32_t* col_idx) {
    ro_pattern p = {kind, sink, 1, 1, tw, sw};
    uint64_t R = ro_grid_rows(f, s, B);
    uint8_t* hit = (uint8_t*)malloc(R ? R : 1);
    for (uint64_t I = 0; I < R; ++I) ro_block_row(f, s, B, &p, R, I, hit, col_idx + row_ptr[I]);
    free(hit);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* block.hpp:218-237  serialize (.ramk, little endian)                       */
/* returns the byte count; writes only when out != NULL                       */
/* ------------------------------------------------------------------------ */
static size_t put_le(uint8_t* out, size_t pos, uint64_t v, int bytes) {
    if (out)
        for (int b = 0; b < bytes; ++b) out[pos + b] = (uint8_t)(v >> (8 * b));
    return pos + bytes;
}
size_t ro_serialize(uint32_t f, uint32_t s, uint32_t B, int kind, int sink, uint64_t R,
                    const uint64_t* row_ptr, const uint32_t* col_idx, uint8_t* out) {
    size_t pos = 0;
    const char magic[4] = {'R', 'A', 'M', 'K'};
    for (int c = 0; c < 4; ++c) pos = put_le(out, pos, (uint8_t)magic[c], 1);
    pos = put_le(out, pos, 1, 2);
    pos = put_le(out, pos, f, 4);
    pos = put_le(out, pos, s, 4);
    pos = put_le(out, pos, B, 4);
    pos = put_le(out, pos, (uint8_t)kind, 1);
    pos = put_le(out, pos, sink ? 1 : 0, 1);
    pos = put_le(out, pos, (uint32_t)R, 4);
    for (uint64_t I = 0; I <= R; ++I) pos = put_le(out, pos, row_ptr[I], 8);
    for (uint64_t e = 0; e < row_ptr[R]; ++e) pos = put_le(out, pos, col_idx[e], 4);
    return pos;
}

/* ------------------------------------------------------------------------ */
/* attention.hpp:89-104  random_instance: mt19937_64 + libstdc++             */
/* normal_distribution<double> (Marsaglia polar, cached second value).       */
/* ------------------------------------------------------------------------ */
typedef struct {
    uint64_t mt[312];
    int idx;
} ro_mt64;
static void mt64_seed(ro_mt64* g, uint64_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    g->idx = 312;
}
static uint64_t mt64_next(ro_mt64* g) {
    const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
    if (g->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            uint64_t x = (g->mt[i] & UM) | (g->mt[(i + 1) % 312] & LM);
            uint64_t xa = x >> 1;
            if (x & 1) xa ^= 0xB5026F5AA96619E9ULL;
            g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
        }
        g->idx = 0;
    }
    uint64_t y = g->mt[g->idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}
/* generate_canonical<double,53>(mt19937_64): one draw / 2^64, clamped < 1 */
static double mt64_canonical(ro_mt64* g) {
    double r = (double)mt64_next(g) / 18446744073709551616.0;
    if (r >= 1.0) r = nextafter(1.0, 0.0);
    return r;
}
typedef struct {
    ro_mt64 g;
    int saved_ok;
    double saved;
} ro_normal;
static double ro_normal_next(ro_normal* st) {
    if (st->saved_ok) {
        st->saved_ok = 0;
        return st->saved;
    }
    double x, y, r2;
    do {
        x = 2.0 * mt64_canonical(&st->g) - 1.0;
        y = 2.0 * mt64_canonical(&st->g) - 1.0;
        r2 = x * x + y * y;
    } while (r2 > 1.0 || r2 == 0.0);
    double mult = sqrt(-2.0 * log(r2) / r2);
    st->saved = x * mult;
    st->saved_ok = 1;
    return y * mult;
}
/* q, k, v: n*d doubles each, filled Q then K then V (attention.hpp:100-102) */
void ro_random_instance(uint64_t n, uint32_t d, uint64_t seed, double* q, double* k, double* v) {
    ro_normal st;
    mt64_seed(&st.g, seed);
    st.saved_ok = 0;
    for (uint64_t e = 0; e < n * d; ++e) q[e] = ro_normal_next(&st);
    for (uint64_t e = 0; e < n * d; ++e) k[e] = ro_normal_next(&st);
    for (uint64_t e = 0; e < n * d; ++e) v[e] = ro_normal_next(&st);
}

/* ------------------------------------------------------------------------ */
/* Host thread fan-out (restates parallel.hpp:31-58: static chunks).         */
/* ------------------------------------------------------------------------ */
typedef void (*ro_body)(void* ctx, uint64_t idx);
typedef struct {
    ro_body fn;
    void* ctx;
    uint64_t lo, hi;
} ro_chunk;
static void* ro_chunk_run(void* a) {
    ro_chunk* c = (ro_chunk*)a;
    for (uint64_t i = c->lo; i < c->hi; ++i) c->fn(c->ctx, i);
    return NULL;
}
static int ro_threads(void) {
    const char* env = getenv("RADIAL_THREADS");
    long v = env ? strtol(env, NULL, 10) : 0;
    if (v >= 1) return (int)v;
    long hw = sysconf(_SC_NPROCESSORS_ONLN);
    return hw > 0 ? (int)hw : 1;
}
static void ro_parallel_for(uint64_t count, ro_body fn, void* ctx) {
    int w = ro_threads();
    if (w <= 1 || count < 2) {
        for (uint64_t i = 0; i < count; ++i) fn(ctx, i);
        return;
    }
    if ((uint64_t)w > count) w = (int)count;
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * w);
    ro_chunk* ch = (ro_chunk*)malloc(sizeof(ro_chunk) * w);
    uint64_t chunk = (count + w - 1) / w;
    int started = 0;
    for (int t = 0; t < w; ++t) {
        uint64_t lo = (uint64_t)t * chunk, hi = lo + chunk < count ? lo + chunk : count;
        if (lo >= hi) break;
        ch[t].fn = fn;
        ch[t].ctx = ctx;
        ch[t].lo = lo;
        ch[t].hi = hi;
        pthread_create(&th[t], NULL, ro_chunk_run, &ch[t]);
        ++started;
    }
    for (int t = 0; t < started; ++t) pthread_join(th[t], NULL);
    free(th);
    free(ch);
}

/* ------------------------------------------------------------------------ */
/* attention.hpp:229-270  masked_attention(inst, BlockLayout), restated for  */
/* a chosen set of query rows (rows are independent, so this is exact for    */
/* each row). Inputs are fp32 (bf16-rounded by the caller) or fp64;          */
/* arithmetic is fp64 as in the reference. The logit is q.k * (1/sqrt(d))    */
/* (attention.hpp:128-136); `scale` overrides it when > 0.                   */
/* out: n_rows x d doubles; lse (optional): natural-log partition per row.   */
/* ------------------------------------------------------------------------ */
typedef struct {
    uint64_t n;
    uint32_t d;
    const float* qf;
    const float* kf;
    const float* vf;
    const double* qd;
    const double* kd;
    const double* vd;
    uint32_t B;
    const uint64_t* row_ptr; /* NULL => dense over all keys */
    const uint32_t* col_idx;
    const uint64_t* rows;
    double* out;
    double* lse;
    double scale;
    int status;
    uint64_t bad_row;
} ro_attn_ctx;

static inline double ro_at(const float* f, const double* dd, uint64_t idx) { return f ? (double)f[idx] : dd[idx]; }

static void ro_attn_row(void* vctx, uint64_t r) {
    ro_attn_ctx* c = (ro_attn_ctx*)vctx;
    const uint64_t u = c->rows[r];
    const uint32_t d = c->d;
    const uint64_t n = c->n;
    double* o = c->out + r * d;
    for (uint32_t e = 0; e < d; ++e) o[e] = 0.0;
    /* gather kept keys (attention.hpp:245-254) */
    uint64_t cap = 0, cnt = 0;
    uint64_t* cols = NULL;
    double* lg = NULL;
    double m = -INFINITY;
    uint64_t I = u / c->B;
    uint64_t e0 = c->row_ptr ? c->row_ptr[I] : 0;
    uint64_t e1 = c->row_ptr ? c->row_ptr[I + 1] : (n + c->B - 1) / c->B;
    for (uint64_t e = e0; e < e1; ++e) {
        uint64_t J = c->row_ptr ? c->col_idx[e] : e;
        uint64_t v_hi = (J + 1) * c->B < n ? (J + 1) * c->B : n;
        for (uint64_t v = J * c->B; v < v_hi; ++v) {
            double dot = 0.0;
            for (uint32_t x = 0; x < d; ++x)
                dot += ro_at(c->qf, c->qd, u * d + x) * ro_at(c->kf, c->kd, v * d + x);
            double l = dot * c->scale;
            if (cnt == cap) {
                cap = cap ? cap * 2 : 1024;
                cols = (uint64_t*)realloc(cols, cap * sizeof(uint64_t));
                lg = (double*)realloc(lg, cap * sizeof(double));
            }
            cols[cnt] = v;
            lg[cnt] = l;
            ++cnt;
            if (l > m) m = l;
        }
    }
    if (cnt == 0) { /* attention.hpp:255-258 */
        /* report the lowest empty row, independent of thread timing */
        uint64_t cur = __atomic_load_n(&c->bad_row, __ATOMIC_RELAXED);
        while (u < cur && !__atomic_compare_exchange_n(&c->bad_row, &cur, u, 0, __ATOMIC_RELAXED,
                                                       __ATOMIC_RELAXED)) {
        }
        __atomic_store_n(&c->status, 2, __ATOMIC_RELAXED);
        free(cols);
        free(lg);
        return;
    }
    double denom = 0.0; /* attention.hpp:259-267 */
    for (uint64_t t = 0; t < cnt; ++t) {
        double w = exp(lg[t] - m);
        denom += w;
        for (uint32_t x = 0; x < d; ++x) o[x] += w * ro_at(c->vf, c->vd, cols[t] * d + x);
    }
    for (uint32_t x = 0; x < d; ++x) o[x] /= denom;
    if (c->lse) c->lse[r] = m + log(denom);
    free(cols);
    free(lg);
}

/* returns 0, or 2 when a row keeps no keys (*bad_row = that token) */
int ro_attention_rows_f32(uint64_t n, uint32_t d, const float* q, const float* k, const float* v,
                          uint32_t B, const uint64_t* row_ptr, const uint32_t* col_idx,
                          const uint64_t* rows, uint64_t n_rows, double scale, double* out,
                          double* lse, uint64_t* bad_row) {
    ro_attn_ctx c = {n, d, q, k, v, NULL, NULL, NULL, B, row_ptr, col_idx, rows, out, lse,
                     scale > 0 ? scale : 1.0 / sqrt((double)d), 0, UINT64_MAX};
    ro_parallel_for(n_rows, ro_attn_row, &c);
    if (bad_row) *bad_row = c.bad_row;
    return c.status;
}
int ro_attention_rows_f64(uint64_t n, uint32_t d, const double* q, const double* k, const double* v,
                          uint32_t B, const uint64_t* row_ptr, const uint32_t* col_idx,
                          const uint64_t* rows, uint64_t n_rows, double scale, double* out,
                          double* lse, uint64_t* bad_row) {
    ro_attn_ctx c = {n, d, NULL, NULL, NULL, q, k, v, B, row_ptr, col_idx, rows, out, lse,
                     scale > 0 ? scale : 1.0 / sqrt((double)d), 0, UINT64_MAX};
    ro_parallel_for(n_rows, ro_attn_row, &c);
    if (bad_row) *bad_row = c.bad_row;
    return c.status;
}

/* ------------------------------------------------------------------------ */
/* Backward of attention.hpp:229-270 (no reference exists; SPEC.md:8 scopes  */
/* training out).  Exact fp64 gradients over exactly the kept blocks:        */
/*   P = softmax(S), S = scale * Q K^T restricted to kept blocks             */
/*   dV = P^T dO ; dP = dO V^T ; dS = P o (dP - rowsum(dO o O))              */
/*   dQ = scale * dS K ; dK = scale * dS^T Q                                 */
/* Serial over rows (desk-scale checker); dq/dk/dv: n x d, zeroed here.      */
/* ------------------------------------------------------------------------ */
int ro_attention_bwd_f32(uint64_t n, uint32_t d, const float* q, const float* k, const float* v,
                         const float* dout, uint32_t B, const uint64_t* row_ptr,
                         const uint32_t* col_idx, double scale, double* dq, double* dk,
                         double* dv) {
    if (scale <= 0) scale = 1.0 / sqrt((double)d);
    memset(dq, 0, sizeof(double) * n * d);
    memset(dk, 0, sizeof(double) * n * d);
    memset(dv, 0, sizeof(double) * n * d);
    double* o = (double*)malloc(sizeof(double) * d);
    uint64_t cap = 0;
    uint64_t* cols = NULL;
    double* p = NULL;
    for (uint64_t u = 0; u < n; ++u) {
        uint64_t I = u / B, cnt = 0;
        double m = -INFINITY;
        uint64_t e0 = row_ptr ? row_ptr[I] : 0, e1 = row_ptr ? row_ptr[I + 1] : (n + B - 1) / B;
        for (uint64_t e = e0; e < e1; ++e) {
            uint64_t J = row_ptr ? col_idx[e] : e;
            uint64_t v_hi = (J + 1) * B < n ? (J + 1) * B : n;
            for (uint64_t t = J * B; t < v_hi; ++t) {
                double dot = 0.0;
                for (uint32_t x = 0; x < d; ++x) dot += (double)q[u * d + x] * (double)k[t * d + x];
                if (cnt == cap) {
                    cap = cap ? cap * 2 : 1024;
                    cols = (uint64_t*)realloc(cols, cap * sizeof(uint64_t));
                    p = (double*)realloc(p, cap * sizeof(double));
                }
                cols[cnt] = t;
                p[cnt] = dot * scale;
                if (p[cnt] > m) m = p[cnt];
                ++cnt;
            }
        }
        if (cnt == 0) {
            free(o);
            free(cols);
            free(p);
            return 2;
        }
        double denom = 0.0;
        for (uint64_t t = 0; t < cnt; ++t) {
            p[t] = exp(p[t] - m);
            denom += p[t];
        }
        for (uint32_t x = 0; x < d; ++x) o[x] = 0.0;
        for (uint64_t t = 0; t < cnt; ++t) {
            p[t] /= denom;
            for (uint32_t x = 0; x < d; ++x) o[x] += p[t] * (double)v[cols[t] * d + x];
        }
        double Di = 0.0;
        for (uint32_t x = 0; x < d; ++x) Di += (double)dout[u * d + x] * o[x];
        for (uint64_t t = 0; t < cnt; ++t) {
            uint64_t kv = cols[t];
            double dp = 0.0;
            for (uint32_t x = 0; x < d; ++x) {
                dp += (double)dout[u * d + x] * (double)v[kv * d + x];
                dv[kv * d + x] += p[t] * (double)dout[u * d + x];
            }
            double ds = p[t] * (dp - Di);
            for (uint32_t x = 0; x < d; ++x) {
                dq[u * d + x] += scale * ds * (double)k[kv * d + x];
                dk[kv * d + x] += scale * ds * (double)q[u * d + x];
            }
        }
    }
    free(o);
    free(cols);
    free(p);
    return 0;
}

int ro_version(void) { return 1; }

/* ------------------------------------------------------------------------ */
/* attention.hpp:184-225  masked_attention(inst, PatternSpec): token-exact   */
/* softmax over the keys of for_each_kept_interval (mask.hpp:238-272), for   */
/* every kind (power: mask.hpp:246-270), restated for chosen query rows.    */
/* ------------------------------------------------------------------------ */
typedef struct {
    uint64_t n;
    uint32_t d, f, s;
    const float *q, *k, *v;
    ro_pattern pat;
    const uint64_t* rows;
    double* out;
    double* lse;
    double scale;
    int status;
} ro_tok_ctx;

/* Kept keys of query token u = (i, k) in the order for_each_kept_interval visits them        */
/* (mask.hpp:238-272): frame-structured kinds walk kept_span per key frame; power             */
/* (mask.hpp:246-270) keeps u and u +- 2^t, plus all of frame 0 under the sink.               */
typedef void (*ro_key_fn)(void* st, uint64_t v);

static void ro_tok_keys(const ro_tok_ctx* c, uint64_t u, ro_key_fn fn, void* st) {
    const uint32_t s = c->s;
    if (c->pat.kind == RO_KIND_POWER) {
        if (c->pat.sink)
            for (uint64_t v = 0; v < s; ++v) fn(st, v);
        if (!(c->pat.sink && u < s)) fn(st, u);
        for (uint64_t t = 1; t < c->n; t <<= 1) {
            if (u >= t && !(c->pat.sink && u - t < s)) fn(st, u - t);
            if (u + t < c->n && !(c->pat.sink && u + t < s)) fn(st, u + t);
        }
        return;
    }
    const uint32_t i = (uint32_t)(u / s), kpos = (uint32_t)(u % s);
    for (uint32_t j = 0; j < c->f; ++j) {
        uint32_t lo, hi;
        if (ro_kept_span(c->pat.kind, c->pat.sink, c->pat.tw, c->pat.sw, s, i, kpos, kpos, j, &lo, &hi) != 1) continue;
        for (uint64_t v = (uint64_t)j * s + lo; v <= (uint64_t)j * s + hi; ++v) fn(st, v);
    }
}

typedef struct {
    const ro_tok_ctx* c;
    uint64_t u;
    double m, denom;
    double* o;
} ro_tok_state;

static double ro_tok_logit(const ro_tok_state* t, uint64_t v) {
    const uint32_t d = t->c->d;
    double dot = 0.0;
    for (uint32_t x = 0; x < d; ++x) dot += (double)t->c->q[t->u * d + x] * (double)t->c->k[v * d + x];
    return dot * t->c->scale;
}

static void ro_tok_max(void* vs, uint64_t v) {
    ro_tok_state* t = (ro_tok_state*)vs;
    const double lg = ro_tok_logit(t, v);
    if (lg > t->m) t->m = lg;
}

static void ro_tok_acc(void* vs, uint64_t v) {
    ro_tok_state* t = (ro_tok_state*)vs;
    const uint32_t d = t->c->d;
    const double w = exp(ro_tok_logit(t, v) - t->m);
    t->denom += w;
    for (uint32_t x = 0; x < d; ++x) t->o[x] += w * (double)t->c->v[v * d + x];
}

static void ro_tok_row(void* vctx, uint64_t r) {
    ro_tok_ctx* c = (ro_tok_ctx*)vctx;
    const uint32_t d = c->d;
    ro_tok_state t = {c, c->rows[r], -INFINITY, 0.0, c->out + r * d};
    for (uint32_t e = 0; e < d; ++e) t.o[e] = 0.0;
    ro_tok_keys(c, t.u, ro_tok_max, &t); /* pass 1: max over kept logits */
    if (t.m == -INFINITY) {
        c->status = 2;
        return;
    }
    ro_tok_keys(c, t.u, ro_tok_acc, &t);
    for (uint32_t x = 0; x < d; ++x) t.o[x] /= t.denom;
    if (c->lse) c->lse[r] = t.m + log(t.denom);
}

int ro_token_attention_rows_f32(uint64_t n, uint32_t d, const float* q, const float* k, const float* v,
                                uint32_t f, uint32_t s, int kind, int sink, uint32_t tw, uint32_t sw,
                                const uint64_t* rows, uint64_t n_rows, double scale, double* out,
                                double* lse) {
    ro_tok_ctx c = {n, d, f, s, q, k, v, {kind, sink, 1, 1, tw, sw}, rows, out, lse,
                    scale > 0 ? scale : 1.0 / sqrt((double)d), 0};
    ro_parallel_for(n_rows, ro_tok_row, &c);
    return c.status;
}
