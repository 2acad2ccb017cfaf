/* TEST INFRASTRUCTURE ONLY — plain-C restatement of the reference hot path.
 * See specdec_oracle.h for scope and the citation convention.  Compiled with
 * -ffp-contract=off and no -march, like the reference's Release build
 * (proj/CMakeLists.txt:8-11), so every float op is a separately rounded
 * IEEE-754 single operation in the reference's order. */
#include "specdec_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

enum { OK = 0, E_CONFIG = 1, E_CAPACITY = 2, E_CONTRACT = 3, E_IO = 4, E_ERROR = 5 };

static __thread char g_err[512];

static int fail(int code, const char* fmt, ...) {
    static const char* prefix[] = {"", "config: ", "capacity: ", "contract: ", "io: ", ""};
    va_list ap;
    va_start(ap, fmt);
    int n = snprintf(g_err, sizeof g_err, "%s", prefix[code]);
    vsnprintf(g_err + n, sizeof g_err - (size_t)n, fmt, ap);
    va_end(ap);
    return code;
}
#define CHECK(cond, code, ...)                          \
    do {                                                \
        if (!(cond)) return fail((code), __VA_ARGS__);  \
    } while (0)
#define TRY(expr)                 \
    do {                          \
        int rc__ = (expr);        \
        if (rc__ != OK) return rc__; \
    } while (0)

const char* so_last_error(void) { return g_err; }

uint64_t so_fnv1a(const void* data, int64_t nbytes) {
    uint64_t hash = 14695981039346656037ULL;
    const unsigned char* b = (const unsigned char*)data;
    for (int64_t i = 0; i < nbytes; ++i) {
        hash ^= b[i];
        hash *= 1099511628211ULL;
    }
    return hash;
}

/* ---------------------------------------------------------------- rng.hpp:15-46 */
uint64_t so_splitmix_next(uint64_t* state) {
    uint64_t z = (*state += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
static float unit_float(uint64_t* st) { /* rng.hpp:23-25 */
    return (float)(so_splitmix_next(st) >> 40) * 0x1.0p-24f;
}
static double unit_double(uint64_t* st) { /* rng.hpp:28-30 */
    return (double)(so_splitmix_next(st) >> 11) * 0x1.0p-53;
}
uint64_t so_mix_seed(uint64_t a, uint64_t b, uint64_t c) { /* rng.hpp:43-46 */
    uint64_t st = a ^ (b * 0xD1B54A32D192ED03ULL) ^ (c * 0x8CB92BA72F3D8DD7ULL);
    return so_splitmix_next(&st);
}

/* ------------------------------------------------------------ model layout */
typedef struct {
    int64_t ln1_g, ln1_b, wq, bq, wk, bk, wv, bv, wo, bo, ln2_g, ln2_b, w_fc, b_fc, w_proj, b_proj;
} layer_off;

struct so_model {
    so_config cfg;
    int h, m;
    float* w; /* all tensors, declaration order (model.cpp:166-175) */
    int64_t n;
    int64_t tok, pos, lnf_g, lnf_b, lm;
    layer_off* lay;
};

int so_config_validate(const so_config* c) { /* model.cpp:12-18 */
    CHECK(c->num_layers >= 1, E_CONFIG, "num_layers must be >= 1");
    CHECK(c->num_heads >= 1, E_CONFIG, "num_heads must be >= 1");
    CHECK(c->head_dim >= 1, E_CONFIG, "head_dim must be >= 1");
    CHECK(c->vocab_size >= 2, E_CONFIG, "vocab_size must be >= 2");
    CHECK(c->max_positions >= 1, E_CONFIG, "max_positions must be >= 1");
    return OK;
}

/* model.cpp:91-118: allocate with identity LayerNorms and zero biases */
static int model_alloc(const so_config* c, so_model** out) {
    TRY(so_config_validate(c));
    so_model* m = (so_model*)calloc(1, sizeof *m);
    m->cfg = *c;
    int h = c->num_heads * c->head_dim, mm = 4 * h;
    m->h = h;
    m->m = mm;
    m->lay = (layer_off*)calloc((size_t)c->num_layers, sizeof(layer_off));
    int64_t at = 0;
#define TAKE(field, count) (field = at, at += (int64_t)(count))
    TAKE(m->tok, (int64_t)c->vocab_size * h);
    TAKE(m->pos, (int64_t)c->max_positions * h);
    for (int l = 0; l < c->num_layers; ++l) {
        layer_off* o = &m->lay[l];
        TAKE(o->ln1_g, h); TAKE(o->ln1_b, h);
        TAKE(o->wq, (int64_t)h * h); TAKE(o->bq, h);
        TAKE(o->wk, (int64_t)h * h); TAKE(o->bk, h);
        TAKE(o->wv, (int64_t)h * h); TAKE(o->bv, h);
        TAKE(o->wo, (int64_t)h * h); TAKE(o->bo, h);
        TAKE(o->ln2_g, h); TAKE(o->ln2_b, h);
        TAKE(o->w_fc, (int64_t)mm * h); TAKE(o->b_fc, mm);
        TAKE(o->w_proj, (int64_t)h * mm); TAKE(o->b_proj, h);
    }
    TAKE(m->lnf_g, h);
    TAKE(m->lnf_b, h);
    TAKE(m->lm, (int64_t)c->vocab_size * h);
#undef TAKE
    m->n = at;
    m->w = (float*)calloc((size_t)at, sizeof(float));
    if (m->w == NULL) {
        free(m->lay);
        free(m);
        return fail(E_ERROR, "out of host memory for %lld weights", (long long)at);
    }
    for (int l = 0; l < c->num_layers; ++l) {
        for (int i = 0; i < h; ++i) {
            m->w[m->lay[l].ln1_g + i] = 1.0f;
            m->w[m->lay[l].ln2_g + i] = 1.0f;
        }
    }
    for (int i = 0; i < h; ++i) m->w[m->lnf_g + i] = 1.0f;
    *out = m;
    return OK;
}

static void fill_uniform(float* t, int64_t n, uint64_t* st, float limit) { /* model.cpp:76-78 */
    for (int64_t i = 0; i < n; ++i) t[i] = (2.0f * unit_float(st) - 1.0f) * limit;
}
static float xavier_limit(int fan_in, int fan_out) { /* model.cpp:80-82 */
    return sqrtf(6.0f / (float)(fan_in + fan_out));
}

int so_model_init(const so_config* c, so_model** out) { /* model.cpp:120-139 */
    so_model* m;
    TRY(model_alloc(c, &m));
    int h = m->h, mm = m->m;
    uint64_t st = c->init_seed;
    fill_uniform(m->w + m->tok, (int64_t)c->vocab_size * h, &st, 0.1f);
    fill_uniform(m->w + m->pos, (int64_t)c->max_positions * h, &st, 0.1f);
    for (int l = 0; l < c->num_layers; ++l) {
        layer_off* o = &m->lay[l];
        fill_uniform(m->w + o->wq, (int64_t)h * h, &st, xavier_limit(h, h));
        fill_uniform(m->w + o->wk, (int64_t)h * h, &st, xavier_limit(h, h));
        fill_uniform(m->w + o->wv, (int64_t)h * h, &st, xavier_limit(h, h));
        fill_uniform(m->w + o->wo, (int64_t)h * h, &st, xavier_limit(h, h));
        fill_uniform(m->w + o->w_fc, (int64_t)mm * h, &st, xavier_limit(h, mm));
        fill_uniform(m->w + o->w_proj, (int64_t)h * mm, &st, xavier_limit(mm, h));
    }
    fill_uniform(m->w + m->lm, (int64_t)c->vocab_size * h, &st, xavier_limit(h, c->vocab_size));
    *out = m;
    return OK;
}

void so_model_free(so_model* m) {
    if (m == NULL) return;
    free(m->w);
    free(m->lay);
    free(m);
}

const float* so_model_weights(const so_model* m, int64_t* count) {
    *count = m->n;
    return m->w;
}
void so_model_get_config(const so_model* m, so_config* out) { *out = m->cfg; }

uint64_t so_model_checksum(const so_model* m) { /* model.cpp:223-233, FNV-1a */
    uint64_t hash = 14695981039346656037ULL;
    const unsigned char* b = (const unsigned char*)m->w;
    for (int64_t i = 0; i < m->n * (int64_t)sizeof(float); ++i) {
        hash ^= b[i];
        hash *= 1099511628211ULL;
    }
    return hash;
}

/* model.cpp:143-221: SDCK v1 = "SDCK", u32 1, i32 dims[5], u64 seed, fp32 tensors */
int so_model_save(const so_model* m, const char* path) {
    FILE* f = fopen(path, "wb");
    CHECK(f != NULL, E_IO, "cannot open checkpoint for writing: %s", path);
    uint32_t ver = 1;
    int32_t dims[5] = {m->cfg.num_layers, m->cfg.num_heads, m->cfg.head_dim, m->cfg.vocab_size,
                       m->cfg.max_positions};
    int ok = fwrite("SDCK", 1, 4, f) == 4 && fwrite(&ver, 4, 1, f) == 1 &&
             fwrite(dims, 4, 5, f) == 5 && fwrite(&m->cfg.init_seed, 8, 1, f) == 1 &&
             fwrite(m->w, sizeof(float), (size_t)m->n, f) == (size_t)m->n;
    ok = (fclose(f) == 0) && ok;
    CHECK(ok, E_IO, "checkpoint write failed: %s", path);
    return OK;
}

int so_model_load(const char* path, so_model** out) {
    FILE* f = fopen(path, "rb");
    CHECK(f != NULL, E_IO, "cannot open checkpoint: %s", path);
    char magic[4];
    uint32_t ver = 0;
    int32_t dims[5];
    so_config c;
    int rc = OK;
    if (fread(magic, 1, 4, f) != 4) rc = fail(E_IO, "checkpoint truncated while reading magic");
    else if (memcmp(magic, "SDCK", 4) != 0) rc = fail(E_IO, "not a model checkpoint: %s", path);
    else if (fread(&ver, 4, 1, f) != 1) rc = fail(E_IO, "checkpoint truncated while reading version");
    else if (ver != 1) rc = fail(E_IO, "unsupported checkpoint version %u", ver);
    else if (fread(dims, 4, 5, f) != 5) rc = fail(E_IO, "checkpoint truncated while reading dimensions");
    else if (fread(&c.init_seed, 8, 1, f) != 1) rc = fail(E_IO, "checkpoint truncated while reading seed");
    if (rc != OK) {
        fclose(f);
        return rc;
    }
    c.num_layers = dims[0];
    c.num_heads = dims[1];
    c.head_dim = dims[2];
    c.vocab_size = dims[3];
    c.max_positions = dims[4];
    so_model* m;
    rc = model_alloc(&c, &m);
    if (rc != OK) {
        fclose(f);
        return rc;
    }
    if (fread(m->w, sizeof(float), (size_t)m->n, f) != (size_t)m->n) {
        rc = fail(E_IO, "checkpoint truncated while reading weights");
    } else {
        char extra;
        if (fread(&extra, 1, 1, f) != 0) rc = fail(E_IO, "checkpoint has trailing bytes: %s", path);
    }
    fclose(f);
    if (rc != OK) {
        so_model_free(m);
        return rc;
    }
    *out = m;
    return OK;
}

/* ------------------------------------------------------ ragged.cpp:19-36 */
int so_restore_indices(const int32_t* counts, int batch, int flat, int32_t* sample, int32_t* pos) {
    CHECK(flat >= 0, E_CONTRACT, "flat index must be nonnegative");
    int s = 0, p = flat;
    for (int i = 0; i < batch; ++i) {
        if (p >= counts[i]) {
            s += 1;
            p -= counts[i];
        } else {
            break;
        }
    }
    CHECK(s < batch, E_CONTRACT, "flat index %d outside batch", flat);
    *sample = s;
    *pos = p;
    return OK;
}

/* ------------------------------------------------- kv_cache.cpp:96-314 */
struct so_cache {
    int layout, L, B, cap, kv;
    float* keys;   /* [L][B*cap][kv] */
    float* values;
    uint8_t* pad;  /* [B*cap], padded layout only */
    int32_t* committed; /* committed_ (unpad) / committed_rows_ (padded) */
    int32_t* logical;   /* padded only */
    int32_t* staged;    /* written_ (unpad) / staged_ (padded) */
    int64_t useful, padding;
};

int so_cache_new(int layout, int L, int B, int cap, int kv, so_cache** out) {
    CHECK(L >= 1 && B >= 1 && cap >= 1 && kv >= 1, E_CONFIG, "cache dimensions must be positive");
    so_cache* c = (so_cache*)calloc(1, sizeof *c);
    c->layout = layout;
    c->L = L;
    c->B = B;
    c->cap = cap;
    c->kv = kv;
    size_t per = (size_t)B * cap * kv * L;
    c->keys = (float*)calloc(per, sizeof(float));
    c->values = (float*)calloc(per, sizeof(float));
    c->pad = (uint8_t*)calloc((size_t)B * cap, 1);
    c->committed = (int32_t*)calloc((size_t)B, 4);
    c->logical = (int32_t*)calloc((size_t)B, 4);
    c->staged = (int32_t*)calloc((size_t)B, 4);
    if (c->keys == NULL || c->values == NULL) {
        so_cache_free(c);
        return fail(E_ERROR, "out of host memory for the cache");
    }
    *out = c;
    return OK;
}

void so_cache_free(so_cache* c) {
    if (c == NULL) return;
    free(c->keys);
    free(c->values);
    free(c->pad);
    free(c->committed);
    free(c->logical);
    free(c->staged);
    free(c);
}

static int check_sample(const so_cache* c, int s) {
    CHECK(s >= 0 && s < c->B, E_CONTRACT, "cache sample out of range");
    return OK;
}
static int check_slot(const so_cache* c, int s, int pos, int layer) { /* kv_cache.cpp:93-103 */
    CHECK(s >= 0 && s < c->B, E_CONTRACT, "cache sample out of range");
    CHECK(layer >= 0 && layer < c->L, E_CONTRACT, "cache layer out of range");
    CHECK(pos >= 0, E_CONTRACT, "cache position negative");
    CHECK(pos < c->cap, E_CAPACITY, "cache position %d exceeds capacity %d", pos, c->cap);
    return OK;
}
static float* row_ptr(float* store, const so_cache* c, int s, int row, int layer) {
    return store + ((size_t)layer * c->B * c->cap + (size_t)s * c->cap + (size_t)row) * c->kv;
}

int so_cache_committed(const so_cache* c, int s, int32_t* out) {
    TRY(check_sample(c, s));
    *out = c->committed[s];
    return OK;
}
int so_cache_logical(const so_cache* c, int s, int32_t* out) {
    TRY(check_sample(c, s));
    *out = c->layout == 0 ? c->committed[s] : c->logical[s];
    return OK;
}
int so_cache_start_offset(const so_cache* c, int s, int32_t* out) { /* kv_cache.cpp:116-120 */
    CHECK(c->layout == 0, E_CONTRACT, "not an unpad arena");
    TRY(check_sample(c, s));
    *out = s * c->cap;
    return OK;
}

int so_cache_write_kv(so_cache* c, int s, int pos, int layer, const float* k, const float* v) {
    /* kv_cache.cpp:128-138 (unpad), 203-213 (padded) */
    TRY(check_slot(c, s, pos, layer));
    memcpy(row_ptr(c->keys, c, s, pos, layer), k, sizeof(float) * (size_t)c->kv);
    memcpy(row_ptr(c->values, c, s, pos, layer), v, sizeof(float) * (size_t)c->kv);
    if (layer == 0) {
        if (c->layout == 1) c->pad[(size_t)s * c->cap + pos] = 0;
        if (c->staged[s] < pos + 1) c->staged[s] = pos + 1;
        c->useful += 1;
    }
    return OK;
}

int so_cache_mark_hole(so_cache* c, int s, int pos) { /* kv_cache.cpp:90-92, 215-219 */
    CHECK(c->layout == 1, E_CONTRACT, "this cache layout has no masked holes");
    TRY(check_slot(c, s, pos, 0));
    c->pad[(size_t)s * c->cap + pos] = 1;
    if (c->staged[s] < pos + 1) c->staged[s] = pos + 1;
    return OK;
}

int so_cache_gather(const so_cache* c, int s, int upto, int layer, float* k, float* v,
                    int32_t* count) { /* kv_cache.cpp:140-150, 221-235 */
    TRY(check_slot(c, s, upto, layer));
    size_t kv = (size_t)c->kv;
    if (c->layout == 0) {
        CHECK(upto < c->staged[s], E_CONTRACT, "read past the written extent");
        memcpy(k, row_ptr(c->keys, c, s, 0, layer), sizeof(float) * kv * (size_t)(upto + 1));
        memcpy(v, row_ptr(c->values, c, s, 0, layer), sizeof(float) * kv * (size_t)(upto + 1));
        *count = upto + 1;
        return OK;
    }
    int n = 0;
    for (int row = 0; row <= upto; ++row) {
        if (c->pad[(size_t)s * c->cap + row]) continue;
        memcpy(k + (size_t)n * kv, row_ptr(c->keys, c, s, row, layer), sizeof(float) * kv);
        memcpy(v + (size_t)n * kv, row_ptr(c->values, c, s, row, layer), sizeof(float) * kv);
        ++n;
    }
    *count = n;
    return OK;
}

int so_cache_commit(so_cache* c, int s, int tau) { /* kv_cache.cpp:152-161 */
    CHECK(c->layout == 0, E_CONTRACT, "not an unpad arena");
    TRY(check_sample(c, s));
    CHECK(tau >= 1, E_CONTRACT, "commit needs tau >= 1");
    CHECK(tau <= c->staged[s] - c->committed[s], E_CONTRACT,
          "commit exceeds the slots written this step");
    c->committed[s] += tau;
    c->staged[s] = c->committed[s];
    return OK;
}

int so_cache_commit_prefill(so_cache* c, const int32_t* samples, const int32_t* lens, int n) {
    /* kv_cache.cpp:237-267 */
    CHECK(c->layout == 1, E_CONTRACT, "not a padded grid");
    CHECK(n >= 1, E_CONTRACT, "prefill commit needs matching sample and length lists");
    int rows = -1;
    for (int i = 0; i < n; ++i) {
        int s = samples[i], len = lens[i];
        CHECK(s >= 0 && s < c->B, E_CONTRACT, "cache sample out of range");
        CHECK(len >= 1, E_CONTRACT, "prompt length must be >= 1");
        CHECK(c->committed[s] == 0, E_CONTRACT, "prefill commit on a non-empty sample");
        if (rows < 0) rows = c->staged[s];
        CHECK(c->staged[s] == rows, E_CONTRACT, "prefill commit requires equally staged samples");
        CHECK(len <= rows, E_CONTRACT, "prompt length exceeds staged rows");
        for (int r = 0; r < rows - len; ++r)
            CHECK(c->pad[(size_t)s * c->cap + r], E_CONTRACT, "prefill left-pad row was not marked as a hole");
        for (int r = rows - len; r < rows; ++r)
            CHECK(!c->pad[(size_t)s * c->cap + r], E_CONTRACT, "prefill prompt row was never written");
    }
    for (int i = 0; i < n; ++i) {
        c->committed[samples[i]] = rows;
        c->logical[samples[i]] = lens[i];
    }
    return OK;
}

int so_cache_commit_padded(so_cache* c, const int32_t* samples, const int32_t* taus, int n) {
    /* kv_cache.cpp:269-314 */
    CHECK(c->layout == 1, E_CONTRACT, "not a padded grid");
    CHECK(n >= 1, E_CONTRACT, "padded commit needs matching sample and tau lists");
    int tau_max = 0;
    for (int i = 0; i < n; ++i) {
        CHECK(taus[i] >= 1, E_CONTRACT, "commit needs tau >= 1");
        if (taus[i] > tau_max) tau_max = taus[i];
    }
    int base = -1;
    for (int i = 0; i < n; ++i) {
        int s = samples[i];
        CHECK(s >= 0 && s < c->B, E_CONTRACT, "cache sample out of range");
        if (base < 0) base = c->committed[s];
        CHECK(c->committed[s] == base, E_CONTRACT, "padded commit requires aligned samples");
        CHECK(base + tau_max <= c->cap, E_CAPACITY, "padded commit exceeds cache capacity");
        CHECK(taus[i] <= c->staged[s] - base, E_CONTRACT, "commit exceeds the slots written this step");
        for (int r = base; r < base + taus[i]; ++r)
            CHECK(!c->pad[(size_t)s * c->cap + r], E_CONTRACT, "accepted row was never written");
    }
    for (int i = 0; i < n; ++i) {
        int s = samples[i];
        for (int r = base + taus[i]; r < base + tau_max; ++r) {
            for (int l = 0; l < c->L; ++l) {
                memset(row_ptr(c->keys, c, s, r, l), 0, sizeof(float) * (size_t)c->kv);
                memset(row_ptr(c->values, c, s, r, l), 0, sizeof(float) * (size_t)c->kv);
            }
            c->pad[(size_t)s * c->cap + r] = 1;
            c->padding += 1;
        }
        c->committed[s] += tau_max;
        c->logical[s] += taus[i];
        c->staged[s] = c->committed[s];
    }
    return OK;
}

int64_t so_ledger_useful(const so_cache* c) { return c->useful; }
int64_t so_ledger_padding(const so_cache* c) { return c->padding; }

/* ----------------------------------------------------- model.cpp:47-74 */
static void linear(const float* w, const float* b, int out_dim, int in_dim, const float* x,
                   float* y) {
    for (int o = 0; o < out_dim; ++o) {
        float acc = b != NULL ? b[o] : 0.0f;
        const float* row = w + (size_t)o * in_dim;
        for (int i = 0; i < in_dim; ++i) acc += row[i] * x[i];
        y[o] = acc;
    }
}
static void layer_norm(const float* x, const float* g, const float* b, int dim, float* y) {
    float mean = 0.0f;
    for (int i = 0; i < dim; ++i) mean += x[i];
    mean /= (float)dim;
    float var = 0.0f;
    for (int i = 0; i < dim; ++i) {
        float d = x[i] - mean;
        var += d * d;
    }
    var /= (float)dim;
    float inv = 1.0f / sqrtf(var + 1e-5f);
    for (int i = 0; i < dim; ++i) y[i] = (x[i] - mean) * inv * g[i] + b[i];
}
static float gelu(float x) {
    const float c = 0.7978845608028654f;
    return 0.5f * x * (1.0f + tanhf(c * (x + 0.044715f * x * x * x)));
}

int32_t so_greedy_next(const float* row, int vocab) { /* model.cpp:34-41 */
    int best = 0;
    for (int i = 1; i < vocab; ++i)
        if (row[i] > row[best]) best = i;
    return best;
}

/* model.cpp:256-373 */
int so_forward_planned(const so_model* m, so_cache* c, const int32_t* tokens, int n,
                       const int32_t* sample, const int32_t* logical, const int32_t* slot,
                       const int32_t* store, float* logits, int32_t* argmax) {
    const so_config* cfg = &m->cfg;
    CHECK(n > 0, E_CONTRACT, "forward pass over zero tokens");
    CHECK(c->kv == m->h, E_CONTRACT, "cache width does not match the model");
    CHECK(c->L == cfg->num_layers, E_CONTRACT, "cache depth does not match the model");
    int h = m->h, mm = m->m, heads = cfg->num_heads, hd = cfg->head_dim, V = cfg->vocab_size;
    float scale = 1.0f / sqrtf((float)hd);
    for (int t = 0; t < n; ++t) {
        CHECK(tokens[t] >= 0 && tokens[t] < V, E_CONTRACT, "token id out of vocabulary");
        CHECK(sample[t] >= 0 && sample[t] < c->B, E_CONTRACT, "plan sample out of range");
        CHECK(logical[t] >= 0, E_CONTRACT, "negative position");
        CHECK(logical[t] < cfg->max_positions, E_CAPACITY, "position %d exceeds max_positions %d",
              logical[t], cfg->max_positions);
        if (!store[t]) TRY(so_cache_mark_hole(c, sample[t], slot[t]));
    }
    const float* W = m->w;
    float* hs = (float*)malloc(sizeof(float) * (size_t)n * h);
    float* q_all = (float*)malloc(sizeof(float) * (size_t)n * h);
    float* scratch = (float*)malloc(sizeof(float) * (size_t)(6 * h + mm));
    float* xbuf = scratch, *kvec = scratch + h, *vvec = scratch + 2 * h, *ctx = scratch + 3 * h;
    float* attn = scratch + 4 * h, *mlp_in = scratch + 5 * h, *fc = scratch + 6 * h;
    float* kbuf = (float*)malloc(sizeof(float) * (size_t)c->cap * h);
    float* vbuf = (float*)malloc(sizeof(float) * (size_t)c->cap * h);
    float* scores = (float*)malloc(sizeof(float) * (size_t)c->cap);
    float* lrow = (float*)malloc(sizeof(float) * (size_t)V);
    int rc = OK;
    for (int t = 0; t < n; ++t) {
        const float* e = W + m->tok + (size_t)tokens[t] * h;
        const float* p = W + m->pos + (size_t)logical[t] * h;
        for (int i = 0; i < h; ++i) hs[(size_t)t * h + i] = e[i] + p[i];
    }
    for (int l = 0; l < cfg->num_layers && rc == OK; ++l) {
        const layer_off* o = &m->lay[l];
        for (int t = 0; t < n && rc == OK; ++t) { /* phase 1: model.cpp:307-318 */
            layer_norm(hs + (size_t)t * h, W + o->ln1_g, W + o->ln1_b, h, xbuf);
            linear(W + o->wq, W + o->bq, h, h, xbuf, q_all + (size_t)t * h);
            linear(W + o->wk, W + o->bk, h, h, xbuf, kvec);
            linear(W + o->wv, W + o->bv, h, h, xbuf, vvec);
            if (store[t]) rc = so_cache_write_kv(c, sample[t], slot[t], l, kvec, vvec);
        }
        for (int t = 0; t < n && rc == OK; ++t) { /* phase 2: model.cpp:320-358 */
            int32_t count = 0;
            rc = so_cache_gather(c, sample[t], slot[t], l, kbuf, vbuf, &count);
            if (rc != OK) break;
            if (count < 1) {
                rc = fail(E_CONTRACT, "token with an empty visible set");
                break;
            }
            const float* q = q_all + (size_t)t * h;
            for (int hh = 0; hh < heads; ++hh) {
                const float* qh = q + hh * hd;
                for (int j = 0; j < count; ++j) {
                    const float* kh = kbuf + (size_t)j * h + hh * hd;
                    float acc = 0.0f;
                    for (int d = 0; d < hd; ++d) acc += qh[d] * kh[d];
                    scores[j] = acc * scale;
                }
                float mx = scores[0];
                for (int j = 1; j < count; ++j) mx = (mx < scores[j]) ? scores[j] : mx;
                float denom = 0.0f;
                for (int j = 0; j < count; ++j) {
                    scores[j] = expf(scores[j] - mx);
                    denom += scores[j];
                }
                float* ch = ctx + hh * hd;
                for (int d = 0; d < hd; ++d) ch[d] = 0.0f;
                for (int j = 0; j < count; ++j) {
                    float wgt = scores[j] / denom;
                    const float* vh = vbuf + (size_t)j * h + hh * hd;
                    for (int d = 0; d < hd; ++d) ch[d] += wgt * vh[d];
                }
            }
            linear(W + o->wo, W + o->bo, h, h, ctx, attn);
            float* row = hs + (size_t)t * h;
            for (int i = 0; i < h; ++i) row[i] += attn[i];
            layer_norm(row, W + o->ln2_g, W + o->ln2_b, h, mlp_in);
            linear(W + o->w_fc, W + o->b_fc, mm, h, mlp_in, fc);
            for (int i = 0; i < mm; ++i) fc[i] = gelu(fc[i]);
            linear(W + o->w_proj, W + o->b_proj, h, mm, fc, xbuf);
            for (int i = 0; i < h; ++i) row[i] += xbuf[i];
        }
    }
    for (int t = 0; t < n && rc == OK; ++t) { /* model.cpp:361-371 */
        layer_norm(hs + (size_t)t * h, W + m->lnf_g, W + m->lnf_b, h, xbuf);
        float* out = logits != NULL ? logits + (size_t)t * V : lrow;
        linear(W + m->lm, NULL, V, h, xbuf, out);
        for (int i = 0; i < V; ++i) {
            if (!isfinite(out[i])) {
                rc = fail(E_ERROR, "non-finite logit produced");
                break;
            }
        }
        if (argmax != NULL) argmax[t] = so_greedy_next(out, V);
    }
    free(hs);
    free(q_all);
    free(scratch);
    free(kbuf);
    free(vbuf);
    free(scores);
    free(lrow);
    return rc;
}

/* model.cpp:235-254 */
int so_forward(const so_model* m, so_cache* c, const int32_t* tokens, const int32_t* counts,
               int batch, const int32_t* slot_sample, const int32_t* slot_pos, float* logits,
               int32_t* argmax) {
    CHECK(batch >= 1, E_CONTRACT, "batch must have at least one sample");
    CHECK(batch <= c->B, E_CONTRACT, "batch has more samples than the cache");
    int n = 0;
    for (int s = 0; s < batch; ++s) n += counts[s];
    int32_t* buf = (int32_t*)malloc(sizeof(int32_t) * (size_t)(4 * n + 1));
    int32_t *ps = buf, *pl = buf + n, *pw = buf + 2 * n, *st = buf + 3 * n;
    int rc = OK;
    for (int i = 0; i < n && rc == OK; ++i) {
        int32_t s, p;
        rc = so_restore_indices(counts, batch, i, &s, &p);
        if (rc != OK) break;
        int expected = c->committed[s] + p;
        if (slot_sample[i] != s || slot_pos[i] != expected) {
            rc = fail(E_CONTRACT, "slot %d does not continue its sample", i);
            break;
        }
        ps[i] = s;
        pl[i] = expected;
        pw[i] = expected;
        st[i] = 1;
    }
    if (rc == OK) rc = so_forward_planned(m, c, tokens, n, ps, pl, pw, st, logits, argmax);
    free(buf);
    return rc;
}

/* engine.cpp:60-76 */
int so_verify(const float* rows, int nrows, int vocab, const int32_t* drafts, int k,
              int32_t* accepted, int32_t* tau) {
    CHECK(nrows == k + 1, E_CONTRACT,
          "verification needs one logits row per draft plus the bonus row");
    for (int j = 0; j <= k; ++j) {
        int32_t picked = so_greedy_next(rows + (size_t)j * vocab, vocab);
        accepted[j] = picked;
        if (j == k) {
            *tau = k + 1;
        } else if (picked != drafts[j]) {
            *tau = j + 1;
            break;
        }
    }
    return OK;
}

/* ------------------------------------------------------ predictors.cpp */
int so_retrieval_predict(const int32_t* ctx, int len, int match_len, int copy_len, int32_t* out,
                         int32_t* nout) { /* predictors.cpp:39-59 */
    CHECK(match_len >= 1, E_CONTRACT, "match length must be >= 1");
    CHECK(copy_len >= 1, E_CONTRACT, "copy length must be >= 1");
    *nout = 0;
    int suffix = len - match_len;
    if (suffix <= 0) return OK;
    for (int start = suffix - 1; start >= 0; --start) {
        int match = 1;
        for (int i = 0; i < match_len; ++i) {
            if (ctx[start + i] != ctx[suffix + i]) {
                match = 0;
                break;
            }
        }
        if (!match) continue;
        int from = start + match_len;
        int take = copy_len < len - from ? copy_len : len - from;
        for (int i = 0; i < take; ++i) out[i] = ctx[from + i];
        *nout = take;
        return OK;
    }
    return OK;
}

int so_draft_predict(const so_model* d, const int32_t* ctx, int len, int k, int32_t* out) {
    /* predictors.cpp:9-37 */
    CHECK(k >= 1, E_CONTRACT, "draft length must be >= 1");
    CHECK(len >= 1, E_CONTRACT, "draft prediction needs a context");
    CHECK(len + k <= d->cfg.max_positions, E_CAPACITY, "context plus draft length exceeds max_positions");
    so_cache* c;
    TRY(so_cache_new(0, d->cfg.num_layers, 1, d->cfg.max_positions, d->h, &c));
    int32_t* am = (int32_t*)malloc(sizeof(int32_t) * (size_t)len);
    int32_t* pos = (int32_t*)malloc(sizeof(int32_t) * (size_t)len);
    int32_t* zeros = (int32_t*)calloc((size_t)len, sizeof(int32_t));
    for (int i = 0; i < len; ++i) pos[i] = i;
    int32_t cnt = len;
    int rc = so_forward(d, c, ctx, &cnt, 1, zeros, pos, NULL, am);
    if (rc == OK) rc = so_cache_commit(c, 0, len);
    if (rc == OK) {
        int32_t next = am[len - 1];
        out[0] = next;
        for (int i = 1; i < k && rc == OK; ++i) {
            int32_t one = 1, p = c->committed[0], z = 0, a = 0;
            rc = so_forward(d, c, &next, &one, 1, &z, &p, NULL, &a);
            if (rc == OK) rc = so_cache_commit(c, 0, 1);
            next = a;
            out[i] = next;
        }
    }
    free(am);
    free(pos);
    free(zeros);
    so_cache_free(c);
    return rc;
}

/* --------------------------------------------------------- engine.cpp */
static int engine_validate(const so_engine_config* e) { /* engine.cpp:48-58 */
    if (e->predictor != 1) CHECK(e->k >= 1, E_CONFIG, "k must be >= 1");
    CHECK(e->match_len >= 1, E_CONFIG, "match_len must be >= 1");
    CHECK(e->copy_len >= 1, E_CONFIG, "copy_len must be >= 1");
    CHECK(e->batch_size >= 1, E_CONFIG, "batch_size must be >= 1");
    CHECK(e->max_new_tokens >= 0, E_CONFIG, "max_new_tokens must be >= 0");
    CHECK(e->synthetic_accuracy >= 0.0 && e->synthetic_accuracy < 1.0, E_CONFIG,
          "synthetic accuracy must lie in [0, 1)");
    return OK;
}

typedef struct {
    int32_t* tok; /* BOS + prompt + generated */
    int len, generated, finished;
} state_t;

static int predict(const so_engine_config* e, const state_t* st, const so_model* target,
                   const so_model* draft, int step, int s, int32_t* out, int32_t* nout) {
    /* engine.cpp:173-188 */
    if (e->predictor == 1) return so_retrieval_predict(st->tok, st->len, e->match_len, e->copy_len, out, nout);
    if (e->predictor == 0) {
        *nout = e->k;
        return so_draft_predict(draft, st->tok, st->len, e->k, out);
    }
    /* synthetic: predictors.cpp:61-72 */
    CHECK(e->synthetic_accuracy >= 0.0 && e->synthetic_accuracy < 1.0, E_CONFIG,
          "predictor accuracy must lie in [0, 1)");
    TRY(so_draft_predict(target, st->tok, st->len, e->k, out));
    uint64_t rs = so_mix_seed(e->seed, (uint64_t)step, (uint64_t)s);
    for (int i = 0; i < e->k; ++i)
        if (unit_double(&rs) >= e->synthetic_accuracy) out[i] = (out[i] + 1) % target->cfg.vocab_size;
    *nout = e->k;
    return OK;
}

static int decode_greedy(const so_engine_config* e, const so_model* target, state_t* st) {
    /* engine.cpp:206-289 */
    const so_config* tc = &target->cfg;
    for (int s = 0; s < e->batch_size; ++s)
        CHECK(st[s].len + e->max_new_tokens <= tc->max_positions, E_CAPACITY,
              "prompt plus generation budget exceeds max_positions");
    if (e->max_new_tokens == 0) return OK;
    float* rows = NULL;
    for (int s = 0; s < e->batch_size; ++s) {
        state_t* S = &st[s];
        so_cache* c;
        TRY(so_cache_new(0, tc->num_layers, 1, tc->max_positions, target->h, &c));
        int plen = S->len;
        int32_t* pos = (int32_t*)malloc(sizeof(int32_t) * (size_t)plen);
        int32_t* zer = (int32_t*)calloc((size_t)plen, sizeof(int32_t));
        int32_t* am = (int32_t*)malloc(sizeof(int32_t) * (size_t)plen);
        for (int i = 0; i < plen; ++i) pos[i] = i;
        int32_t cnt = plen;
        int rc = so_forward(target, c, S->tok, &cnt, 1, zer, pos, rows, am);
        if (rc == OK) rc = so_cache_commit(c, 0, plen);
        int32_t next = am[plen - 1];
        free(pos);
        free(zer);
        free(am);
        if (rc == OK) {
            S->tok[S->len++] = next;
            S->generated = 1;
            while (rc == OK && S->generated < e->max_new_tokens && !(e->stop_on_eos && next == 1)) {
                int32_t one = 1, p = c->committed[0], z = 0, a = 0;
                rc = so_forward(target, c, &next, &one, 1, &z, &p, NULL, &a);
                if (rc == OK) rc = so_cache_commit(c, 0, 1);
                next = a;
                S->tok[S->len++] = next;
                S->generated += 1;
            }
        }
        so_cache_free(c);
        if (rc != OK) return rc;
    }
    return OK;
}

int so_decode(const so_engine_config* e, const so_model* target, const so_model* draft,
              const int32_t* prompts, const int32_t* prompt_lens, int32_t* gen_tokens,
              int32_t* gen_counts, int32_t* rec, int64_t rec_cap, int64_t* n_rec,
              int64_t* ledger) {
    TRY(engine_validate(e));
    const so_config* tc = &target->cfg;
    int b = e->batch_size, V = tc->vocab_size;
    *n_rec = 0;
    ledger[0] = ledger[1] = 0;
    int reach = e->predictor == 1 ? e->copy_len : e->k;
    int maxlen = 0;
    state_t* st = (state_t*)calloc((size_t)b, sizeof(state_t));
    int at = 0;
    for (int s = 0; s < b; ++s) {
        st[s].tok = (int32_t*)malloc(sizeof(int32_t) * (size_t)(prompt_lens[s] + e->max_new_tokens + reach + 8));
        memcpy(st[s].tok, prompts + at, sizeof(int32_t) * (size_t)prompt_lens[s]);
        st[s].len = prompt_lens[s];
        at += prompt_lens[s];
        if (prompt_lens[s] > maxlen) maxlen = prompt_lens[s];
    }
    int rc = OK;
    so_cache* c = NULL;
    float* rows = NULL;
    int32_t *flat = NULL, *ps = NULL, *pl = NULL, *pw = NULL, *pst = NULL, *am = NULL;
    int32_t *drafts = NULL, *dcount = NULL, *first_row = NULL;
#define BAIL(x)                 \
    do {                        \
        rc = (x);               \
        if (rc != OK) goto done; \
    } while (0)
    if (e->mode == 0) {
        BAIL(decode_greedy(e, target, st));
        goto finish;
    }
    if (e->mode != 1 && e->mode != 2) BAIL(fail(E_CONFIG, "speculative decoding needs the vanilla or ems mode"));
    if (e->predictor == 0) {
        if (draft == NULL) BAIL(fail(E_CONFIG, "draft predictor needs a draft model"));
        if (draft->cfg.vocab_size != V) BAIL(fail(E_CONFIG, "draft and target vocabularies differ"));
    }
    for (int s = 0; s < b; ++s) { /* engine.cpp:157-171 */
        int need = st[s].len + e->max_new_tokens + reach;
        if (need > tc->max_positions)
            BAIL(fail(E_CAPACITY, "prompt plus generation budget needs %d positions but the model has %d",
                      need, tc->max_positions));
    }
    if (e->max_new_tokens == 0) goto finish;
    int aligned = e->mode == 1;
    BAIL(so_cache_new(aligned, tc->num_layers, b, tc->max_positions, target->h, &c));
    int kmax_cap = (e->predictor == 1 ? e->copy_len : e->k);
    int tmax = b * (maxlen > kmax_cap + 1 ? maxlen : kmax_cap + 1);
    flat = (int32_t*)malloc(sizeof(int32_t) * (size_t)tmax);
    ps = (int32_t*)malloc(sizeof(int32_t) * (size_t)tmax);
    pl = (int32_t*)malloc(sizeof(int32_t) * (size_t)tmax);
    pw = (int32_t*)malloc(sizeof(int32_t) * (size_t)tmax);
    pst = (int32_t*)malloc(sizeof(int32_t) * (size_t)tmax);
    am = (int32_t*)malloc(sizeof(int32_t) * (size_t)tmax);
    drafts = (int32_t*)malloc(sizeof(int32_t) * (size_t)b * (kmax_cap + 1));
    dcount = (int32_t*)calloc((size_t)b, sizeof(int32_t));
    first_row = (int32_t*)malloc(sizeof(int32_t) * (size_t)b);
    rows = (float*)malloc(sizeof(float) * (size_t)(kmax_cap + 1) * V);

    /* prefill: engine.cpp:330-385 */
    {
        int n = 0;
        if (aligned) {
            for (int s = 0; s < b; ++s) {
                int len = st[s].len, holes = maxlen - len;
                for (int r = 0; r < holes; ++r) BAIL(so_cache_mark_hole(c, s, r));
                for (int i = 0; i < len; ++i) {
                    flat[n] = st[s].tok[i];
                    ps[n] = s;
                    pl[n] = i;
                    pw[n] = holes + i;
                    pst[n] = 1;
                    ++n;
                }
                first_row[s] = n - 1;
            }
            BAIL(so_forward_planned(target, c, flat, n, ps, pl, pw, pst, NULL, am));
            int32_t* ids = (int32_t*)malloc(sizeof(int32_t) * (size_t)b);
            int32_t* lens = (int32_t*)malloc(sizeof(int32_t) * (size_t)b);
            for (int s = 0; s < b; ++s) {
                ids[s] = s;
                lens[s] = st[s].len;
            }
            rc = so_cache_commit_prefill(c, ids, lens, b);
            free(ids);
            free(lens);
            BAIL(rc);
        } else {
            int32_t* counts = (int32_t*)malloc(sizeof(int32_t) * (size_t)b);
            for (int s = 0; s < b; ++s) {
                counts[s] = st[s].len;
                for (int i = 0; i < st[s].len; ++i) {
                    flat[n] = st[s].tok[i];
                    ps[n] = s;
                    pl[n] = i;
                    ++n;
                }
                first_row[s] = n - 1;
            }
            rc = so_forward(target, c, flat, counts, b, ps, pl, NULL, am);
            free(counts);
            BAIL(rc);
            for (int s = 0; s < b; ++s) BAIL(so_cache_commit(c, s, st[s].len));
        }
        for (int s = 0; s < b; ++s) {
            int32_t first = am[first_row[s]];
            st[s].tok[st[s].len++] = first;
            st[s].generated = 1;
            st[s].finished = st[s].generated >= e->max_new_tokens || (e->stop_on_eos && first == 1);
        }
    }

    /* decode loop: engine.cpp:391-489 */
    for (int step = 0;; ++step) {
        int active = 0, kmax = 0;
        for (int s = 0; s < b; ++s) active += !st[s].finished;
        if (active == 0) break;
        for (int s = 0; s < b; ++s) {
            dcount[s] = 0;
            if (st[s].finished) continue;
            BAIL(predict(e, &st[s], target, draft, step, s, drafts + (size_t)s * (kmax_cap + 1), &dcount[s]));
            if (dcount[s] > kmax) kmax = dcount[s];
        }
        int n = 0;
        if (aligned) { /* engine.cpp:408-426 */
            int mrow = 1 + kmax, base = -1;
            for (int s = 0; s < b; ++s) {
                if (st[s].finished) continue;
                if (base < 0) base = c->committed[s];
                if (c->committed[s] != base) BAIL(fail(E_ERROR, "internal: aligned samples drifted apart"));
                first_row[s] = n;
                int ks = dcount[s], logical = c->logical[s];
                for (int o = 0; o < mrow; ++o) {
                    int real = o <= ks;
                    flat[n] = real ? (o == 0 ? st[s].tok[st[s].len - 1] : drafts[(size_t)s * (kmax_cap + 1) + o - 1]) : 2;
                    ps[n] = s;
                    pl[n] = logical + o;
                    pw[n] = base + o;
                    pst[n] = real;
                    ++n;
                }
            }
            BAIL(so_forward_planned(target, c, flat, n, ps, pl, pw, pst, NULL, am));
        } else { /* engine.cpp:427-444 */
            int32_t* counts = (int32_t*)calloc((size_t)b, sizeof(int32_t));
            for (int s = 0; s < b; ++s) {
                if (st[s].finished) continue;
                first_row[s] = n;
                counts[s] = 1 + dcount[s];
                int committed = c->committed[s];
                for (int o = 0; o <= dcount[s]; ++o) {
                    flat[n] = o == 0 ? st[s].tok[st[s].len - 1] : drafts[(size_t)s * (kmax_cap + 1) + o - 1];
                    ps[n] = s;
                    pl[n] = committed + o;
                    ++n;
                }
            }
            rc = so_forward(target, c, flat, counts, b, ps, pl, NULL, am);
            free(counts);
            BAIL(rc);
        }
        int32_t* samples = (int32_t*)malloc(sizeof(int32_t) * (size_t)active);
        int32_t* taus = (int32_t*)malloc(sizeof(int32_t) * (size_t)active);
        int na = 0;
        for (int s = 0; s < b; ++s) { /* engine.cpp:446-475 */
            if (st[s].finished) continue;
            int ks = dcount[s];
            const int32_t* d = drafts + (size_t)s * (kmax_cap + 1);
            int vt = ks + 1;
            int32_t acc[64];
            for (int j = 0; j <= ks; ++j) { /* verify() over the argmax of each row */
                acc[j] = am[first_row[s] + j];
                if (j < ks && acc[j] != d[j]) {
                    vt = j + 1;
                    break;
                }
            }
            int remaining = e->max_new_tokens - st[s].generated;
            int tau = vt < remaining ? vt : remaining;
            if (e->stop_on_eos) {
                for (int j = 0; j < tau; ++j) {
                    if (acc[j] == 1) {
                        tau = j + 1;
                        break;
                    }
                }
            }
            for (int j = 0; j < tau; ++j) st[s].tok[st[s].len++] = acc[j];
            st[s].generated += tau;
            st[s].finished = st[s].generated >= e->max_new_tokens ||
                             (e->stop_on_eos && st[s].tok[st[s].len - 1] == 1);
            if (*n_rec < rec_cap) {
                int32_t* r = rec + *n_rec * 6;
                r[0] = step;
                r[1] = s;
                r[2] = ks;
                r[3] = tau;
                r[4] = tau < vt;
                r[5] = 0;
            }
            *n_rec += 1;
            samples[na] = s;
            taus[na] = tau;
            ++na;
        }
        if (aligned) {
            rc = so_cache_commit_padded(c, samples, taus, na);
        } else {
            for (int i = 0; i < na && rc == OK; ++i) rc = so_cache_commit(c, samples[i], taus[i]);
        }
        free(samples);
        free(taus);
        BAIL(rc);
    }
    ledger[0] = c->useful;
    ledger[1] = c->padding;
finish:
    for (int s = 0; s < b; ++s) {
        gen_counts[s] = st[s].generated;
        memcpy(gen_tokens + (size_t)s * e->max_new_tokens, st[s].tok + st[s].len - st[s].generated,
               sizeof(int32_t) * (size_t)st[s].generated);
    }
done:
#undef BAIL
    for (int s = 0; s < b; ++s) free(st[s].tok);
    free(st);
    so_cache_free(c);
    free(rows);
    free(flat);
    free(ps);
    free(pl);
    free(pw);
    free(pst);
    free(am);
    free(drafts);
    free(dcount);
    free(first_row);
    return rc;
}
