/*
 * relay_oracle.c — the CPU ORACLE for the RelayGen (arXiv 2602.06454) hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2602_06454_b200/ + librelay.so) never links, imports or calls it, and
 * this file includes no header from include/ or paper_2602_06454_b200/csrc/.
 *
 * Plain, slow, obviously correct: every quantity is the paper's definition
 * written out in fp64 with plain loops.  No blocking, fusion or reordering.
 * Citations: "P:n" = /root/reference/PAPER.md line n (LaTeX source), "S:n" =
 * SPEC.md line n.  Readings of silent/ambiguous passages are listed in
 * DESIGN.md ("Readings of the paper", R1..R20) and referenced here as [Rk].
 *
 * Parity pins (tests/test_oracle_pins.py) fix each function to something other
 * than itself: worked examples (S:58-60, S:76-78, S:223-225, S:232-234,
 * S:241-242), closed forms (V=2: m = tanh(d/2)), invariances, a hand-traced
 * golden trace (tests/golden/trace_fixture.json) and brute force over tiny
 * inputs.  No function here is "parity unpinned".
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- decode */
/* Element j of a logit row, widened exactly to double.
 * dtype 0 = bf16 (the top 16 bits of an IEEE binary32), 1 = IEEE binary16,
 * 2 = IEEE binary32.  Both 16-bit formats widen exactly. */
static double decode_bf16(uint16_t h) {
    uint32_t bits = ((uint32_t)h) << 16;
    float f;
    memcpy(&f, &bits, sizeof f);
    return (double)f;
}

static double decode_f16(uint16_t h) {
    int sign = (h >> 15) & 1;
    int expo = (h >> 10) & 0x1f;
    int mant = h & 0x3ff;
    double v;
    if (expo == 0x1f) {
        v = mant ? NAN : INFINITY;
    } else if (expo == 0) {
        v = ldexp((double)mant, -24);                 /* subnormal: mant * 2^-24 */
    } else {
        v = ldexp((double)(mant | 0x400), expo - 25); /* 1.mant * 2^(e-15) */
    }
    return sign ? -v : v;
}

double oracle_elem(const void* row, int dtype, int64_t j) {
    if (dtype == 0) return decode_bf16(((const uint16_t*)row)[j]);
    if (dtype == 1) return decode_f16(((const uint16_t*)row)[j]);
    return (double)((const float*)row)[j];
}

/* ------------------------------------------------------------ row margin */
/* P:139-147 (§3.2): p_t = softmax(z_t), m_t = p_t,(1) - p_t,(2).
 * Readings: [R1] softmax at temperature 1 (inv_temperature = 1) unless the
 * caller scales z by iota; [R2] over the full vocabulary; [R3] top-1/top-2
 * indices order entries by (value desc, index asc) with IEEE equality, so
 * -0 == +0, and are taken on the UNSCALED values; [R4] a row holding NaN or
 * +inf -> status 1, an all -inf row -> status 2, both with indices -1 and
 * margin/lse NaN.  Returns the status, or -1 when vocab < 2 (invalid call). */
int oracle_margin_row(const void* row, int dtype, int64_t vocab, double inv_temperature,
                      int32_t* i1_out, int32_t* i2_out, double* margin_out, double* lse_out) {
    int64_t j;
    if (vocab < 2) return -1;
    for (j = 0; j < vocab; j++) {
        double z = oracle_elem(row, dtype, j);
        if (isnan(z) || (isinf(z) && z > 0)) {
            *i1_out = -1; *i2_out = -1; *margin_out = NAN; *lse_out = NAN;
            return 1;
        }
    }
    int any_finite = 0;
    for (j = 0; j < vocab; j++)
        if (!isinf(oracle_elem(row, dtype, j))) any_finite = 1;
    if (!any_finite) {
        *i1_out = -1; *i2_out = -1; *margin_out = NAN; *lse_out = NAN;
        return 2;
    }
    /* i1: walking indices upward, a strictly larger value replaces the holder,
     * so the lowest index among equal maxima is kept. */
    int64_t i1 = 0;
    for (j = 1; j < vocab; j++)
        if (oracle_elem(row, dtype, j) > oracle_elem(row, dtype, i1)) i1 = j;
    /* i2: the same rule over every index except i1. */
    int64_t i2 = (i1 == 0) ? 1 : 0;
    for (j = 0; j < vocab; j++) {
        if (j == i1) continue;
        if (oracle_elem(row, dtype, j) > oracle_elem(row, dtype, i2)) i2 = j;
    }
    /* p = softmax(z * iota): p_j = exp(z_j*iota - M) / S, M = z_(1)*iota. */
    double M = oracle_elem(row, dtype, i1) * inv_temperature;
    double S = 0.0;
    for (j = 0; j < vocab; j++) {
        double z = oracle_elem(row, dtype, j);
        if (isinf(z)) continue;                       /* exp(-inf) = 0 */
        S += exp(z * inv_temperature - M);
    }
    double z2 = oracle_elem(row, dtype, i2);
    double p1 = 1.0 / S;
    double p2 = isinf(z2) ? 0.0 : exp(z2 * inv_temperature - M) / S;
    *i1_out = (int32_t)i1;
    *i2_out = (int32_t)i2;
    *margin_out = p1 - p2;
    *lse_out = M + log(S);
    return 0;
}

/* Many rows, optionally on several host threads (row blocks; each row is the
 * single-row definition above, so the thread count changes nothing but time). */
typedef struct {
    const uint8_t* logits; int dtype; int64_t row0, row1, vocab, row_stride;
    double inv_temperature;
    double* margin; int32_t* top1; int32_t* top2; double* lse; int8_t* status;
} rows_job_t;

static void* rows_worker(void* arg) {
    rows_job_t* jb = (rows_job_t*)arg;
    size_t esz = (jb->dtype == 2) ? 4 : 2;
    for (int64_t r = jb->row0; r < jb->row1; r++) {
        const void* row = jb->logits + (size_t)r * (size_t)jb->row_stride * esz;
        int32_t a, b; double m, l;
        int st = oracle_margin_row(row, jb->dtype, jb->vocab, jb->inv_temperature, &a, &b, &m, &l);
        jb->margin[r] = m; jb->top1[r] = a; jb->top2[r] = b; jb->lse[r] = l;
        jb->status[r] = (int8_t)st;
    }
    return NULL;
}

int oracle_margin_rows(const void* logits, int dtype, int64_t n_rows, int64_t vocab,
                       int64_t row_stride, double inv_temperature, int n_threads,
                       double* margin, int32_t* top1, int32_t* top2, double* lse, int8_t* status) {
    if (vocab < 2 || row_stride < vocab || n_rows < 0) return -1;
    if (n_threads < 1) n_threads = 1;
    if (n_threads > 256) n_threads = 256;
    pthread_t th[256];
    rows_job_t jobs[256];
    int64_t per = (n_rows + n_threads - 1) / n_threads;
    int started = 0;
    for (int t = 0; t < n_threads; t++) {
        int64_t a = (int64_t)t * per, b = a + per;
        if (a > n_rows) a = n_rows;
        if (b > n_rows) b = n_rows;
        jobs[t] = (rows_job_t){(const uint8_t*)logits, dtype, a, b, vocab, row_stride,
                               inv_temperature, margin, top1, top2, lse, status};
        if (n_threads == 1) { rows_worker(&jobs[t]); continue; }
        pthread_create(&th[t], NULL, rows_worker, &jobs[t]);
        started++;
    }
    for (int t = 0; t < started; t++) pthread_join(th[t], NULL);
    return 0;
}

/* --------------------------------------------------------------- cue scan */
/* Which trajectory holds position t: the k with offsets[k] <= t < offsets[k+1]
 * (plain linear walk).  traj_offsets == NULL means one trajectory [0, n_tok). */
static int64_t traj_of(const int64_t* off, int32_t n_traj, int64_t n_tok, int64_t t,
                       int64_t* a_out, int64_t* b_out) {
    if (!off) { *a_out = 0; *b_out = n_tok; return 0; }
    for (int32_t k = 0; k < n_traj; k++)
        if (off[k] <= t && t < off[k + 1]) { *a_out = off[k]; *b_out = off[k + 1]; return k; }
    *a_out = *b_out = -1;
    return -1;
}

/* Token classes (N4, text-faithful cues): a pattern element e >= 0 is the
 * token id e; e < 0 is class c = -1 - e, matched by any token v with
 * classes[c * vocab + v] != 0 (e.g. "So " = "So" followed by any
 * space-initial token, Table 6) [R18]. */
static int elem_matches(int32_t tok, int32_t e, const uint8_t* classes, int32_t n_classes,
                        int64_t vocab) {
    if (e >= 0) return tok == e;
    int32_t c = -1 - e;
    if (!classes || c >= n_classes || tok < 0 || tok >= vocab) return 0;
    return classes[(int64_t)c * vocab + tok] != 0;
}

static int in_class(int32_t tok, int32_t c, const uint8_t* classes, int64_t vocab) {
    return tok >= 0 && tok < vocab && classes[(int64_t)c * vocab + tok] != 0;
}

static int pattern_matches_at(const int32_t* tokens, int64_t s, int64_t b,
                              const int32_t* pat_tokens, const int32_t* pat_offsets, int32_t p,
                              const uint8_t* classes, int32_t n_classes, int64_t vocab) {
    int64_t len = pat_offsets[p + 1] - pat_offsets[p];
    if (s + len > b) return 0;                       /* must fit inside the trajectory */
    for (int64_t k = 0; k < len; k++)
        if (!elem_matches(tokens[s + k], pat_tokens[pat_offsets[p] + k], classes, n_classes, vocab))
            return 0;
    return 1;
}

/* Cue occurrences by "simple token matching".
 * Readings: [R5] cues are caller-tokenised token-ID patterns; [R6] the cue
 * position is the pattern's first token; [R7] LONGEST mode (0): at each start
 * s, the longest pattern that matches tokens[s..s+len) inside s's trajectory
 * (equal lengths: the lowest pattern index, [R18]); ALL mode (1): for each cue
 * id (ascending) with any matching pattern at s, one occurrence carrying that
 * cue's longest matching pattern.  Starts ascend.
 * Also term[t] = terminator[tokens[t]] ("sentence-ending punctuation",
 * [R8] the caller's terminator set), except, with decimal_rule = {period,
 * digit_end, digit_start} class ids (NULL = off), a period token between a
 * digit-ending token and a digit-starting token of the same trajectory is not
 * a sentence end ("not inside a decimal number") [R19].  Returns
 * the TRUE occurrence count; at most `cap` are written. */
int64_t oracle_cue_scan_ex(const int32_t* tokens, int64_t n_tok, const int64_t* traj_offsets,
                           int32_t n_traj, const int32_t* pat_tokens, const int32_t* pat_offsets,
                           int32_t n_pat, const int32_t* pat_cue, int32_t n_cues,
                           const uint8_t* terminator, uint32_t mode,
                           const uint8_t* classes, int32_t n_classes, int64_t vocab,
                           const int32_t* decimal_rule,
                           uint8_t* term, int32_t* occ_pos, int32_t* occ_pat, int64_t cap) {
    int64_t n = 0;
    for (int64_t t = 0; t < n_tok; t++) {
        term[t] = terminator[tokens[t]] ? 1 : 0;
        if (term[t] && decimal_rule && classes) {
            int64_t a, b;
            traj_of(traj_offsets, n_traj, n_tok, t, &a, &b);
            if (t - 1 >= a && t + 1 < b && in_class(tokens[t], decimal_rule[0], classes, vocab) &&
                in_class(tokens[t - 1], decimal_rule[1], classes, vocab) &&
                in_class(tokens[t + 1], decimal_rule[2], classes, vocab))
                term[t] = 0;
        }
    }
    for (int64_t s = 0; s < n_tok; s++) {
        int64_t a, b;
        if (traj_of(traj_offsets, n_traj, n_tok, s, &a, &b) < 0) continue;
        if (mode == 0) {
            int32_t best = -1;
            for (int32_t p = 0; p < n_pat; p++) {
                if (!pattern_matches_at(tokens, s, b, pat_tokens, pat_offsets, p, classes, n_classes,
                                        vocab))
                    continue;
                if (best < 0 || (pat_offsets[p + 1] - pat_offsets[p]) >
                                (pat_offsets[best + 1] - pat_offsets[best])) best = p;
            }
            if (best >= 0) {
                if (n < cap) { occ_pos[n] = (int32_t)s; occ_pat[n] = best; }
                n++;
            }
        } else {
            for (int32_t c = 0; c < n_cues; c++) {
                int32_t best = -1;
                for (int32_t p = 0; p < n_pat; p++) {
                    if (pat_cue[p] != c) continue;
                    if (!pattern_matches_at(tokens, s, b, pat_tokens, pat_offsets, p, classes,
                                            n_classes, vocab))
                        continue;
                    if (best < 0 || (pat_offsets[p + 1] - pat_offsets[p]) >
                                    (pat_offsets[best + 1] - pat_offsets[best])) best = p;
                }
                if (best >= 0) {
                    if (n < cap) { occ_pos[n] = (int32_t)s; occ_pat[n] = best; }
                    n++;
                }
            }
        }
    }
    return n;
}

int64_t oracle_cue_scan(const int32_t* tokens, int64_t n_tok, const int64_t* traj_offsets,
                        int32_t n_traj, const int32_t* pat_tokens, const int32_t* pat_offsets,
                        int32_t n_pat, const int32_t* pat_cue, int32_t n_cues,
                        const uint8_t* terminator, uint32_t mode,
                        uint8_t* term, int32_t* occ_pos, int32_t* occ_pat, int64_t cap) {
    return oracle_cue_scan_ex(tokens, n_tok, traj_offsets, n_traj, pat_tokens, pat_offsets, n_pat,
                              pat_cue, n_cues, terminator, mode, NULL, 0, 0, NULL, term, occ_pos,
                              occ_pat, cap);
}

/* ------------------------------------------------- post-sentence windows */
/* "the average probability margin over the remainder of the sentence in which
 * the cue appears", "from the cue position to the next sentence
 * boundary", "from that token until the end of the sentence".
 * Readings: [R9] window [s, e] inclusive of the cue token and of the boundary
 * token; e = the first t >= s in s's trajectory with term[t]; [R10]
 * with no terminator, e = the trajectory's last token; [R11] the
 * low-margin fraction counts m_t < tau (strict).  A window holding a NaN
 * margin gets mean = min = lowfrac = NaN and invalid = 1. */
void oracle_windows(const float* margin, const uint8_t* term, int64_t n_tok,
                    const int64_t* traj_offsets, int32_t n_traj,
                    const int32_t* occ_pos, int64_t n_occ, float tau,
                    int32_t* seg_end, double* seg_mean, double* seg_min, double* seg_lowfrac,
                    double* seg_sum, int32_t* seg_low, int8_t* seg_invalid) {
    for (int64_t i = 0; i < n_occ; i++) {
        int64_t s = occ_pos[i], a, b;
        traj_of(traj_offsets, n_traj, n_tok, s, &a, &b);
        int64_t e = s;
        while (e < b - 1 && !term[e]) e++;
        double sum = 0.0, mn = INFINITY;
        int32_t low = 0, bad = 0;
        for (int64_t t = s; t <= e; t++) {
            double m = (double)margin[t];
            if (isnan(m)) { bad = 1; continue; }
            sum += m;
            if (m < mn) mn = m;
            if (margin[t] < tau) low++;
        }
        double len = (double)(e - s + 1);
        seg_end[i] = (int32_t)e;
        seg_sum[i] = bad ? NAN : sum;
        seg_low[i] = low;
        seg_invalid[i] = (int8_t)bad;
        seg_mean[i] = bad ? NAN : sum / len;
        seg_min[i] = bad ? NAN : mn;
        seg_lowfrac[i] = bad ? NAN : (double)low / len;
    }
}

/* ------------------------------------------------ statistics + selection */
/* One summary per cue and one global summary (defined here independently of
 * include/relay.h; the test compares them field by field). */
typedef struct {
    int64_t n;            /* cue: valid occurrences counted; global: positions */
    double mean;          /* cue: mean of window means ([R12]); global: mean margin */
    double std;           /* population std */
    double se;            /* std / sqrt(n) */
    double token_mean;    /* cue: sum of window sums / sum of window lengths; global: = mean */
    double min;           /* min margin inside the windows (global: over positions) */
    double low_frac;      /* #{m < tau} / #tokens (windows, or positions) */
    int64_t n_triggers;   /* first occurrence in its sentence [R13] */
    int64_t n_invalid;    /* windows (global: positions) holding a NaN margin, excluded */
    int32_t selected;     /* P:249-250 selection */
} oracle_summary_t;

/* Per cue and global.  Occurrences at
 * s >= think_end_pos[traj] (when given) are left out of the per-cue table and
 * positions t >= think_end_pos[traj] out of the global moments [R14]; the
 * trigger test looks at every occurrence.  Selection ([R15]):
 * rule 0 = mean_c >= mu + SE_global ("by at least one standard error");
 * rule 1 = mean_c >= mu + se_c; rule 2 = mean_c > mu (App. B);
 * rule 3 = every candidate (the "all candidates" ablation);
 * always also n_c >= min_count.  With fewer than two global positions
 * std and se are NaN and nothing is selected. */
void oracle_cue_stats(const float* margin, int64_t n_tok, const int64_t* traj_offsets,
                      int32_t n_traj, const int64_t* think_end_pos,
                      const int32_t* occ_pos, const int32_t* occ_pat, int64_t n_occ,
                      const int32_t* pat_cue, int32_t n_cues, float tau,
                      const int32_t* seg_end, const double* seg_mean, const double* seg_min,
                      const double* seg_sum, const int32_t* seg_low, const int8_t* seg_invalid,
                      int64_t min_count, int32_t rule, oracle_summary_t* out) {
    /* global */
    oracle_summary_t* g = &out[n_cues];
    memset(g, 0, sizeof *g);
    double gsum = 0.0, gmin = INFINITY;
    int64_t gn = 0, glow = 0, gbad = 0;
    for (int64_t t = 0; t < n_tok; t++) {
        int64_t a, b;
        int64_t k = traj_of(traj_offsets, n_traj, n_tok, t, &a, &b);
        if (k < 0) continue;
        if (think_end_pos && t >= think_end_pos[k]) continue;
        double m = (double)margin[t];
        if (isnan(m)) { gbad++; continue; }
        gn++; gsum += m;
        if (m < gmin) gmin = m;
        if (margin[t] < tau) glow++;
    }
    double gmean = gn ? gsum / (double)gn : NAN;
    double gss = 0.0;
    for (int64_t t = 0; t < n_tok; t++) {
        int64_t a, b;
        int64_t k = traj_of(traj_offsets, n_traj, n_tok, t, &a, &b);
        if (k < 0) continue;
        if (think_end_pos && t >= think_end_pos[k]) continue;
        double m = (double)margin[t];
        if (isnan(m)) continue;
        gss += (m - gmean) * (m - gmean);
    }
    g->n = gn;
    g->mean = gmean;
    g->std = (gn >= 2) ? sqrt(gss / (double)gn) : NAN;
    g->se = (gn >= 2) ? g->std / sqrt((double)gn) : NAN;
    g->token_mean = gmean;
    g->min = gn ? gmin : NAN;
    g->low_frac = gn ? (double)glow / (double)gn : NAN;
    g->n_triggers = 0;
    g->n_invalid = gbad;
    g->selected = 0;

    for (int32_t c = 0; c < n_cues; c++) {
        oracle_summary_t* o = &out[c];
        memset(o, 0, sizeof *o);
        double msum = 0.0, wsum = 0.0, lensum = 0.0, lowsum = 0.0, mn = INFINITY;
        int64_t n = 0, trig = 0, bad = 0;
        for (int64_t i = 0; i < n_occ; i++) {
            if (pat_cue[occ_pat[i]] != c) continue;
            int64_t a, b;
            int64_t k = traj_of(traj_offsets, n_traj, n_tok, occ_pos[i], &a, &b);
            if (think_end_pos && occ_pos[i] >= think_end_pos[k]) continue;
            if (seg_invalid[i]) { bad++; continue; }
            n++;
            msum += seg_mean[i];
            wsum += seg_sum[i];
            lensum += (double)(seg_end[i] - occ_pos[i] + 1);
            lowsum += (double)seg_low[i];
            if (seg_min[i] < mn) mn = seg_min[i];
            /* [R13] trigger = no other occurrence starts earlier in the same
             * sentence (same trajectory, same window end). */
            int first = 1;
            for (int64_t j = 0; j < n_occ; j++) {
                int64_t a2, b2;
                if (occ_pos[j] >= occ_pos[i]) continue;
                if (traj_of(traj_offsets, n_traj, n_tok, occ_pos[j], &a2, &b2) != k) continue;
                if (seg_end[j] == seg_end[i]) { first = 0; break; }
            }
            trig += first;
        }
        double mean = n ? msum / (double)n : NAN;
        double ss = 0.0;
        for (int64_t i = 0; i < n_occ; i++) {
            if (pat_cue[occ_pat[i]] != c) continue;
            int64_t a, b;
            int64_t k = traj_of(traj_offsets, n_traj, n_tok, occ_pos[i], &a, &b);
            if (think_end_pos && occ_pos[i] >= think_end_pos[k]) continue;
            if (seg_invalid[i]) continue;
            ss += (seg_mean[i] - mean) * (seg_mean[i] - mean);
        }
        o->n = n;
        o->mean = mean;
        o->std = n ? sqrt(ss / (double)n) : NAN;
        o->se = n ? o->std / sqrt((double)n) : NAN;
        o->token_mean = n ? wsum / lensum : NAN;
        o->min = n ? mn : NAN;
        o->low_frac = n ? lowsum / lensum : NAN;
        o->n_triggers = trig;
        o->n_invalid = bad;
        int sel = 0;
        if (n >= 1 && n >= min_count && gn >= 2) {
            if (rule == 0) sel = mean >= g->mean + g->se;
            else if (rule == 1) sel = mean >= g->mean + o->se;
            else if (rule == 2) sel = mean > g->mean;
            else sel = 1;  /* rule 3: every candidate (tab:cue_selection_ablation) */
        }
        o->selected = sel;
    }
}

/* ---------------------------------------------------- decode-step switch */
/* Runtime switching (§4.1, §4.3, fig:mechanism P:209-216).
 * state bit0: active model (0 large, 1 small); bit1: answer stage.
 * hist[7]: the tokens of the current large-model turn, oldest first,
 * right-aligned, -1 padded.  Flags: 0 NONE, 1 L2S, 2 S2L, 3 TO_ANSWER,
 * 4 S2L_BUDGET.  Priority </think> > cue > terminator > budget [R16]:
 *   answer stage                    -> NONE (the small model finishes)
 *   tok == think_end                -> TO_ANSWER, state = answer|small
 *   large & a pattern is a suffix of hist++tok -> L2S with its cue,
 *                                     unless margin_gate >= 0 and margin < gate
 *   small & terminator[tok]         -> S2L
 *   small & max_small_segment > 0 & small_run+1 >= max -> S2L_BUDGET
 *   otherwise NONE; large appends tok to hist, small increments small_run.
 * Every switch clears hist and small_run.  Cues emitted by the small model
 * are ignored.  Returns the flag; *cue_out = cue id or -1. */
int oracle_step_one_ex(int32_t tok, float margin, uint8_t* state, int32_t* hist /*[7]*/,
                       int32_t* small_run, const int32_t* pat_tokens, const int32_t* pat_offsets,
                       int32_t n_pat, const int32_t* pat_cue, const uint8_t* terminator,
                       int64_t vocab, int32_t think_end_token, float margin_gate,
                       int32_t max_small_segment, const uint8_t* classes, int32_t n_classes,
                       int32_t* cue_out) {
    const int H = 7;
    *cue_out = -1;
    if (tok < 0 || tok >= vocab) return 0;
    if (*state & 2) return 0;
    if (tok == think_end_token) {
        *state = 3;
        for (int k = 0; k < H; k++) hist[k] = -1;
        *small_run = 0;
        return 3;
    }
    if ((*state & 1) == 0) {
        /* the sequence hist ++ tok, 8 entries, oldest first */
        int32_t seq[8];
        for (int k = 0; k < H; k++) seq[k] = hist[k];
        seq[H] = tok;
        int32_t best = -1;
        for (int32_t p = 0; p < n_pat; p++) {
            int32_t len = pat_offsets[p + 1] - pat_offsets[p];
            int ok = 1;
            for (int32_t k = 0; k < len; k++)
                if (!elem_matches(seq[8 - len + k], pat_tokens[pat_offsets[p] + k], classes,
                                  n_classes, vocab)) { ok = 0; break; }
            if (ok && (best < 0 || len > pat_offsets[best + 1] - pat_offsets[best])) best = p;
        }
        if (best >= 0 && !(margin_gate >= 0.0f && margin < margin_gate)) {
            *state = 1;
            for (int k = 0; k < H; k++) hist[k] = -1;
            *small_run = 0;
            *cue_out = pat_cue[best];
            return 1;
        }
        for (int k = 0; k < H - 1; k++) hist[k] = hist[k + 1];
        hist[H - 1] = tok;
        return 0;
    }
    if (terminator[tok]) {
        *state = 0;
        for (int k = 0; k < H; k++) hist[k] = -1;
        *small_run = 0;
        return 2;
    }
    if (max_small_segment > 0 && *small_run + 1 >= max_small_segment) {
        *state = 0;
        for (int k = 0; k < H; k++) hist[k] = -1;
        *small_run = 0;
        return 4;
    }
    *small_run += 1;
    return 0;
}

int oracle_step_one(int32_t tok, float margin, uint8_t* state, int32_t* hist /*[7]*/,
                    int32_t* small_run, const int32_t* pat_tokens, const int32_t* pat_offsets,
                    int32_t n_pat, const int32_t* pat_cue, const uint8_t* terminator,
                    int64_t vocab, int32_t think_end_token, float margin_gate,
                    int32_t max_small_segment, int32_t* cue_out) {
    return oracle_step_one_ex(tok, margin, state, hist, small_run, pat_tokens, pat_offsets, n_pat,
                              pat_cue, terminator, vocab, think_end_token, margin_gate,
                              max_small_segment, NULL, 0, cue_out);
}

/* --------------------------------------------- fused sampler (N2) --------
 * The decode-side sampling the paper runs with every model (P:332-333:
 * "temperature 0.6 and top-p sampling at 0.95", and for Qwen3 "top-k to 20"),
 * read as [R20]: order the row by (value desc, index asc) [R3]; keep the first
 * K; p_i = exp((z_i - z_(1)) / T) for those K (softmax at temperature T
 * restricted to the top K, unnormalised); keep the first L of them, L = the
 * smallest l with p_0 + ... + p_(l-1) >= top_p * (p_0 + ... + p_(K-1)) (the
 * tokens whose higher-ranked mass is below top_p, at least one); draw the
 * token by inverse CDF with the caller's uniform u in [0, 1): the first i
 * with p_0 + ... + p_i > u * (p_0 + ... + p_(L-1)).  top_k in [1, vocab], or 0
 * for no top-k truncation (K = vocab).
 * A row with status != 0 (NaN / +inf / no finite entry, [R4]) samples -1. */
typedef struct { double v; int64_t i; } ranked_t;

/* (value desc, index asc) [R3] */
static int ranked_cmp(const void* a, const void* b) {
    const ranked_t* x = (const ranked_t*)a;
    const ranked_t* y = (const ranked_t*)b;
    if (x->v > y->v) return -1;
    if (x->v < y->v) return 1;
    return (x->i < y->i) ? -1 : (x->i > y->i);
}

int32_t oracle_sample_row(const void* row, int dtype, int64_t vocab, double inv_temperature,
                          int32_t top_k, double top_p, double u) {
    int32_t i1, i2;
    double m, l;
    if (top_k < 0) return -1;
    if (oracle_margin_row(row, dtype, vocab, 1.0, &i1, &i2, &m, &l) != 0) return -1;
    if (top_k == 0 || top_k > vocab) top_k = (int32_t)vocab;   /* 0: no top-k (R1-Distill) */
    /* the row in (value desc, index asc) order: a library sort */
    ranked_t* all = (ranked_t*)malloc(sizeof(ranked_t) * (size_t)vocab);
    for (int64_t j = 0; j < vocab; j++) { all[j].v = oracle_elem(row, dtype, j); all[j].i = j; }
    qsort(all, (size_t)vocab, sizeof(ranked_t), ranked_cmp);
    int64_t* idx = (int64_t*)malloc(sizeof(int64_t) * (size_t)top_k);
    double* p = (double*)malloc(sizeof(double) * (size_t)top_k);
    for (int32_t r = 0; r < top_k; r++) idx[r] = all[r].i;
    free(all);
    double z1 = oracle_elem(row, dtype, idx[0]);
    double total = 0.0;
    for (int32_t r = 0; r < top_k; r++) {
        double z = oracle_elem(row, dtype, idx[r]);
        p[r] = isinf(z) ? 0.0 : exp((z - z1) * inv_temperature);
        total += p[r];
    }
    int32_t L = 0;
    double above = 0.0;
    while (L < top_k && (L == 0 || above < top_p * total)) { above += p[L]; L++; }
    double kept = 0.0;
    for (int32_t r = 0; r < L; r++) kept += p[r];
    double target = u * kept, cum = 0.0;
    int32_t tok = (int32_t)idx[L - 1];
    for (int32_t r = 0; r < L; r++) {
        cum += p[r];
        if (cum > target) { tok = (int32_t)idx[r]; break; }
    }
    free(idx);
    free(p);
    return tok;
}

/* ------------------------------------------- offload estimate (N3) --------
 * Large-model utilization of the runtime switching (§4.3; the
 * quantity of tab:speedup's "utilization") estimated
 * offline from a trace and a selected cue set [R17]:
 *   reasoning = positions [a, te), te = think_end_pos[k] (b when NULL);
 *   positions [te, b) are the answer stage (small model);
 *   in each sentence (same trajectory, same window end e) the FIRST
 *   occurrence (in list order: by start, then cue id) of a selected cue that
 *   completes inside the
 *   reasoning stage (c = s + len - 1 < te) hands the rest of the sentence to
 *   the small model: positions c+1 .. min(e, te-1);
 *   every other reasoning position is generated by the large model.
 * out[k] = {large, small_reasoning, answer} token counts of trajectory k. */
void oracle_offload(int64_t n_tok, const int64_t* traj_offsets, int32_t n_traj,
                    const int64_t* think_end_pos, const int32_t* occ_pos, const int32_t* occ_pat,
                    int64_t n_occ, const int32_t* seg_end, const int32_t* pat_offsets,
                    const int32_t* pat_cue, const uint8_t* cue_selected, int64_t* out) {
    int32_t nt = traj_offsets ? n_traj : 1;
    for (int32_t k = 0; k < nt; k++) {
        int64_t a = traj_offsets ? traj_offsets[k] : 0;
        int64_t b = traj_offsets ? traj_offsets[k + 1] : n_tok;
        int64_t te = think_end_pos ? think_end_pos[k] : b;
        if (te > b) te = b;
        if (te < a) te = a;
        int64_t small = 0;
        for (int64_t i = 0; i < n_occ; i++) {
            int64_t s = occ_pos[i];
            if (s < a || s >= b) continue;
            int32_t p = occ_pat[i];
            if (!cue_selected[pat_cue[p]]) continue;
            int64_t c = s + (pat_offsets[p + 1] - pat_offsets[p]) - 1;
            if (c >= te) continue;
            /* first selected occurrence of its sentence (list order: by start,
             * then by cue id in ALL mode)? */
            int first = 1;
            for (int64_t j = 0; j < i; j++) {
                if (occ_pos[j] < a) continue;
                if (seg_end[j] != seg_end[i]) continue;
                if (cue_selected[pat_cue[occ_pat[j]]]) { first = 0; break; }
            }
            if (!first) continue;
            int64_t last = seg_end[i] < te - 1 ? seg_end[i] : te - 1;
            if (last > c) small += last - c;
        }
        out[3 * k + 0] = (te - a) - small;
        out[3 * k + 1] = small;
        out[3 * k + 2] = b - te;
    }
}
