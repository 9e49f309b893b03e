/*
 * odc_resub — don't-care based resubstitution for the LUT3 S-box circuits
 * (tools/sboxgen, csrc/sbox_circuits/), a second offline optimiser next to
 * sboxgen.c's decomposition + rip-up search and exact_resyn.py's exact
 * MFFC resynthesis (which match a gate's FULL truth table).
 *
 * Every gate g has observability don't-cares: input rows (of the 64) on which
 * flipping g changes none of the four S-box outputs.  On its care set CARE(g)
 * a gate may be replaced by
 *   - an existing signal s or ~s (0-resub: g's maximum fanout-free cone dies), or
 *   - a new LUT3 of three existing signals (1-resub: the cone minus one dies),
 * where the candidate signals avoid g's transitive fanout (no cycles).  Moves
 * that free gates are taken greedily; neutral 1-resubs (same size, different
 * structure) form a random walk over the plateau so later moves can find
 * gains.  Inversions are free: consumers are LUT3s (their immediate absorbs
 * an input complement) or outputs (a polarity flag, absorbed by the Feistel
 * lop3).  Every accepted circuit is re-verified exhaustively.
 *
 * Usage: odc_resub <box 0..7> <in.txt> <out.txt> <iterations> <seed>
 * Writes out.txt whenever the circuit shrinks below its starting size.
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

typedef uint64_t tt_t;
#define MAXS 128

static const uint8_t SBOX[8][64] = {
    {14, 4, 13, 1, 2, 15, 11, 8, 3, 10, 6, 12, 5, 9, 0, 7, 0, 15, 7, 4, 14, 2, 13, 1, 10, 6, 12, 11, 9, 5, 3, 8,
     4, 1, 14, 8, 13, 6, 2, 11, 15, 12, 9, 7, 3, 10, 5, 0, 15, 12, 8, 2, 4, 9, 1, 7, 5, 11, 3, 14, 10, 0, 6, 13},
    {15, 1, 8, 14, 6, 11, 3, 4, 9, 7, 2, 13, 12, 0, 5, 10, 3, 13, 4, 7, 15, 2, 8, 14, 12, 0, 1, 10, 6, 9, 11, 5,
     0, 14, 7, 11, 10, 4, 13, 1, 5, 8, 12, 6, 9, 3, 2, 15, 13, 8, 10, 1, 3, 15, 4, 2, 11, 6, 7, 12, 0, 5, 14, 9},
    {10, 0, 9, 14, 6, 3, 15, 5, 1, 13, 12, 7, 11, 4, 2, 8, 13, 7, 0, 9, 3, 4, 6, 10, 2, 8, 5, 14, 12, 11, 15, 1,
     13, 6, 4, 9, 8, 15, 3, 0, 11, 1, 2, 12, 5, 10, 14, 7, 1, 10, 13, 0, 6, 9, 8, 7, 4, 15, 14, 3, 11, 5, 2, 12},
    {7, 13, 14, 3, 0, 6, 9, 10, 1, 2, 8, 5, 11, 12, 4, 15, 13, 8, 11, 5, 6, 15, 0, 3, 4, 7, 2, 12, 1, 10, 14, 9,
     10, 6, 9, 0, 12, 11, 7, 13, 15, 1, 3, 14, 5, 2, 8, 4, 3, 15, 0, 6, 10, 1, 13, 8, 9, 4, 5, 11, 12, 7, 2, 14},
    {2, 12, 4, 1, 7, 10, 11, 6, 8, 5, 3, 15, 13, 0, 14, 9, 14, 11, 2, 12, 4, 7, 13, 1, 5, 0, 15, 10, 3, 9, 8, 6,
     4, 2, 1, 11, 10, 13, 7, 8, 15, 9, 12, 5, 6, 3, 0, 14, 11, 8, 12, 7, 1, 14, 2, 13, 6, 15, 0, 9, 10, 4, 5, 3},
    {12, 1, 10, 15, 9, 2, 6, 8, 0, 13, 3, 4, 14, 7, 5, 11, 10, 15, 4, 2, 7, 12, 9, 5, 6, 1, 13, 14, 0, 11, 3, 8,
     9, 14, 15, 5, 2, 8, 12, 3, 7, 0, 4, 10, 1, 13, 11, 6, 4, 3, 2, 12, 9, 5, 15, 10, 11, 14, 1, 7, 6, 0, 8, 13},
    {4, 11, 2, 14, 15, 0, 8, 13, 3, 12, 9, 7, 5, 10, 6, 1, 13, 0, 11, 7, 4, 9, 1, 10, 14, 3, 5, 12, 2, 15, 8, 6,
     1, 4, 11, 13, 12, 3, 7, 14, 10, 15, 6, 8, 0, 5, 9, 2, 6, 11, 13, 8, 1, 4, 10, 7, 9, 5, 0, 15, 14, 2, 3, 12},
    {13, 2, 8, 4, 6, 15, 11, 1, 10, 9, 3, 14, 5, 0, 12, 7, 1, 15, 13, 8, 10, 3, 7, 4, 12, 5, 6, 11, 0, 14, 9, 2,
     7, 11, 4, 1, 9, 12, 14, 2, 0, 6, 10, 13, 15, 3, 5, 8, 2, 1, 14, 7, 4, 10, 8, 13, 15, 12, 9, 0, 3, 5, 6, 11}};

typedef struct {
    int n;                 /* signals 0..n-1; 0..5 inputs */
    int in[MAXS][3];
    uint8_t lut[MAXS];
    int alive[MAXS];
    int out[4], inv[4];
    tt_t tt[MAXS];
    int order[MAXS], norder;  /* live gates, topological */
} circ_t;

static tt_t TARGET[4];
static long n_neutral = 0, n_gain = 0, n_zero = 0, n_two = 0;
static int g_two = 0; /* 2-resub enabled (ODC_TWO=1): slow, ~1e9 checks per gate */
static uint64_t rng = 0x9E3779B97F4A7C15ull;
static uint64_t rnd(void) {
    rng ^= rng << 13;
    rng ^= rng >> 7;
    rng ^= rng << 17;
    return rng;
}

static tt_t lut_eval(uint8_t lut, tt_t a, tt_t b, tt_t c) {
    tt_t r = 0;
    for (int m = 0; m < 8; m++)
        if ((lut >> m) & 1) r |= ((m & 4) ? a : ~a) & ((m & 2) ? b : ~b) & ((m & 1) ? c : ~c);
    return r;
}

/* LUT with LUT(a,b,c) == T on M (unconstrained minterms 0), or -1 */
static int find_lut3(tt_t a, tt_t b, tt_t c, tt_t T, tt_t M) {
    int l = 0;
    for (int m = 0; m < 8; m++) {
        tt_t P = M & ((m & 4) ? a : ~a) & ((m & 2) ? b : ~b) & ((m & 1) ? c : ~c);
        tt_t t = T & P;
        if (t == 0) continue;
        if (t != P) return -1;
        l |= 1 << m;
    }
    return l;
}

static int visit_state[MAXS];
static void topo_visit(circ_t* c, int s) {
    if (s < 6 || visit_state[s]) return;
    visit_state[s] = 1;
    for (int k = 0; k < 3; k++) topo_visit(c, c->in[s][k]);
    c->order[c->norder++] = s;
}

/* topological order of the gates the outputs need; dead gates dropped */
static void rebuild(circ_t* c) {
    memset(visit_state, 0, sizeof visit_state);
    c->norder = 0;
    for (int o = 0; o < 4; o++) topo_visit(c, c->out[o]);
    for (int s = 6; s < c->n; s++) c->alive[s] = visit_state[s];
    for (int k = 0; k < 6; k++) c->tt[k] = 0;
    for (int r = 0; r < 64; r++)
        for (int k = 0; k < 6; k++)
            if ((r >> k) & 1) c->tt[k] |= 1ull << r;
    for (int i = 0; i < c->norder; i++) {
        int g = c->order[i];
        c->tt[g] = lut_eval(c->lut[g], c->tt[c->in[g][0]], c->tt[c->in[g][1]], c->tt[c->in[g][2]]);
    }
}

static int gates(const circ_t* c) { return c->norder; }

static int correct(const circ_t* c) {
    for (int o = 0; o < 4; o++)
        if ((c->tt[c->out[o]] ^ (c->inv[o] ? ~0ull : 0ull)) != TARGET[o]) return 0;
    return 1;
}

static void tfo(const circ_t* c, int g, int* mark) {
    memset(mark, 0, sizeof(int) * MAXS);
    mark[g] = 1;
    for (int i = 0; i < c->norder; i++) {
        int s = c->order[i];
        for (int k = 0; k < 3; k++)
            if (mark[c->in[s][k]]) mark[s] = 1;
    }
}

/* rows on which flipping g changes an output */
static tt_t care_of(const circ_t* c, int g, const int* mark) {
    tt_t v[MAXS];
    memcpy(v, c->tt, sizeof(tt_t) * c->n);
    v[g] = ~v[g];
    for (int i = 0; i < c->norder; i++) {
        int s = c->order[i];
        if (s != g && mark[s]) v[s] = lut_eval(c->lut[s], v[c->in[s][0]], v[c->in[s][1]], v[c->in[s][2]]);
    }
    tt_t d = 0;
    for (int o = 0; o < 4; o++) d |= v[c->out[o]] ^ c->tt[c->out[o]];
    return d;
}

/* replace every use of g by s (complemented if neg) */
static void redirect(circ_t* c, int g, int s, int neg) {
    for (int i = 0; i < c->norder; i++) {
        int u = c->order[i];
        for (int k = 0; k < 3; k++)
            if (c->in[u][k] == g) {
                c->in[u][k] = s;
                if (neg) { /* complement input k in the LUT */
                    uint8_t l = 0;
                    const int bit = 2 - k; /* input 0 is the MSB of the minterm index */
                    for (int m = 0; m < 8; m++)
                        if ((c->lut[u] >> m) & 1) l |= 1 << (m ^ (1 << bit));
                    c->lut[u] = l;
                }
            }
    }
    for (int o = 0; o < 4; o++)
        if (c->out[o] == g) {
            c->out[o] = s;
            c->inv[o] ^= neg;
        }
}

static int load(circ_t* c, const char* path) {
    FILE* f = fopen(path, "r");
    if (!f) return 0;
    memset(c, 0, sizeof *c);
    c->n = 6;
    char w[16];
    while (fscanf(f, "%15s", w) == 1) {
        if (!strcmp(w, "box")) {
            int b, n;
            if (fscanf(f, "%d gates %d", &b, &n) != 2) return 0;
        } else if (!strcmp(w, "g")) {
            int id, a, b, cc;
            unsigned l;
            if (fscanf(f, "%d %d %d %d %x", &id, &a, &b, &cc, &l) != 5) return 0;
            if (id + 1 > c->n) c->n = id + 1;
            c->in[id][0] = a;
            c->in[id][1] = b;
            c->in[id][2] = cc;
            c->lut[id] = (uint8_t)l;
        } else if (!strcmp(w, "o")) {
            int o, s, inv;
            if (fscanf(f, "%d %d %d", &o, &s, &inv) != 3) return 0;
            c->out[o] = s;
            c->inv[o] = inv;
        } else {
            return 0; /* Feistel-top lines are not handled */
        }
    }
    fclose(f);
    rebuild(c);
    return 1;
}

/* compact ids in topological order and write the sboxgen text format */
static void save(const circ_t* c, int box, const char* path) {
    int id[MAXS];
    for (int k = 0; k < 6; k++) id[k] = k;
    for (int i = 0; i < c->norder; i++) id[c->order[i]] = 6 + i;
    FILE* f = fopen(path, "w");
    fprintf(f, "box %d gates %d\n", box, c->norder);
    for (int i = 0; i < c->norder; i++) {
        int g = c->order[i];
        fprintf(f, "g %d %d %d %d 0x%02x\n", 6 + i, id[c->in[g][0]], id[c->in[g][1]], id[c->in[g][2]], c->lut[g]);
    }
    for (int o = 0; o < 4; o++) fprintf(f, "o %d %d %d\n", o, id[c->out[o]], c->inv[o]);
    fclose(f);
}

/* one move at gate g: 0-resub if possible, else a 1-resub (improving if
 * available, else a random neutral one with probability p_neutral) */
static int move(circ_t* c, int g, int p_neutral_pct) {
    int mark[MAXS];
    tfo(c, g, mark);
    const tt_t care = care_of(c, g, mark);
    const tt_t T = c->tt[g];
    const int before = gates(c);
    /* 0-resub */
    int cand[MAXS], nc = 0;
    for (int s = 0; s < c->n; s++)
        if ((s < 6 || c->alive[s]) && !mark[s]) cand[nc++] = s;
    for (int i = nc - 1; i > 0; i--) { /* shuffle */
        int j = (int)(rnd() % (uint64_t)(i + 1)), t = cand[i];
        cand[i] = cand[j];
        cand[j] = t;
    }
    for (int i = 0; i < nc; i++) {
        const int s = cand[i];
        const tt_t d = (c->tt[s] ^ T) & care, dn = (~c->tt[s] ^ T) & care;
        if (d == 0 || dn == 0) {
            circ_t t = *c;
            redirect(&t, g, s, d != 0);
            rebuild(&t);
            if (correct(&t) && gates(&t) < before) {
                *c = t;
                ++n_zero;
                return before - gates(c);
            }
        }
    }
    /* 1-resub: new LUT3 for g over candidates outside its fanout */
    int best_gain = -1000, ba = -1, bb = -1, bc = -1, bl = 0, seen = 0;
    for (int i = 0; i < nc; i++)
        for (int j = i + 1; j < nc; j++)
            for (int k = j + 1; k < nc; k++) {
                const int l = find_lut3(c->tt[cand[i]], c->tt[cand[j]], c->tt[cand[k]], T, care);
                if (l < 0) continue;
                circ_t t = *c;
                t.in[g][0] = cand[i];
                t.in[g][1] = cand[j];
                t.in[g][2] = cand[k];
                t.lut[g] = (uint8_t)l;
                rebuild(&t);
                if (!correct(&t)) continue;
                const int gain = before - gates(&t);
                ++seen;
                /* reservoir choice among the best gains */
                if (gain > best_gain || (gain == best_gain && rnd() % (uint64_t)seen == 0)) {
                    if (gain > best_gain) seen = 1;
                    best_gain = gain;
                    ba = cand[i];
                    bb = cand[j];
                    bc = cand[k];
                    bl = l;
                }
            }
    if (best_gain <= 0 && g_two) {
        /* 2-resub: g' = LUT3(h, x, y), h = LUT3(a, b, c) new, when g's
         * fanout-free cone has >= 3 gates (gain >= 1) */
        circ_t t = *c;
        t.in[g][0] = t.in[g][1] = t.in[g][2] = 0;
        rebuild(&t);
        const int mffc = before - gates(&t) + 1;
        if (mffc >= 3 && c->n < MAXS) {
            for (int i = 0; i < nc; i++)
                for (int j = i + 1; j < nc; j++)
                    for (int k = j + 1; k < nc; k++) {
                        const tt_t A = c->tt[cand[i]], B = c->tt[cand[j]], C = c->tt[cand[k]];
                        for (int l = 1; l < 255; l++) {
                            const tt_t H = lut_eval((uint8_t)l, A, B, C);
                            for (int x = 0; x < nc; x++)
                                for (int y = x + 1; y < nc; y++) {
                                    const int l2 = find_lut3(H, c->tt[cand[x]], c->tt[cand[y]], T, care);
                                    if (l2 < 0) continue;
                                    circ_t u = *c;
                                    const int h = u.n++;
                                    u.in[h][0] = cand[i];
                                    u.in[h][1] = cand[j];
                                    u.in[h][2] = cand[k];
                                    u.lut[h] = (uint8_t)l;
                                    u.in[g][0] = h;
                                    u.in[g][1] = cand[x];
                                    u.in[g][2] = cand[y];
                                    u.lut[g] = (uint8_t)l2;
                                    rebuild(&u);
                                    if (correct(&u) && gates(&u) < before) {
                                        *c = u;
                                        ++n_two;
                                        return before - gates(c);
                                    }
                                }
                        }
                    }
        }
    }
    if (ba < 0) return 0;
    if (best_gain > 0 || (best_gain == 0 && (int)(rnd() % 100) < p_neutral_pct)) {
        c->in[g][0] = ba;
        c->in[g][1] = bb;
        c->in[g][2] = bc;
        c->lut[g] = (uint8_t)bl;
        rebuild(c);
        if (best_gain > 0) ++n_gain;
        else ++n_neutral;
        return best_gain;
    }
    return 0;
}

int main(int argc, char** argv) {
    if (argc < 6) {
        fprintf(stderr, "usage: %s box in.txt out.txt iterations seed\n", argv[0]);
        return 2;
    }
    const int box = atoi(argv[1]);
    const long iters = atol(argv[4]);
    rng ^= (uint64_t)atoll(argv[5]) * 0xD1B54A32D192ED03ull;
    for (int o = 0; o < 4; o++) {
        TARGET[o] = 0;
        for (int r = 0; r < 64; r++) {
            const int row = ((r >> 4) & 2) | (r & 1), col = (r >> 1) & 0xF;
            if ((SBOX[box][row * 16 + col] >> o) & 1) TARGET[o] |= 1ull << r;
        }
    }
    circ_t c, best;
    if (!load(&c, argv[2]) || !correct(&c)) {
        fprintf(stderr, "cannot load a correct circuit from %s\n", argv[2]);
        return 1;
    }
    g_two = getenv("ODC_TWO") && atoi(getenv("ODC_TWO"));
    const int start = gates(&c);
    best = c;
    fprintf(stderr, "box %d: start %d gates\n", box, start);
    for (long it = 0; it < iters; it++) {
        const int g = c.order[rnd() % (uint64_t)c.norder];
        move(&c, g, 60);
        if (gates(&c) < gates(&best)) {
            best = c;
            save(&best, box, argv[3]);
            fprintf(stderr, "box %d: %d gates at iteration %ld\n", box, gates(&best), it);
        }
        if (it % 20000 == 19999) {
            if (gates(&c) > gates(&best)) c = best; /* never happens: moves do not grow */
            fprintf(stderr, "box %d: iteration %ld, current %d, best %d (neutral %ld, 1-resub gains %ld, 0-resub %ld, 2-resub %ld)\n",
                    box, it + 1, gates(&c), gates(&best), n_neutral, n_gain, n_zero, n_two);
        }
    }
    printf("box %d: %d -> %d gates\n", box, start, gates(&best));
    return 0;
}
