/*
 * sa_lut3 — simulated annealing over fixed-size LUT3 networks for one DES
 * S-box (a Cartesian-genetic-programming-style search, the third approach
 * next to sboxgen.c's constructive decomposition and odc_resub.c's
 * don't-care resubstitution).
 *
 * A candidate is n gates g_i = LUT_i(a, b, c) with a, b, c any earlier
 * signal (the six S-box inputs or gates < i).  Each of the four S-box
 * outputs may be taken from any signal, in either polarity (consumers are
 * lop3s or the Feistel lop3, which absorb an inversion), so the cost is
 *   sum over outputs o of min over signals s of popcount(tt[s] ^ T_o),
 * min'd with the complement — 0 means a correct n-gate circuit.  Moves
 * rewire one input of one gate or change its LUT; a move is accepted with
 * the Metropolis rule; restarts from random or from a seed circuit.
 *
 * Usage: sa_lut3 <box> <gates> <seconds> <seed> <out.txt> [init.txt]
 * Writes out.txt (sboxgen format, verified) when it finds a correct circuit.
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

typedef uint64_t tt_t;
#define MAXG 40

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

static int NG;            /* gates */
static tt_t TGT[4];
static uint64_t rng = 0x9E3779B97F4A7C15ull;
static inline uint64_t rnd(void) {
    rng ^= rng << 13;
    rng ^= rng >> 7;
    rng ^= rng << 17;
    return rng;
}
static inline double urand(void) { return (rnd() >> 11) * (1.0 / 9007199254740992.0); }

typedef struct {
    int in[MAXG][3];
    uint8_t lut[MAXG];
    tt_t tt[6 + MAXG];
} net_t;

static inline tt_t lut_eval(uint8_t lut, tt_t a, tt_t b, tt_t c) {
    tt_t r = 0;
    for (int m = 0; m < 8; m++)
        if ((lut >> m) & 1) r |= ((m & 4) ? a : ~a) & ((m & 2) ? b : ~b) & ((m & 1) ? c : ~c);
    return r;
}

static void eval_from(net_t* n, int g0) {
    for (int g = g0; g < NG; g++)
        n->tt[6 + g] = lut_eval(n->lut[g], n->tt[n->in[g][0]], n->tt[n->in[g][1]], n->tt[n->in[g][2]]);
}

/* cost and, optionally, the chosen output signals / polarities */
static int cost(const net_t* n, int* osig, int* oinv) {
    int total = 0;
    for (int o = 0; o < 4; o++) {
        int best = 65, bs = 0, bi = 0;
        for (int s = 0; s < 6 + NG; s++) {
            const int d = __builtin_popcountll(n->tt[s] ^ TGT[o]);
            if (d < best) best = d, bs = s, bi = 0;
            if (64 - d < best) best = 64 - d, bs = s, bi = 1;
        }
        total += best;
        if (osig) osig[o] = bs, oinv[o] = bi;
    }
    return total;
}

static void randomize(net_t* n) {
    for (int g = 0; g < NG; g++) {
        for (int k = 0; k < 3; k++) n->in[g][k] = (int)(rnd() % (uint64_t)(6 + g));
        n->lut[g] = (uint8_t)rnd();
    }
    eval_from(n, 0);
}

static int load(net_t* n, const char* path) {
    FILE* f = fopen(path, "r");
    if (!f) return 0;
    char w[16];
    int g = 0;
    while (fscanf(f, "%15s", w) == 1) {
        if (!strcmp(w, "box")) {
            int b, m;
            if (fscanf(f, "%d gates %d", &b, &m) != 2) return 0;
        } else if (!strcmp(w, "g")) {
            int id, a, b, c;
            unsigned l;
            if (fscanf(f, "%d %d %d %d %x", &id, &a, &b, &c, &l) != 5) return 0;
            if (g >= NG) { fclose(f); return 0; }
            n->in[g][0] = a; n->in[g][1] = b; n->in[g][2] = c;
            n->lut[g] = (uint8_t)l;
            ++g;
        } else {
            int x, y, z;
            if (fscanf(f, "%d %d %d", &x, &y, &z) != 3) return 0;
        }
    }
    fclose(f);
    for (; g < NG; g++) { /* pad with dummies */
        for (int k = 0; k < 3; k++) n->in[g][k] = (int)(rnd() % (uint64_t)(6 + g));
        n->lut[g] = (uint8_t)rnd();
    }
    eval_from(n, 0);
    return 1;
}

static void save(const net_t* n, int box, const char* path) {
    int osig[4], oinv[4];
    cost(n, osig, oinv);
    FILE* f = fopen(path, "w");
    fprintf(f, "box %d gates %d\n", box, NG);
    for (int g = 0; g < NG; g++)
        fprintf(f, "g %d %d %d %d 0x%02x\n", 6 + g, n->in[g][0], n->in[g][1], n->in[g][2], n->lut[g]);
    for (int o = 0; o < 4; o++) fprintf(f, "o %d %d %d\n", o, osig[o], oinv[o]);
    fclose(f);
}

int main(int argc, char** argv) {
    if (argc < 6) {
        fprintf(stderr, "usage: %s box gates seconds seed out.txt [init.txt]\n", argv[0]);
        return 2;
    }
    const int box = atoi(argv[1]);
    NG = atoi(argv[2]);
    const double secs = atof(argv[3]);
    rng ^= (uint64_t)atoll(argv[4]) * 0xD1B54A32D192ED03ull;
    if (NG < 1 || NG > MAXG) return 2;
    for (int o = 0; o < 4; o++) {
        TGT[o] = 0;
        for (int r = 0; r < 64; r++) {
            const int row = ((r >> 4) & 2) | (r & 1), col = (r >> 1) & 0xF;
            if ((SBOX[box][row * 16 + col] >> o) & 1) TGT[o] |= 1ull << r;
        }
    }
    net_t cur;
    memset(&cur, 0, sizeof cur);
    for (int k = 0; k < 6; k++) {
        cur.tt[k] = 0;
        for (int r = 0; r < 64; r++)
            if ((r >> k) & 1) cur.tt[k] |= 1ull << r;
    }
    const int have_init = argc > 6;
    if (have_init ? !load(&cur, argv[6]) : (randomize(&cur), 0)) {
        fprintf(stderr, "bad init\n");
        return 1;
    }
    int c = cost(&cur, NULL, NULL), best = c;
    const time_t t_end = time(NULL) + (time_t)secs;
    long it = 0, restarts = 0;
    double T = 2.0;
    net_t save_n;
    while (time(NULL) < t_end) {
        for (int inner = 0; inner < 200000; inner++, it++) {
            const int g = (int)(rnd() % (uint64_t)NG);
            const int old_in[3] = {cur.in[g][0], cur.in[g][1], cur.in[g][2]};
            const uint8_t old_lut = cur.lut[g];
            const uint64_t r = rnd();
            if (r & 1) {
                cur.in[g][(r >> 1) % 3] = (int)((r >> 8) % (uint64_t)(6 + g));
                cur.lut[g] = (uint8_t)(r >> 40);  /* a rewired gate gets a fresh function */
            } else {
                cur.lut[g] ^= (uint8_t)(1u << ((r >> 1) & 7));
            }
            memcpy(save_n.tt, cur.tt, sizeof cur.tt);
            eval_from(&cur, g);
            const int nc = cost(&cur, NULL, NULL);
            if (nc <= c || urand() < exp((c - nc) / T)) {
                c = nc;
                if (c < best) best = c;
                if (c == 0) {
                    save(&cur, box, argv[5]);
                    printf("box %d: correct %d-gate circuit after %ld moves\n", box, NG, it);
                    return 0;
                }
            } else {
                cur.in[g][0] = old_in[0];
                cur.in[g][1] = old_in[1];
                cur.in[g][2] = old_in[2];
                cur.lut[g] = old_lut;
                memcpy(cur.tt, save_n.tt, sizeof cur.tt);
            }
        }
        T *= 0.97;
        if (T < 0.05) { /* reheat from the seed circuit or a fresh random one */
            T = 2.0;
            ++restarts;
            if (have_init) load(&cur, argv[6]);
            else randomize(&cur);
            c = cost(&cur, NULL, NULL);
        }
    }
    printf("box %d: no %d-gate circuit (best cost %d bits, %ld moves, %ld restarts)\n", box, NG, best, it, restarts);
    return 1;
}
