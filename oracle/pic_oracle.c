/* CPU oracle for the kernelweave.pic hot path -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference PIC cycle (reference:
 * /root/reference/pkg/src/kernelweave/pic/{kernels,particles}.py and
 * kw/atomics.py) used by tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg as the checker and the CPU timing
 * port.  It is never linked into, or called by, the product library.
 *
 * Parity: pinned bitwise against golden dumps of the unmodified reference
 * (tests/golden/make_golden.py, tests/test_oracle_golden.py).
 *
 * Build: oracle/Makefile (gcc -O2 -ffp-contract=off -fopenmp).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#if defined(__FP_FAST_FMA) && !defined(ORACLE_ALLOW_FMA)
/* contraction is disabled by -ffp-contract=off; this only documents intent */
#endif

typedef struct {
    int64_t n_sc, cap;
    const int32_t *head, *next_f;
    uint8_t *occ;
    void *ox, *oy, *oz, *ux, *uy, *uz, *w;
    void *epx, *epy, *epz, *bpx, *bpy, *bpz;
    void *oox, *ooy, *ooz;
    int32_t *cx, *cy, *cz, *ocx, *ocy, *ocz;
} orc_store;

typedef struct {
    int64_t nx, ny, nz;
    double dx, dy, dz;
    void *Ex, *Ey, *Ez, *Bx, *By, *Bz, *Jx, *Jy, *Jz;
} orc_fields;

typedef struct {
    int32_t *head, *tail, *next_f, *prev_f, *owner, *nfilled, *free_stack;
    int64_t *free_top;
} orc_pool;

static inline int64_t pymod(int64_t a, int64_t n) {
    int64_t r = a % n;
    return r < 0 ? r + n : r;
}

/* pic/fields.py:24-31 STAGGER, in the order Ex Ey Ez Bx By Bz. */
static const double ORC_STAGGER[6][3] = {
    {1.0, 0.5, 0.5}, {0.5, 1.0, 0.5}, {0.5, 0.5, 1.0},
    {0.5, 1.0, 1.0}, {1.0, 0.5, 1.0}, {1.0, 1.0, 0.5},
};

int orc_version(void) { return 1; }

/* splitmix64 */
static uint64_t orc_rng_next(uint64_t *s) {
    uint64_t z = (*s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

/* Tile merge order of the deposit: 0 = ascending super cells (the Serial
 * back-end); otherwise the seed of a random permutation (BlockPool-like). */
static uint64_t orc_merge_seed = 0;
void orc_set_merge_seed(uint64_t seed) { orc_merge_seed = seed; }
/* Particle order within each frame of a tile: 0 ascending slots (Serial). */
static int orc_reverse_slots = 0;
void orc_set_reverse_slots(int on) { orc_reverse_slots = on; }

#define FT float
#define SFX _f32
#include "pic_oracle_impl.h"
#undef FT
#undef SFX

#define FT double
#define SFX _f64
#include "pic_oracle_impl.h"
#undef FT
#undef SFX

/* pic/particles.py:214-235 `_scan_leavers`: canonical order (super cell
 * ascending, chain order, slot ascending). */
int64_t orc_scan_leavers(const orc_store *st, const int32_t *nfilled, int64_t scx, int64_t scy,
                         int64_t scz, int64_t gx, int64_t gy, int32_t *out_f, int32_t *out_s,
                         int32_t *out_dest) {
    int64_t n = 0;
    for (int64_t sc = 0; sc < st->n_sc; ++sc) {
        for (int32_t f = st->head[sc]; f >= 0; f = st->next_f[f]) {
            if (nfilled[f] <= 0) continue;
            for (int64_t s = 0; s < st->cap; ++s) {
                int64_t q = (int64_t)f * st->cap + s;
                if (!st->occ[q]) continue;
                int64_t dsc = (st->cx[q] / scx) + gx * ((st->cy[q] / scy) + gy * (st->cz[q] / scz));
                if (dsc != sc) {
                    out_f[n] = f;
                    out_s[n] = (int32_t)s;
                    out_dest[n] = (int32_t)dsc;
                    ++n;
                }
            }
        }
    }
    return n;
}

/* pic/particles.py:290-313 `_unlink_empty`. */
void orc_unlink_empty(orc_pool *pl, int64_t n_sc) {
    for (int64_t sc = 0; sc < n_sc; ++sc) {
        int32_t f = pl->head[sc];
        while (f >= 0) {
            int32_t nxt = pl->next_f[f];
            if (pl->nfilled[f] == 0) {
                int32_t p = pl->prev_f[f], q = pl->next_f[f];
                if (p >= 0) pl->next_f[p] = q; else pl->head[sc] = q;
                if (q >= 0) pl->prev_f[q] = p; else pl->tail[sc] = p;
                pl->owner[f] = -1;
                pl->next_f[f] = -1;
                pl->prev_f[f] = -1;
                pl->free_stack[pl->free_top[0]] = f;
                pl->free_top[0] += 1;
            }
            f = nxt;
        }
    }
}

/* ---- test support: the GPU's shared-reciprocal division ------------------
 * The CUDA advance computes the push's and the move's three quotients by one
 * divisor as q0 = RN(a r), e = fma(-q0, b, a), q = copysign(fma(e, r, q0), a)
 * with r = RN(1 / b) (Markstein).  This checks that construction against
 * IEEE a / b on n pseudo-random pairs drawn like the kernel's operands:
 * numerators of either sign over 2^-40 .. 2^4 (including exact zeros of
 * either sign), divisors over 1 .. 2^6.  Returns the number of pairs whose
 * bit patterns differ.  C99 fma() is the same IEEE operation as __fma_rn. */

int64_t orc_div_rcp_check(int64_t n, uint64_t seed) {
    int64_t bad = 0;
    uint64_t st = seed;
    for (int64_t i = 0; i < n; ++i) {
        const uint64_t u1 = orc_rng_next(&st), u2 = orc_rng_next(&st), u3 = orc_rng_next(&st);
        const double m1 = 1.0 + (double)(u1 >> 11) * 0x1.0p-53;         /* [1, 2) */
        const double m2 = 1.0 + (double)(u2 >> 11) * 0x1.0p-53;
        const int e1 = (int)(u3 % 45) - 40, e2 = (int)((u3 >> 8) % 7);
        double a = ldexp(m1, e1), b = ldexp(m2, e2);
        if ((u3 >> 16) & 1) a = -a;
        if (((u3 >> 17) & 1023) == 0) a = ((u3 >> 27) & 1) ? -0.0 : 0.0;
        const double r = 1.0 / b;
        const double q0 = a * r;
        const double e = fma(-q0, b, a);
        /* b > 0: the quotient carries a's sign (csrc/common.cuh div_rcp) */
        const double q = copysign(fma(e, r, q0), a);
        const double ref = a / b;
        uint64_t x, y;
        memcpy(&x, &q, 8);
        memcpy(&y, &ref, 8);
        bad += x != y;
    }
    return bad;
}

/* The same construction for the PCS weights' a / 6 (csrc/advance.cuh div6:
 * r = RN(1/6)) over non-negative numerators 2^-60 .. 4 and exact zero. */
int64_t orc_div6_check(int64_t n, uint64_t seed) {
    int64_t bad = 0;
    uint64_t st = seed;
    const double b = 6.0, r = 1.0 / 6.0;
    for (int64_t i = 0; i < n; ++i) {
        const uint64_t u1 = orc_rng_next(&st), u3 = orc_rng_next(&st);
        const double m1 = 1.0 + (double)(u1 >> 11) * 0x1.0p-53;
        const int e1 = (int)(u3 % 62) - 60;
        double a = ldexp(m1, e1);
        if (((u3 >> 17) & 1023) == 0) a = 0.0;
        const double q0 = a * r;
        const double e = fma(-q0, b, a);
        /* b > 0: the quotient carries a's sign (csrc/common.cuh div_rcp) */
        const double q = copysign(fma(e, r, q0), a);
        const double ref = a / b;
        uint64_t x, y;
        memcpy(&x, &q, 8);
        memcpy(&y, &ref, 8);
        bad += x != y;
    }
    return bad;
}
