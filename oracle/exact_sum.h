/*
 * exact_sum.h -- the nodal assembly sum of the oracle, computed exactly and rounded once
 * (reading R27).  TEST INFRASTRUCTURE ONLY (oracle-internal; the product never
 * includes it).
 *
 * PAPER.md:L342 defines f_int,k through the assembly operator A: the sum of the element
 * contributions f_{e,a} over the elements e that hold node k.  The paper fixes no
 * floating-point evaluation order for it; this oracle takes the value of that sum to be the
 * exact real sum of the fp64 contributions, rounded once to the nearest fp64 (ties to even).
 * That value does not depend on the order of the terms.
 *
 * Method: a fixed-point accumulator spanning the whole fp64 range.  Every finite double is
 * m * 2^e with an integer 0 <= m < 2^53 and -1074 <= e <= 971; limb i of the accumulator
 * holds bits [32 i, 32 i + 32) of the exact integer sum * 2^1120 in a signed 64-bit word
 * (room for 2^31 additions between carry passes).  The final value is rounded by reading
 * the bits of the normalised integer: 53 bits (fewer below 2^-1022), the round bit, the
 * sticky bits.  Pinned against Python's fractions.Fraction sums (exact rationals, whose
 * float() is correctly rounded) in tests/test_oracle_exact_sum.py.
 */
#ifndef ORC_EXACT_SUM_H
#define ORC_EXACT_SUM_H
#include <math.h>
#include <stdint.h>
#include <string.h>

#define XS_LIMBS 68   /* bits up to 2^(32*68) > 2^(971+53+1120) */
#define XS_BIAS 1120  /* weight of bit 0 is 2^-1120 (< 2^-1074, the smallest subnormal) */

typedef struct {
    int64_t w[XS_LIMBS];
    double nonfinite; /* plain sum of the non-finite terms (inf / nan propagate) */
    int has_nonfinite;
} xsum;

static inline void xsum_init(xsum *a) {
    memset(a->w, 0, sizeof(a->w));
    a->nonfinite = 0.0;
    a->has_nonfinite = 0;
}

static inline void xsum_add(xsum *a, double x) {
    if (!isfinite(x)) {
        a->nonfinite = a->nonfinite + x;
        a->has_nonfinite = 1;
        return;
    }
    uint64_t bits;
    memcpy(&bits, &x, 8);
    const int neg = (int)(bits >> 63);
    const int ef = (int)((bits >> 52) & 0x7ff);
    uint64_t m = bits & ((UINT64_C(1) << 52) - 1);
    int e;
    if (ef == 0) {
        e = -1074; /* zero or subnormal */
    } else {
        m |= UINT64_C(1) << 52;
        e = ef - 1075;
    }
    if (m == 0) return;
    const int p = e + XS_BIAS; /* bit position of m's bit 0 */
    const int i = p >> 5, r = p & 31;
    const unsigned __int128 v = (unsigned __int128)m << r; /* < 2^85: three 32-bit pieces */
    const int64_t p0 = (int64_t)(uint64_t)(v & 0xffffffffu);
    const int64_t p1 = (int64_t)(uint64_t)((v >> 32) & 0xffffffffu);
    const int64_t p2 = (int64_t)(uint64_t)(v >> 64);
    if (neg) {
        a->w[i] -= p0; a->w[i + 1] -= p1; a->w[i + 2] -= p2;
    } else {
        a->w[i] += p0; a->w[i + 1] += p1; a->w[i + 2] += p2;
    }
}

/* carry pass: every limb below the top into [0, 2^32), the sign in the top limb */
static inline void xsum_carry(int64_t *w) {
    for (int i = 0; i < XS_LIMBS - 1; ++i) {
        const int64_t c = w[i] >> 32; /* floor division by 2^32 (arithmetic shift) */
        w[i] -= c * ((int64_t)1 << 32);
        w[i + 1] += c;
    }
}

static inline int xs_bit(const int64_t *w, int pos) { return (int)((w[pos >> 5] >> (pos & 31)) & 1); }

/* the exact sum rounded to the nearest double, ties to even (+0.0 for an exact zero) */
static inline double xsum_round(const xsum *a) {
    if (a->has_nonfinite) return a->nonfinite;
    int64_t w[XS_LIMBS];
    memcpy(w, a->w, sizeof(w));
    xsum_carry(w);
    int neg = 0;
    if (w[XS_LIMBS - 1] < 0) { /* negative: round the magnitude, then negate */
        neg = 1;
        for (int i = 0; i < XS_LIMBS; ++i) w[i] = -w[i];
        xsum_carry(w);
    }
    int h = XS_LIMBS - 1;
    while (h >= 0 && w[h] == 0) --h;
    if (h < 0) return 0.0;
    int top = 31;
    while (!((w[h] >> top) & 1)) --top;
    const int P = 32 * h + top;                /* position of the leading bit */
    int nb = P - (XS_BIAS - 1074) + 1;         /* bits down to weight 2^-1074 */
    if (nb > 53) nb = 53;
    const int L = P - nb + 1;                  /* lowest kept bit */
    uint64_t M = 0;
    for (int pos = P; pos >= L; --pos) M = (M << 1) | (uint64_t)xs_bit(w, pos);
    int round = 0, sticky = 0;
    if (L > 0) {
        round = xs_bit(w, L - 1);
        for (int pos = L - 2; pos >= 0 && !sticky; --pos) {
            if ((pos & 31) == 31 && w[pos >> 5] == 0) { pos -= 31; continue; } /* whole zero limb */
            sticky = xs_bit(w, pos);
        }
    }
    if (round && (sticky || (M & 1))) M += 1;
    const double r = ldexp((double)M, L - XS_BIAS); /* exact (or +inf past the fp64 range) */
    return neg ? -r : r;
}

#endif
