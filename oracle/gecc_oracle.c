/* TEST INFRASTRUCTURE ONLY -- see gecc_oracle.h for the parity status header.
 *
 * Plain-C restatement of the reference's batched EC path.  Every function
 * names the reference lines (under /root/reference/proj/) whose behaviour it
 * follows.  Written from the behaviour, not transliterated: one translation
 * unit, AoS value types, explicit error codes instead of exceptions, and the
 * curve passed as data so SM2 and secp256k1 share the code.
 */
#include "gecc_oracle.h"

#include <stdlib.h>
#include <string.h>

typedef struct { uint32_t w[8]; } u256;
typedef struct { uint32_t w[16]; } u512;

typedef struct {
    u256 q;
    uint32_t q_inv; /* -q^-1 mod 2^32 */
    u256 r, r2;
    int is_sm2_prime;
} field_t;

typedef struct { u256 x, y; int inf; } aff_t;  /* Montgomery coordinates */
typedef struct { u256 X, Y, Z; } jac_t;         /* Z == 0 <=> infinity */

typedef struct {
    field_t fp, fn;
    u256 a, b;
    aff_t g;
    aff_t ladder[256]; /* ladder[i] = 2^i * G, batch_point.cpp:341-350 */
} curve_t;

enum { ST_OK = 0, ST_INVALID_ARG = 1, ST_MALFORMED = 2, ST_INVALID_PEER = 3,
       ST_DEGENERATE = 4, ST_NONCE_EXHAUSTED = 5, ST_INTERNAL = 7 };

/* ------------------------------------------------------------------ ledger */
static _Thread_local uint64_t g_led[4]; /* modmul, modadd, modsub, modinv (field.hpp:19-24) */

void go_ledger_read(uint64_t out[4]) { memcpy(out, g_led, sizeof g_led); }
void go_ledger_reset(void) { memset(g_led, 0, sizeof g_led); }

/* ------------------------------------------------------------------- limbs */
static const u256 U256_ZERO = {{0}};

static int is_zero(const u256* a) {
    uint32_t acc = 0;
    for (int i = 0; i < 8; ++i) acc |= a->w[i];
    return acc == 0;
}
static int equal(const u256* a, const u256* b) { return memcmp(a, b, sizeof *a) == 0; }

/* limbs.hpp:115-122 */
static int cmp(const u256* a, const u256* b) {
    for (int i = 7; i >= 0; --i)
        if (a->w[i] != b->w[i]) return a->w[i] < b->w[i] ? -1 : 1;
    return 0;
}
/* limbs.hpp:75-85 */
static uint32_t add_c(u256* out, const u256* a, const u256* b) {
    uint64_t c = 0;
    for (int i = 0; i < 8; ++i) {
        c += (uint64_t)a->w[i] + b->w[i];
        out->w[i] = (uint32_t)c;
        c >>= 32;
    }
    return (uint32_t)c;
}
/* limbs.hpp:87-97 */
static uint32_t sub_b(u256* out, const u256* a, const u256* b) {
    uint64_t br = 0;
    for (int i = 0; i < 8; ++i) {
        uint64_t t = (uint64_t)a->w[i] - b->w[i] - br;
        out->w[i] = (uint32_t)t;
        br = (t >> 32) & 1;
    }
    return (uint32_t)br;
}
/* limbs.hpp:101-113, row-by-row schoolbook */
static void mul_wide(u512* out, const u256* a, const u256* b) {
    memset(out, 0, sizeof *out);
    for (int i = 0; i < 8; ++i) {
        uint64_t carry = 0;
        for (int j = 0; j < 8; ++j) {
            uint64_t t = (uint64_t)a->w[j] * b->w[i] + out->w[i + j] + carry;
            out->w[i + j] = (uint32_t)t;
            carry = t >> 32;
        }
        out->w[i + 8] = (uint32_t)carry;
    }
}
static unsigned bit_of(const u256* a, unsigned i) { return (a->w[i >> 5] >> (i & 31)) & 1u; }

/* limbs.cpp:5-27 */
static void from_be(u256* out, const uint8_t* p) {
    for (int i = 0; i < 8; ++i) {
        const uint8_t* s = p + 4 * (7 - i);
        out->w[i] = ((uint32_t)s[0] << 24) | ((uint32_t)s[1] << 16) | ((uint32_t)s[2] << 8) | s[3];
    }
}
static void to_be(uint8_t* p, const u256* a) {
    for (int i = 0; i < 8; ++i) {
        uint8_t* d = p + 4 * (7 - i);
        d[0] = (uint8_t)(a->w[i] >> 24); d[1] = (uint8_t)(a->w[i] >> 16);
        d[2] = (uint8_t)(a->w[i] >> 8);  d[3] = (uint8_t)a->w[i];
    }
}

/* ------------------------------------------------------------------- field */
/* field.cpp:24-35 */
static void add_mod_raw(u256* out, const u256* a, const u256* b, const field_t* f) {
    u256 s;
    uint32_t c = add_c(&s, a, b);
    if (c || cmp(&s, &f->q) >= 0) sub_b(out, &s, &f->q);
    else *out = s;
}
static void sub_mod_raw(u256* out, const u256* a, const u256* b, const field_t* f) {
    u256 d;
    if (sub_b(&d, a, b)) add_c(out, &d, &f->q);
    else *out = d;
}

/* field.cpp:50-78 -- word-serial SOS with a 17-word accumulator */
static void reduce_generic(u256* out, const u512* c, const field_t* f) {
    uint32_t acc[17];
    memcpy(acc, c->w, 64);
    acc[16] = 0;
    for (int i = 0; i < 8; ++i) {
        uint32_t m = acc[i] * f->q_inv;
        uint64_t carry = 0;
        for (int j = 0; j < 8; ++j) {
            uint64_t t = (uint64_t)m * f->q.w[j] + acc[i + j] + carry;
            acc[i + j] = (uint32_t)t;
            carry = t >> 32;
        }
        for (int k = i + 8; carry && k < 17; ++k) {
            uint64_t t = (uint64_t)acc[k] + carry;
            acc[k] = (uint32_t)t;
            carry = t >> 32;
        }
    }
    u256 hi;
    memcpy(hi.w, acc + 8, 32);
    if (acc[16] || cmp(&hi, &f->q) >= 0) sub_b(&hi, &hi, &f->q);
    *out = hi;
}

/* field.cpp:88-128 -- SCA-256: q_inv == 1, so m_j is the word itself and
 * m*q = m*2^256 - m*2^224 - m*2^96 + m*2^64 - m is signed single-word deltas.
 * Two words are eliminated per pass with one signed-carry sweep. */
static void reduce_sm2(u256* out, const u512* c, const field_t* f) {
    int64_t acc[17];
    for (int i = 0; i < 16; ++i) acc[i] = c->w[i];
    acc[16] = 0;
    for (int k = 0; k < 4; ++k) {
        const int j = 2 * k;
        const int64_t m0 = acc[j], m1 = acc[j + 1], d = m1 - m0;
        int64_t carry = 0;
        for (int w = j + 2; w < 17; ++w) {
            int64_t delta = 0;
            switch (w - j) {           /* field.cpp:101-112 */
                case 2: delta = m0; break;
                case 3: delta = d; break;
                case 4: delta = -m1; break;
                case 7: delta = -m0; break;
                case 8: delta = -d; break;
                case 9: delta = m1; break;
                default: break;
            }
            int64_t t = acc[w] + delta + carry;
            acc[w] = t & 0xFFFFFFFFll;
            carry = t >> 32; /* arithmetic shift: borrows stay signed */
        }
        acc[j] = acc[j + 1] = 0;
    }
    u256 hi;
    for (int i = 0; i < 8; ++i) hi.w[i] = (uint32_t)acc[8 + i];
    if (acc[16] || cmp(&hi, &f->q) >= 0) sub_b(&hi, &hi, &f->q);
    *out = hi;
}

/* field.cpp:130-141 */
static void mul_raw(u256* out, const u256* a, const u256* b, const field_t* f) {
    u512 t;
    mul_wide(&t, a, b);
    if (f->is_sm2_prime) reduce_sm2(out, &t, f);
    else reduce_generic(out, &t, f);
}
/* ledgered ops, field.cpp:205-227 */
static void fe_mul(u256* out, const u256* a, const u256* b, const field_t* f) {
    g_led[0]++;
    mul_raw(out, a, b, f);
}
static void fe_add(u256* out, const u256* a, const u256* b, const field_t* f) {
    g_led[1]++;
    add_mod_raw(out, a, b, f);
}
static void fe_sub(u256* out, const u256* a, const u256* b, const field_t* f) {
    g_led[2]++;
    sub_mod_raw(out, a, b, f);
}
/* field.cpp:144-151 + 239-246: a^(q-2), MSB-first, one tally of modinv.
 * Returns 0 on success, -1 for a == 0 (the reference throws). */
static int fe_inv(u256* out, const u256* a, const field_t* f) {
    if (is_zero(a)) return -1;
    u256 e = f->q, two = {{2}}, r = f->r;
    sub_b(&e, &e, &two);
    g_led[3]++;
    for (int i = 255; i >= 0; --i) {
        mul_raw(&r, &r, &r, f);
        if (bit_of(&e, (unsigned)i)) mul_raw(&r, &r, a, f);
    }
    *out = r;
    return 0;
}
/* field.cpp:194-203 (unledgered) */
static int to_mont(u256* out, const u256* a, const field_t* f) {
    if (cmp(a, &f->q) >= 0) return -1;
    mul_raw(out, a, &f->r2, f);
    return 0;
}
static void from_mont(u256* out, const u256* a, const field_t* f) {
    u256 one = {{1}};
    mul_raw(out, a, &one, f);
}

/* field.cpp:159-179 */
static void field_make(field_t* f, const u256* q, int is_sm2) {
    f->q = *q;
    uint32_t x = q->w[0];
    for (int i = 0; i < 5; ++i) x *= 2u - q->w[0] * x; /* Newton: q^-1 mod 2^32 */
    f->q_inv = ~x + 1u;
    u256 t = {{1}};
    for (int i = 0; i < 256; ++i) add_mod_raw(&t, &t, &t, f);
    f->r = t;
    for (int i = 0; i < 256; ++i) add_mod_raw(&t, &t, &t, f);
    f->r2 = t;
    f->is_sm2_prime = is_sm2;
}

/* ------------------------------------------------------------------- curve */
static aff_t aff_inf(void) { aff_t p; memset(&p, 0, sizeof p); p.inf = 1; return p; }

/* curve.cpp:62-70 */
static int on_curve(const curve_t* c, const aff_t* p) {
    if (p->inf) return 1;
    const field_t* f = &c->fp;
    u256 lhs, x2, rhs, ax;
    fe_mul(&lhs, &p->y, &p->y, f);
    fe_mul(&x2, &p->x, &p->x, f);
    fe_mul(&rhs, &x2, &p->x, f);
    fe_mul(&ax, &c->a, &p->x, f);
    fe_add(&rhs, &rhs, &ax, f);
    fe_add(&rhs, &rhs, &c->b, f);
    return equal(&lhs, &rhs);
}

/* shared tail of the chord and tangent formulas */
static void finish_lambda(aff_t* out, const u256* lam, const u256* x1, const u256* x2,
                          const u256* y1, const field_t* f) {
    u256 xr, t;
    fe_mul(&xr, lam, lam, f);
    fe_sub(&xr, &xr, x1, f);
    fe_sub(&xr, &xr, x2, f);
    fe_sub(&t, x1, &xr, f);
    fe_mul(&t, lam, &t, f);
    fe_sub(&out->y, &t, y1, f);
    out->x = xr;
    out->inf = 0;
}
/* curve.cpp:90-100 */
static aff_t pdbl_affine(const curve_t* c, const aff_t* p) {
    const field_t* f = &c->fp;
    if (p->inf || is_zero(&p->y)) return aff_inf();
    u256 x2, num, den, inv, lam;
    fe_mul(&x2, &p->x, &p->x, f);
    fe_add(&num, &x2, &x2, f);
    fe_add(&num, &num, &x2, f);
    fe_add(&num, &num, &c->a, f);
    fe_add(&den, &p->y, &p->y, f);
    fe_inv(&inv, &den, f);
    fe_mul(&lam, &num, &inv, f);
    aff_t r;
    /* the reference forms 2x by an addition and subtracts it once */
    u256 two_x, xr, t;
    fe_add(&two_x, &p->x, &p->x, f);
    fe_mul(&xr, &lam, &lam, f);
    fe_sub(&xr, &xr, &two_x, f);
    fe_sub(&t, &p->x, &xr, f);
    fe_mul(&t, &lam, &t, f);
    fe_sub(&r.y, &t, &p->y, f);
    r.x = xr;
    r.inf = 0;
    return r;
}

static jac_t jac_inf(const curve_t* c) {
    jac_t j;
    j.X = c->fp.r; j.Y = c->fp.r; j.Z = U256_ZERO;
    return j;
}
static jac_t lift(const curve_t* c, const aff_t* p) { /* curve.cpp:102-107 */
    if (p->inf) return jac_inf(c);
    jac_t j;
    j.X = p->x; j.Y = p->y; j.Z = c->fp.r;
    return j;
}
/* curve.cpp:109-127 */
static jac_t pdbl_jac(const curve_t* c, const jac_t* p) {
    const field_t* f = &c->fp;
    if (is_zero(&p->Z) || is_zero(&p->Y)) return jac_inf(c);
    u256 yy, yy2, s, s4, c4, c8, xx, zz, zz2, m, az, x3, y3, yz, t;
    fe_mul(&yy, &p->Y, &p->Y, f);
    fe_add(&yy2, &yy, &yy, f);
    fe_mul(&s, &p->X, &yy2, f);
    fe_add(&s4, &s, &s, f);
    fe_mul(&c4, &yy2, &yy2, f);
    fe_add(&c8, &c4, &c4, f);
    fe_mul(&xx, &p->X, &p->X, f);
    fe_mul(&zz, &p->Z, &p->Z, f);
    fe_mul(&zz2, &zz, &zz, f);
    fe_add(&m, &xx, &xx, f);
    fe_add(&m, &m, &xx, f);
    fe_mul(&az, &c->a, &zz2, f);
    fe_add(&m, &m, &az, f);
    fe_mul(&x3, &m, &m, f);
    fe_sub(&x3, &x3, &s4, f);
    fe_sub(&x3, &x3, &s4, f);
    fe_sub(&t, &s4, &x3, f);
    fe_mul(&y3, &m, &t, f);
    fe_sub(&y3, &y3, &c8, f);
    fe_mul(&yz, &p->Y, &p->Z, f);
    jac_t r;
    r.X = x3; r.Y = y3;
    fe_add(&r.Z, &yz, &yz, f);
    return r;
}
/* curve.cpp:129-167 */
static jac_t padd_jac(const curve_t* c, const jac_t* p, const jac_t* t) {
    const field_t* f = &c->fp;
    if (is_zero(&p->Z)) return *t;
    if (is_zero(&t->Z)) return *p;
    u256 u1, u2, s1, s2, z1z1, z2z2, tmp;
    int mixed = equal(&t->Z, &f->r);
    fe_mul(&z1z1, &p->Z, &p->Z, f);
    if (mixed) {
        u1 = p->X;
        fe_mul(&u2, &t->X, &z1z1, f);
        s1 = p->Y;
        fe_mul(&tmp, &z1z1, &p->Z, f);
        fe_mul(&s2, &t->Y, &tmp, f);
    } else {
        fe_mul(&z2z2, &t->Z, &t->Z, f);
        fe_mul(&u1, &p->X, &z2z2, f);
        fe_mul(&u2, &t->X, &z1z1, f);
        fe_mul(&tmp, &z2z2, &t->Z, f);
        fe_mul(&s1, &p->Y, &tmp, f);
        fe_mul(&tmp, &z1z1, &p->Z, f);
        fe_mul(&s2, &t->Y, &tmp, f);
    }
    if (equal(&u1, &u2)) {
        if (equal(&s1, &s2)) return pdbl_jac(c, p);
        return jac_inf(c);
    }
    u256 h, r, hh, hhh, v, x3, y3, z3, w;
    fe_sub(&h, &u2, &u1, f);
    fe_sub(&r, &s2, &s1, f);
    fe_mul(&hh, &h, &h, f);
    fe_mul(&hhh, &hh, &h, f);
    fe_mul(&v, &u1, &hh, f);
    fe_mul(&x3, &r, &r, f);
    fe_sub(&x3, &x3, &hhh, f);
    fe_sub(&x3, &x3, &v, f);
    fe_sub(&x3, &x3, &v, f);
    fe_sub(&w, &v, &x3, f);
    fe_mul(&y3, &r, &w, f);
    fe_mul(&w, &s1, &hhh, f);
    fe_sub(&y3, &y3, &w, f);
    if (mixed) fe_mul(&z3, &p->Z, &h, f);
    else {
        fe_mul(&z3, &p->Z, &t->Z, f);
        fe_mul(&z3, &z3, &h, f);
    }
    jac_t o;
    o.X = x3; o.Y = y3; o.Z = z3;
    return o;
}
/* curve.cpp:169-174 */
static aff_t jac_to_aff(const curve_t* c, const jac_t* p) {
    const field_t* f = &c->fp;
    if (is_zero(&p->Z)) return aff_inf();
    u256 zi, zi2, zi3;
    fe_inv(&zi, &p->Z, f);
    fe_mul(&zi2, &zi, &zi, f);
    aff_t r;
    fe_mul(&r.x, &p->X, &zi2, f);
    fe_mul(&zi3, &zi2, &zi, f);
    fe_mul(&r.y, &p->Y, &zi3, f);
    r.inf = 0;
    return r;
}
/* curve.cpp:176-185 -- LSB-first double-and-add, the ground truth */
static aff_t pmul_serial(const curve_t* c, const u256* s, const aff_t* p) {
    aff_t inf = aff_inf();
    jac_t acc = lift(c, &inf), run = lift(c, p);
    for (unsigned i = 0; i < 256; ++i) {
        if (bit_of(s, i)) acc = padd_jac(c, &acc, &run);
        run = pdbl_jac(c, &run);
    }
    return jac_to_aff(c, &acc);
}

/* curve.cpp:192-217 */
static void encode_point(uint8_t* out65, const curve_t* c, const aff_t* p) {
    u256 t;
    out65[0] = 0x04;
    from_mont(&t, &p->x, &c->fp); to_be(out65 + 1, &t);
    from_mont(&t, &p->y, &c->fp); to_be(out65 + 33, &t);
}
static int decode_point(aff_t* out, const curve_t* c, const uint8_t* in65) {
    if (in65[0] != 0x04) return -1;
    u256 x, y;
    from_be(&x, in65 + 1);
    from_be(&y, in65 + 33);
    if (cmp(&x, &c->fp.q) >= 0 || cmp(&y, &c->fp.q) >= 0) return -1;
    to_mont(&out->x, &x, &c->fp);
    to_mont(&out->y, &y, &c->fp);
    out->inf = 0;
    return on_curve(c, out) ? 0 : -1;
}

/* ------------------------------------------------------------ curve tables */
static u256 from_hex_words(const uint32_t msw_first[8]) {
    u256 r;
    for (int i = 0; i < 8; ++i) r.w[7 - i] = msw_first[i];
    return r;
}

static curve_t* g_curves[2];

static curve_t* build_curve(int id) {
    static const uint32_t sm2_p[8] = {0xFFFFFFFEu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0x00000000u, 0xFFFFFFFFu, 0xFFFFFFFFu};
    static const uint32_t sm2_n[8] = {0xFFFFFFFEu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0x7203DF6Bu, 0x21C6052Bu, 0x53BBF409u, 0x39D54123u};
    static const uint32_t sm2_b[8] = {0x28E9FA9Eu, 0x9D9F5E34u, 0x4D5A9E4Bu, 0xCF6509A7u, 0xF39789F5u, 0x15AB8F92u, 0xDDBCBD41u, 0x4D940E93u};
    static const uint32_t sm2_gx[8] = {0x32C4AE2Cu, 0x1F198119u, 0x5F990446u, 0x6A39C994u, 0x8FE30BBFu, 0xF2660BE1u, 0x715A4589u, 0x334C74C7u};
    static const uint32_t sm2_gy[8] = {0xBC3736A2u, 0xF4F6779Cu, 0x59BDCEE3u, 0x6B692153u, 0xD0A9877Cu, 0xC62A4740u, 0x02DF32E5u, 0x2139F0A0u};
    static const uint32_t k1_p[8] = {0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFEu, 0xFFFFFC2Fu};
    static const uint32_t k1_n[8] = {0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFEu, 0xBAAEDCE6u, 0xAF48A03Bu, 0xBFD25E8Cu, 0xD0364141u};
    static const uint32_t k1_b[8] = {0, 0, 0, 0, 0, 0, 0, 7};
    static const uint32_t k1_gx[8] = {0x79BE667Eu, 0xF9DCBBACu, 0x55A06295u, 0xCE870B07u, 0x029BFCDBu, 0x2DCE28D9u, 0x59F2815Bu, 0x16F81798u};
    static const uint32_t k1_gy[8] = {0x483ADA77u, 0x26A3C465u, 0x5DA4FBFCu, 0x0E1108A8u, 0xFD17B448u, 0xA6855419u, 0x9C47D08Fu, 0xFB10D4B8u};

    curve_t* c = (curve_t*)calloc(1, sizeof *c);
    u256 p = from_hex_words(id == 0 ? sm2_p : k1_p);
    u256 n = from_hex_words(id == 0 ? sm2_n : k1_n);
    field_make(&c->fp, &p, id == 0); /* is_sm2_prime selects the add/sub-only route */
    field_make(&c->fn, &n, 0);
    u256 a_plain = U256_ZERO, three = {{3}};
    if (id == 0) sub_b(&a_plain, &p, &three); /* a = q - 3, curve.cpp:12-13 */
    u256 b_plain = from_hex_words(id == 0 ? sm2_b : k1_b);
    u256 gx = from_hex_words(id == 0 ? sm2_gx : k1_gx);
    u256 gy = from_hex_words(id == 0 ? sm2_gy : k1_gy);
    to_mont(&c->a, &a_plain, &c->fp);
    to_mont(&c->b, &b_plain, &c->fp);
    to_mont(&c->g.x, &gx, &c->fp);
    to_mont(&c->g.y, &gy, &c->fp);
    c->g.inf = 0;
    /* batch_point.cpp:341-350: 255 serial affine doublings */
    c->ladder[0] = c->g;
    for (int i = 1; i < 256; ++i) c->ladder[i] = pdbl_affine(c, &c->ladder[i - 1]);
    return c;
}

static const curve_t* curve_of(int id) {
    if (id < 0 || id > 1) return NULL;
    if (!g_curves[id]) {
        uint64_t saved[4];
        memcpy(saved, g_led, sizeof saved); /* table building is not ledgered (capi.cpp:101) */
        g_curves[id] = build_curve(id);
        memcpy(g_led, saved, sizeof saved);
    }
    return g_curves[id];
}

/* ----------------------------------------------------- column-major access */
static u256 col_get(const uint32_t* cols, size_t n, size_t i) {
    u256 v;
    for (size_t k = 0; k < 8; ++k) v.w[k] = cols[k * n + i];
    return v;
}
static void col_set(uint32_t* cols, size_t n, size_t i, const u256* v) {
    for (size_t k = 0; k < 8; ++k) cols[k * n + i] = v->w[k];
}
static aff_t pt_get(const uint32_t* x, const uint32_t* y, const uint8_t* inf, size_t n, size_t i) {
    aff_t p;
    p.x = col_get(x, n, i);
    p.y = col_get(y, n, i);
    p.inf = inf ? (inf[i] != 0) : 0;
    return p;
}
/* batch_point.cpp:41-47: infinity coordinates normalised to zero */
static void pt_set(uint32_t* x, uint32_t* y, uint8_t* inf, size_t n, size_t i, const aff_t* p) {
    col_set(x, n, i, p->inf ? &U256_ZERO : &p->x);
    col_set(y, n, i, p->inf ? &U256_ZERO : &p->y);
    inf[i] = p->inf ? 1 : 0;
}

/* ------------------------------------------------------- lanes / inversion */
/* batch_invert.cpp:8-29: balanced contiguous ranges */
static size_t plan_lanes(size_t total, size_t lanes) {
    if (total == 0) return 0;
    if (lanes == 0) lanes = 1;
    return lanes > total ? total : lanes;
}
static void plan_range(size_t total, size_t lanes, size_t lane, size_t* begin, size_t* end) {
    size_t base = total / lanes, rem = total % lanes;
    *begin = lane * base + (lane < rem ? lane : rem);
    *end = *begin + base + (lane < rem ? 1 : 0);
}
/* BatchConfig::effective_lanes with a single worker (protocol.cpp:88-93) */
static size_t effective_lanes(size_t n, size_t lanes) {
    if (lanes) return lanes;
    return 4 < n ? 4 : (n == 0 ? 1 : n);
}

/* batch_invert.cpp:49-68: one inversion for all lane tails */
static int gather_apply(u256* inv, const u256* tails, size_t L, const field_t* f) {
    u256* grand = (u256*)malloc(L * sizeof(u256));
    grand[0] = tails[0];
    for (size_t i = 1; i < L; ++i) fe_mul(&grand[i], &grand[i - 1], &tails[i], f);
    u256 running;
    if (fe_inv(&running, &grand[L - 1], f)) { free(grand); return -1; }
    for (size_t i = L; i-- > 1;) {
        fe_mul(&inv[i], &running, &grand[i - 1], f);
        fe_mul(&running, &running, &tails[i], f);
    }
    inv[0] = running;
    free(grand);
    return 0;
}

/* batch_invert.cpp:31-47, :70-89, :91-126 */
static int batch_invert(u256* out, const u256* in, size_t n, const field_t* f, size_t lanes) {
    if (n == 0) return 0;
    const size_t L = plan_lanes(n, lanes);
    u256* prefix = (u256*)malloc(n * sizeof(u256));
    u256* tails = (u256*)malloc(L * sizeof(u256));
    u256* tinv = (u256*)malloc(L * sizeof(u256));
    for (size_t lane = 0; lane < L; ++lane) {
        size_t b, e;
        plan_range(n, L, lane, &b, &e);
        for (size_t k = b; k < e; ++k) {
            const u256* factor = is_zero(&in[k]) ? &f->r : &in[k]; /* zero masked to one */
            if (k == b) prefix[k] = *factor;
            else fe_mul(&prefix[k], &prefix[k - 1], factor, f);
        }
        tails[lane] = prefix[e - 1];
    }
    int rc = gather_apply(tinv, tails, L, f);
    for (size_t lane = 0; rc == 0 && lane < L; ++lane) {
        size_t b, e;
        plan_range(n, L, lane, &b, &e);
        u256 running = tinv[lane];
        for (size_t k = e; k-- > b + 1;) {
            fe_mul(&out[k], &running, &prefix[k - 1], f);
            fe_mul(&running, &running, is_zero(&in[k]) ? &f->r : &in[k], f);
        }
        out[b] = running;
        for (size_t k = b; k < e; ++k)
            if (is_zero(&in[k])) out[k] = U256_ZERO;
    }
    free(prefix); free(tails); free(tinv);
    return rc;
}

/* --------------------------------------------------------- batch_padd/pdbl */
enum { K_GENERIC, K_TANGENT, K_INFINITY, K_COPY_LEFT, K_COPY_RIGHT }; /* batch_point.cpp:10-16 */

static aff_t tangent_finish(const curve_t* c, const aff_t* a, const u256* inv) {
    const field_t* f = &c->fp;
    u256 x2, num, lam;
    fe_mul(&x2, &a->x, &a->x, f);
    fe_add(&num, &x2, &x2, f);
    fe_add(&num, &num, &x2, f);
    fe_add(&num, &num, &c->a, f);
    fe_mul(&lam, &num, inv, f);
    aff_t r;
    finish_lambda(&r, &lam, &a->x, &a->x, &a->y, f);
    return r;
}
static aff_t chord_finish(const curve_t* c, const aff_t* a, const aff_t* b, const u256* inv) {
    const field_t* f = &c->fp;
    u256 num, lam;
    fe_sub(&num, &a->y, &b->y, f);
    fe_mul(&lam, &num, inv, f);
    aff_t r;
    finish_lambda(&r, &lam, &a->x, &b->x, &a->y, f);
    return r;
}

/* batch_point.cpp:68-173 */
static int batch_padd(const curve_t* c, size_t n, const aff_t* p, const aff_t* t, aff_t* out,
                      size_t lanes) {
    if (n == 0) return 0;
    const field_t* f = &c->fp;
    const size_t L = plan_lanes(n, lanes);
    u256* prefix = (u256*)malloc(n * sizeof(u256));
    u256* denom = (u256*)malloc(n * sizeof(u256));
    uint8_t* kind = (uint8_t*)malloc(n);
    u256* tails = (u256*)malloc(L * sizeof(u256));
    u256* tinv = (u256*)malloc(L * sizeof(u256));
    for (size_t lane = 0; lane < L; ++lane) {
        size_t b, e;
        plan_range(n, L, lane, &b, &e);
        for (size_t i = b; i < e; ++i) {
            u256 d = f->r;
            if (p[i].inf && t[i].inf) kind[i] = K_INFINITY;
            else if (p[i].inf) kind[i] = K_COPY_RIGHT;
            else if (t[i].inf) kind[i] = K_COPY_LEFT;
            else if (equal(&p[i].x, &t[i].x)) {
                if (equal(&p[i].y, &t[i].y) && !is_zero(&p[i].y)) {
                    kind[i] = K_TANGENT;
                    fe_add(&d, &p[i].y, &p[i].y, f);
                } else kind[i] = K_INFINITY;
            } else {
                kind[i] = K_GENERIC;
                fe_sub(&d, &p[i].x, &t[i].x, f);
            }
            denom[i] = d;
            if (i == b) prefix[i] = d;
            else fe_mul(&prefix[i], &prefix[i - 1], &d, f);
        }
        tails[lane] = prefix[e - 1];
    }
    int rc = gather_apply(tinv, tails, L, f);
    for (size_t lane = 0; rc == 0 && lane < L; ++lane) {
        size_t b, e;
        plan_range(n, L, lane, &b, &e);
        u256 running = tinv[lane];
        for (size_t i = e; i-- > b;) {
            u256 inv = running;
            if (i > b) {
                fe_mul(&inv, &running, &prefix[i - 1], f);
                fe_mul(&running, &running, &denom[i], f);
            }
            switch (kind[i]) {
                case K_GENERIC: out[i] = chord_finish(c, &p[i], &t[i], &inv); break;
                case K_TANGENT: out[i] = tangent_finish(c, &p[i], &inv); break;
                case K_INFINITY: out[i] = aff_inf(); break;
                case K_COPY_LEFT: out[i] = p[i]; break;
                default: out[i] = t[i]; break;
            }
        }
    }
    free(prefix); free(denom); free(kind); free(tails); free(tinv);
    return rc;
}

/* batch_point.cpp:175-231 */
static int batch_pdbl(const curve_t* c, size_t n, const aff_t* p, aff_t* out, size_t lanes) {
    if (n == 0) return 0;
    const field_t* f = &c->fp;
    const size_t L = plan_lanes(n, lanes);
    u256* prefix = (u256*)malloc(n * sizeof(u256));
    u256* denom = (u256*)malloc(n * sizeof(u256));
    u256* tails = (u256*)malloc(L * sizeof(u256));
    u256* tinv = (u256*)malloc(L * sizeof(u256));
    for (size_t lane = 0; lane < L; ++lane) {
        size_t b, e;
        plan_range(n, L, lane, &b, &e);
        for (size_t i = b; i < e; ++i) {
            int degenerate = p[i].inf || is_zero(&p[i].y);
            if (degenerate) denom[i] = f->r;
            else fe_add(&denom[i], &p[i].y, &p[i].y, f);
            if (i == b) prefix[i] = denom[i];
            else fe_mul(&prefix[i], &prefix[i - 1], &denom[i], f);
        }
        tails[lane] = prefix[e - 1];
    }
    int rc = gather_apply(tinv, tails, L, f);
    for (size_t lane = 0; rc == 0 && lane < L; ++lane) {
        size_t b, e;
        plan_range(n, L, lane, &b, &e);
        u256 running = tinv[lane];
        for (size_t i = e; i-- > b;) {
            u256 inv = running;
            if (i > b) {
                fe_mul(&inv, &running, &prefix[i - 1], f);
                fe_mul(&running, &running, &denom[i], f);
            }
            if (p[i].inf || is_zero(&p[i].y)) out[i] = aff_inf();
            else out[i] = tangent_finish(c, &p[i], &inv);
        }
    }
    free(prefix); free(denom); free(tails); free(tinv);
    return rc;
}

/* ------------------------------------------------- fused multiplication */
/* batch_point.cpp:358-426 -- 256 conditional additions of ladder[bit] */
static int batch_fpmul(const curve_t* c, size_t n, const u256* scalars, aff_t* q, size_t lanes) {
    for (size_t j = 0; j < n; ++j) q[j] = aff_inf();
    if (n == 0) return 0;
    const field_t* f = &c->fp;
    const size_t L = plan_lanes(n, lanes);
    u256* partial = (u256*)malloc(n * sizeof(u256)); /* FusedScratch: one element per pair */
    u256* tails = (u256*)malloc(L * sizeof(u256));
    u256* tinv = (u256*)malloc(L * sizeof(u256));
    int rc = 0;
    for (unsigned bit = 0; bit < 256 && rc == 0; ++bit) {
        const aff_t* g = &c->ladder[bit];
        for (size_t lane = 0; lane < L; ++lane) {
            size_t b, e;
            plan_range(n, L, lane, &b, &e);
            u256 acc = f->r;
            for (size_t j = b; j < e; ++j) {
                u256 t2;
                fe_sub(&t2, &g->x, &q[j].x, f);
                int mask = q[j].inf || is_zero(&t2);
                partial[j] = acc;
                fe_mul(&acc, &acc, mask ? &f->r : &t2, f);
            }
            tails[lane] = acc;
        }
        rc = gather_apply(tinv, tails, L, f);
        for (size_t lane = 0; rc == 0 && lane < L; ++lane) {
            size_t b, e;
            plan_range(n, L, lane, &b, &e);
            u256 inv_acc = tinv[lane];
            for (size_t j = e; j-- > b;) {
                u256 t2, t2_inv, num, lam;
                fe_sub(&t2, &g->x, &q[j].x, f);
                int mask = q[j].inf || is_zero(&t2);
                fe_mul(&t2_inv, &inv_acc, &partial[j], f);
                fe_mul(&inv_acc, &inv_acc, mask ? &f->r : &t2, f);
                fe_sub(&num, &g->y, &q[j].y, f);
                fe_mul(&lam, &num, &t2_inv, f);
                aff_t r;
                finish_lambda(&r, &lam, &g->x, &q[j].x, &g->y, f);
                if (q[j].inf) r = *g;
                else if (is_zero(&t2)) r = aff_inf(); /* only an inverse pair can collide (:414-417) */
                if (bit_of(&scalars[j], bit)) {
                    if (r.inf) r = aff_inf();
                    q[j] = r;
                }
            }
        }
    }
    free(partial); free(tails); free(tinv);
    return rc;
}

/* batch_point.cpp:236-339 -- Alg. 3: per bit, doubling and addition
 * denominators of every lane share one running product / one inversion */
static int batch_upmul(const curve_t* c, size_t n, const u256* scalars, const aff_t* points,
                       aff_t* q, size_t lanes) {
    for (size_t j = 0; j < n; ++j) q[j] = aff_inf();
    if (n == 0) return 0;
    const field_t* f = &c->fp;
    const size_t L = plan_lanes(n, lanes);
    aff_t* p = (aff_t*)malloc(n * sizeof(aff_t));
    for (size_t j = 0; j < n; ++j) { /* buffer copy normalises infinity coords to 0 */
        p[j] = points[j];
        if (p[j].inf) p[j] = aff_inf();
    }
    u256* partial = (u256*)malloc(n * sizeof(u256));
    u256* tails = (u256*)malloc(L * sizeof(u256));
    u256* tinv = (u256*)malloc(L * sizeof(u256));
    int rc = 0;
    for (unsigned bit = 0; bit < 256 && rc == 0; ++bit) {
        for (size_t lane = 0; lane < L; ++lane) {
            size_t b, e;
            plan_range(n, L, lane, &b, &e);
            u256 acc = f->r;
            for (size_t j = b; j < e; ++j) {
                u256 t1, t2;
                fe_add(&t1, &p[j].y, &p[j].y, f);
                fe_sub(&t2, &p[j].x, &q[j].x, f);
                int mask1 = p[j].inf || is_zero(&t1);
                int mask2 = p[j].inf || q[j].inf || is_zero(&t2);
                partial[j] = acc;
                fe_mul(&acc, &acc, mask1 ? &f->r : &t1, f);
                fe_mul(&acc, &acc, mask2 ? &f->r : &t2, f);
            }
            tails[lane] = acc;
        }
        rc = gather_apply(tinv, tails, L, f);
        for (size_t lane = 0; rc == 0 && lane < L; ++lane) {
            size_t b, e;
            plan_range(n, L, lane, &b, &e);
            u256 inv_acc = tinv[lane];
            for (size_t j = e; j-- > b;) {
                const aff_t pp = p[j], qq = q[j];
                u256 t1, t2, t1p, t2_inv, t1_inv, num, lam_a, px2, num2, lam_d;
                fe_add(&t1, &pp.y, &pp.y, f);
                int mask1 = pp.inf || is_zero(&t1);
                const u256* t1m = mask1 ? &f->r : &t1;
                fe_mul(&t1p, t1m, &partial[j], f);      /* recomputed partial product */
                fe_mul(&t2_inv, &inv_acc, &t1p, f);
                fe_sub(&num, &pp.y, &qq.y, f);          /* chord R = P + Q */
                fe_mul(&lam_a, &num, &t2_inv, f);
                aff_t r;
                finish_lambda(&r, &lam_a, &pp.x, &qq.x, &pp.y, f);
                fe_sub(&t2, &pp.x, &qq.x, f);
                int mask2 = pp.inf || qq.inf || is_zero(&t2);
                fe_mul(&inv_acc, &inv_acc, mask2 ? &f->r : &t2, f);
                fe_mul(&t1_inv, &inv_acc, &partial[j], f);
                fe_mul(&px2, &pp.x, &pp.x, f);          /* tangent P' = 2P */
                fe_add(&num2, &px2, &px2, f);
                fe_add(&num2, &num2, &px2, f);
                fe_add(&num2, &num2, &c->a, f);
                fe_mul(&lam_d, &num2, &t1_inv, f);
                aff_t dbl;
                finish_lambda(&dbl, &lam_d, &pp.x, &pp.x, &pp.y, f);
                fe_mul(&inv_acc, &inv_acc, t1m, f);

                if (qq.inf) r = pp;
                else if (pp.inf) r = qq;
                else if (is_zero(&t2)) r = equal(&pp.y, &qq.y) ? dbl : aff_inf();
                if (!pp.inf) p[j] = mask1 ? aff_inf() : dbl;
                if (bit_of(&scalars[j], bit)) q[j] = r.inf ? aff_inf() : r;
            }
        }
    }
    free(p); free(partial); free(tails); free(tinv);
    return rc;
}

/* ---------------------------------------------------------------- protocol */
static uint64_t splitmix(uint64_t* x) { /* protocol.cpp:13-19 */
    *x += 0x9E3779B97F4A7C15ull;
    uint64_t z = *x;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
/* protocol.cpp:22-34 + :67-75, with n a parameter */
static u256 nonce_scalar(const curve_t* c, uint64_t seed, uint64_t stream, uint32_t attempt) {
    uint64_t state = seed;
    (void)splitmix(&state);
    state ^= 0xA3EC647659359ACDull * (stream + 1);
    (void)splitmix(&state);
    state ^= 0xC2B2AE3D27D4EB4Full * ((uint64_t)attempt + 1);
    for (;;) {
        u256 raw;
        for (int i = 0; i < 8; i += 2) {
            uint64_t v = splitmix(&state);
            raw.w[i] = (uint32_t)v;
            raw.w[i + 1] = (uint32_t)(v >> 32);
        }
        if (!is_zero(&raw) && cmp(&raw, &c->fn.q) < 0) return raw;
    }
}
static u256 reduce_once(const u256* v, const u256* n) { /* curve.cpp:22-27 */
    u256 r = *v;
    if (cmp(v, n) >= 0) sub_b(&r, v, n);
    return r;
}
static int in_range(const u256* v, const u256* n) { return !is_zero(v) && cmp(v, n) < 0; }

/* protocol.cpp:106-168 on parsed inputs */
static int sign_batch(const curve_t* c, size_t n, const u256* es, const u256* ds,
                      uint64_t seed, uint64_t lane_base, u256* rs, u256* ss, int* status,
                      size_t lanes_cfg) {
    const field_t* nf = &c->fn;
    size_t* pending = (size_t*)malloc((n ? n : 1) * sizeof(size_t));
    size_t* retry = (size_t*)malloc((n ? n : 1) * sizeof(size_t));
    size_t m = n;
    for (size_t i = 0; i < n; ++i) { pending[i] = i; status[i] = ST_OK; }
    int rc = 0;
    for (uint32_t attempt = 0; attempt < 8 && m > 0 && rc == 0; ++attempt) {
        u256* ks = (u256*)malloc(m * sizeof(u256));
        u256* km = (u256*)malloc(m * sizeof(u256));
        u256* kinv = (u256*)malloc(m * sizeof(u256));
        aff_t* rp = (aff_t*)malloc(m * sizeof(aff_t));
        for (size_t i = 0; i < m; ++i) ks[i] = nonce_scalar(c, seed, lane_base + pending[i], attempt);
        size_t lanes = effective_lanes(m, lanes_cfg);
        rc = batch_fpmul(c, m, ks, rp, lanes);
        for (size_t i = 0; i < m; ++i) to_mont(&km[i], &ks[i], nf);
        if (rc == 0) rc = batch_invert(kinv, km, m, nf, lanes);
        size_t nretry = 0;
        for (size_t i = 0; rc == 0 && i < m; ++i) {
            size_t lane = pending[i];
            if (rp[i].inf) { retry[nretry++] = lane; continue; }
            u256 x, r, e_m, r_m, d_m, t, s;
            from_mont(&x, &rp[i].x, &c->fp);
            r = reduce_once(&x, &nf->q); /* q < 2n: one conditional subtraction */
            if (is_zero(&r)) { retry[nretry++] = lane; continue; }
            to_mont(&e_m, &es[lane], nf);
            to_mont(&r_m, &r, nf);
            to_mont(&d_m, &ds[lane], nf);
            fe_mul(&t, &r_m, &d_m, nf);
            fe_add(&t, &e_m, &t, nf);
            fe_mul(&t, &kinv[i], &t, nf);
            from_mont(&s, &t, nf);
            if (is_zero(&s)) { retry[nretry++] = lane; continue; }
            rs[lane] = r;
            ss[lane] = s;
        }
        memcpy(pending, retry, nretry * sizeof(size_t));
        m = nretry;
        free(ks); free(km); free(kinv); free(rp);
    }
    for (size_t i = 0; i < m; ++i) status[pending[i]] = ST_NONCE_EXHAUSTED;
    free(pending); free(retry);
    return rc;
}

/* ------------------------------------------------------------- C entries */
uint32_t go_field_params(int curve, int which, uint32_t* q, uint32_t* r, uint32_t* r2) {
    const curve_t* c = curve_of(curve);
    const field_t* f = which == 0 ? &c->fp : &c->fn;
    memcpy(q, f->q.w, 32); memcpy(r, f->r.w, 32); memcpy(r2, f->r2.w, 32);
    return f->q_inv;
}
void go_curve_params(int curve, uint32_t* a, uint32_t* b, uint32_t* gx, uint32_t* gy) {
    const curve_t* c = curve_of(curve);
    memcpy(a, c->a.w, 32); memcpy(b, c->b.w, 32);
    memcpy(gx, c->g.x.w, 32); memcpy(gy, c->g.y.w, 32);
}

int go_field_op(int curve, int which, int op, size_t n, const uint32_t* a, const uint32_t* b,
                uint32_t* out) {
    const curve_t* c = curve_of(curve);
    if (!c) return ST_INVALID_ARG;
    const field_t* f = which == 0 ? &c->fp : &c->fn;
    for (size_t i = 0; i < n; ++i) {
        u256 x = col_get(a, n, i), y = b ? col_get(b, n, i) : U256_ZERO, r = U256_ZERO;
        switch (op) {
            case 0: fe_mul(&r, &x, &y, f); break;
            case 1: fe_add(&r, &x, &y, f); break;
            case 2: fe_sub(&r, &x, &y, f); break;
            case 3: if (to_mont(&r, &x, f)) return ST_MALFORMED; break;
            case 4: from_mont(&r, &x, f); break;
            case 5: if (!is_zero(&x)) fe_inv(&r, &x, f); break;
            default: return ST_INVALID_ARG;
        }
        col_set(out, n, i, &r);
    }
    return ST_OK;
}

int go_mont_reduce(int curve, int which, int sm2_route, size_t n, const uint32_t* c16,
                   uint32_t* out) {
    const curve_t* c = curve_of(curve);
    if (!c) return ST_INVALID_ARG;
    const field_t* f = which == 0 ? &c->fp : &c->fn;
    for (size_t i = 0; i < n; ++i) {
        u512 t;
        u256 r;
        for (size_t k = 0; k < 16; ++k) t.w[k] = c16[k * n + i];
        if (sm2_route) reduce_sm2(&r, &t, f); else reduce_generic(&r, &t, f);
        col_set(out, n, i, &r);
    }
    return ST_OK;
}

int go_batch_invert(int curve, int which, size_t n, const uint32_t* in, uint32_t* out,
                    size_t lanes) {
    const curve_t* c = curve_of(curve);
    if (!c) return ST_INVALID_ARG;
    const field_t* f = which == 0 ? &c->fp : &c->fn;
    u256* a = (u256*)malloc((n ? n : 1) * sizeof(u256));
    u256* o = (u256*)malloc((n ? n : 1) * sizeof(u256));
    for (size_t i = 0; i < n; ++i) a[i] = col_get(in, n, i);
    int rc = batch_invert(o, a, n, f, effective_lanes(n, lanes));
    for (size_t i = 0; i < n; ++i) col_set(out, n, i, &o[i]);
    free(a); free(o);
    return rc ? ST_INTERNAL : ST_OK;
}

static aff_t* load_pts(const uint32_t* x, const uint32_t* y, const uint8_t* inf, size_t n) {
    aff_t* p = (aff_t*)malloc((n ? n : 1) * sizeof(aff_t));
    for (size_t i = 0; i < n; ++i) p[i] = pt_get(x, y, inf, n, i);
    return p;
}
static void store_pts(const aff_t* p, uint32_t* x, uint32_t* y, uint8_t* inf, size_t n) {
    for (size_t i = 0; i < n; ++i) pt_set(x, y, inf, n, i, &p[i]);
}
static u256* load_scalars(const uint32_t* s, size_t n) {
    u256* v = (u256*)malloc((n ? n : 1) * sizeof(u256));
    for (size_t i = 0; i < n; ++i) v[i] = col_get(s, n, i);
    return v;
}

int go_batch_padd(int curve, size_t n, const uint32_t* px, const uint32_t* py,
                  const uint8_t* pinf, const uint32_t* tx, const uint32_t* ty,
                  const uint8_t* tinf, uint32_t* ox, uint32_t* oy, uint8_t* oinf, size_t lanes) {
    const curve_t* c = curve_of(curve);
    if (!c) return ST_INVALID_ARG;
    aff_t *p = load_pts(px, py, pinf, n), *t = load_pts(tx, ty, tinf, n);
    aff_t* o = (aff_t*)malloc((n ? n : 1) * sizeof(aff_t));
    int rc = batch_padd(c, n, p, t, o, effective_lanes(n, lanes));
    store_pts(o, ox, oy, oinf, n);
    free(p); free(t); free(o);
    return rc ? ST_INTERNAL : ST_OK;
}
int go_batch_pdbl(int curve, size_t n, const uint32_t* px, const uint32_t* py,
                  const uint8_t* pinf, uint32_t* ox, uint32_t* oy, uint8_t* oinf, size_t lanes) {
    const curve_t* c = curve_of(curve);
    if (!c) return ST_INVALID_ARG;
    aff_t* p = load_pts(px, py, pinf, n);
    aff_t* o = (aff_t*)malloc((n ? n : 1) * sizeof(aff_t));
    int rc = batch_pdbl(c, n, p, o, effective_lanes(n, lanes));
    store_pts(o, ox, oy, oinf, n);
    free(p); free(o);
    return rc ? ST_INTERNAL : ST_OK;
}
int go_batch_fpmul(int curve, size_t n, const uint32_t* scalars, uint32_t* ox, uint32_t* oy,
                   uint8_t* oinf, size_t lanes) {
    const curve_t* c = curve_of(curve);
    if (!c) return ST_INVALID_ARG;
    u256* s = load_scalars(scalars, n);
    aff_t* o = (aff_t*)malloc((n ? n : 1) * sizeof(aff_t));
    int rc = batch_fpmul(c, n, s, o, effective_lanes(n, lanes));
    store_pts(o, ox, oy, oinf, n);
    free(s); free(o);
    return rc ? ST_INTERNAL : ST_OK;
}
int go_batch_upmul(int curve, size_t n, const uint32_t* scalars, const uint32_t* px,
                   const uint32_t* py, const uint8_t* pinf, uint32_t* ox, uint32_t* oy,
                   uint8_t* oinf, size_t lanes) {
    const curve_t* c = curve_of(curve);
    if (!c) return ST_INVALID_ARG;
    u256* s = load_scalars(scalars, n);
    aff_t* p = load_pts(px, py, pinf, n);
    aff_t* o = (aff_t*)malloc((n ? n : 1) * sizeof(aff_t));
    int rc = batch_upmul(c, n, s, p, o, effective_lanes(n, lanes));
    store_pts(o, ox, oy, oinf, n);
    free(s); free(p); free(o);
    return rc ? ST_INTERNAL : ST_OK;
}
int go_pmul_serial(int curve, size_t n, const uint32_t* scalars, const uint32_t* px,
                   const uint32_t* py, const uint8_t* pinf, uint32_t* ox, uint32_t* oy,
                   uint8_t* oinf) {
    const curve_t* c = curve_of(curve);
    if (!c) return ST_INVALID_ARG;
    for (size_t i = 0; i < n; ++i) {
        u256 s = col_get(scalars, n, i);
        aff_t p = pt_get(px, py, pinf, n, i);
        aff_t r = pmul_serial(c, &s, &p);
        pt_set(ox, oy, oinf, n, i, &r);
    }
    return ST_OK;
}
int go_msm(int curve, size_t n, const uint32_t* scalars, const uint32_t* px, const uint32_t* py,
           const uint8_t* pinf, uint32_t* ox, uint32_t* oy, uint8_t* oinf) {
    const curve_t* c = curve_of(curve);
    if (!c) return ST_INVALID_ARG;
    aff_t inf = aff_inf();
    jac_t acc = lift(c, &inf);
    for (size_t i = 0; i < n; ++i) {
        u256 s = col_get(scalars, n, i);
        aff_t p = pt_get(px, py, pinf, n, i);
        jac_t run = lift(c, &p);
        for (unsigned b = 0; b < 256; ++b) {
            if (bit_of(&s, b)) acc = padd_jac(c, &acc, &run);
            run = pdbl_jac(c, &run);
        }
    }
    aff_t r = jac_to_aff(c, &acc);
    pt_set(ox, oy, oinf, 1, 0, &r);
    return ST_OK;
}

void go_nonce(int curve, uint64_t seed, uint64_t stream, uint32_t attempt, uint8_t* out32) {
    u256 k = nonce_scalar(curve_of(curve), seed, stream, attempt);
    to_be(out32, &k);
}

/* capi.cpp:145-169 */
int go_keygen(int curve, uint64_t seed, uint64_t lane_base, size_t count, uint8_t* secrets,
              uint8_t* publics, size_t lanes) {
    const curve_t* c = curve_of(curve);
    if (!c || (count && (!secrets || !publics))) return ST_INVALID_ARG;
    u256* ds = (u256*)malloc((count ? count : 1) * sizeof(u256));
    aff_t* pubs = (aff_t*)malloc((count ? count : 1) * sizeof(aff_t));
    for (size_t i = 0; i < count; ++i) ds[i] = nonce_scalar(c, seed, lane_base + i, 0);
    int rc = batch_fpmul(c, count, ds, pubs, effective_lanes(count, lanes));
    for (size_t i = 0; i < count; ++i) {
        to_be(secrets + 32 * i, &ds[i]);
        encode_point(publics + 65 * i, c, &pubs[i]);
    }
    free(ds); free(pubs);
    return rc ? ST_INTERNAL : ST_OK;
}

/* capi.cpp:171-197 */
int go_sign(int curve, size_t count, const uint8_t* digests, const uint8_t* secrets,
            uint64_t nonce_seed, uint64_t lane_base, uint8_t* signatures, int32_t* lane_status,
            size_t lanes) {
    const curve_t* c = curve_of(curve);
    if (!c || (count && (!digests || !secrets || !signatures))) return ST_INVALID_ARG;
    size_t cap = count ? count : 1;
    u256 *es = (u256*)malloc(cap * sizeof(u256)), *ds = (u256*)malloc(cap * sizeof(u256));
    u256 *rs = (u256*)calloc(cap, sizeof(u256)), *ss = (u256*)calloc(cap, sizeof(u256));
    int* st = (int*)calloc(cap, sizeof(int));
    int rc = ST_OK;
    for (size_t i = 0; i < count && rc == ST_OK; ++i) {
        u256 raw;
        from_be(&raw, digests + 32 * i);
        es[i] = reduce_once(&raw, &c->fn.q);           /* digests are reduced */
        from_be(&ds[i], secrets + 32 * i);
        if (!in_range(&ds[i], &c->fn.q)) rc = ST_MALFORMED; /* secrets are checked */
    }
    if (rc == ST_OK) {
        if (sign_batch(c, count, es, ds, nonce_seed, lane_base, rs, ss, st, lanes)) rc = ST_INTERNAL;
    }
    if (rc == ST_OK) {
        int first = ST_OK;
        memset(signatures, 0, 64 * count);
        for (size_t i = 0; i < count; ++i) {
            if (lane_status) lane_status[i] = st[i];
            if (st[i] != ST_OK) { if (first == ST_OK) first = st[i]; continue; }
            to_be(signatures + 64 * i, &rs[i]);
            to_be(signatures + 64 * i + 32, &ss[i]);
        }
        rc = lane_status ? ST_OK : first; /* capi.cpp:64-73 */
    }
    free(es); free(ds); free(rs); free(ss); free(st);
    return rc;
}

/* capi.cpp:199-228 + protocol.cpp:170-222 */
int go_verify(int curve, size_t count, const uint8_t* digests, const uint8_t* publics,
              const uint8_t* signatures, uint8_t* results, size_t lanes_cfg) {
    const curve_t* c = curve_of(curve);
    if (!c || (count && (!digests || !publics || !signatures || !results))) return ST_INVALID_ARG;
    const field_t* nf = &c->fn;
    size_t cap = count ? count : 1;
    size_t* live = (size_t*)malloc(cap * sizeof(size_t));
    u256 *es = (u256*)malloc(cap * sizeof(u256)), *rs = (u256*)malloc(cap * sizeof(u256));
    u256 *sm = (u256*)malloc(cap * sizeof(u256)), *w = (u256*)malloc(cap * sizeof(u256));
    u256 *u1 = (u256*)malloc(cap * sizeof(u256)), *u2 = (u256*)malloc(cap * sizeof(u256));
    aff_t *pubs = (aff_t*)malloc(cap * sizeof(aff_t)), *A = (aff_t*)malloc(cap * sizeof(aff_t));
    aff_t *B = (aff_t*)malloc(cap * sizeof(aff_t)), *R = (aff_t*)malloc(cap * sizeof(aff_t));
    size_t m = 0;
    memset(results, 0, count);
    for (size_t i = 0; i < count; ++i) {
        u256 r, s, raw;
        aff_t q;
        from_be(&r, signatures + 64 * i);
        from_be(&s, signatures + 64 * i + 32);
        if (decode_point(&q, c, publics + 65 * i)) continue;     /* lane fails, not the call */
        if (!in_range(&r, &nf->q) || !in_range(&s, &nf->q)) continue;
        from_be(&raw, digests + 32 * i);
        live[m] = i;
        es[m] = reduce_once(&raw, &nf->q);
        rs[m] = r;
        to_mont(&sm[m], &s, nf);
        pubs[m] = q;
        ++m;
    }
    int rc = 0;
    if (m) {
        size_t lanes = effective_lanes(m, lanes_cfg);
        rc = batch_invert(w, sm, m, nf, lanes);
        for (size_t i = 0; i < m; ++i) {
            u256 e_m, r_m, t;
            to_mont(&e_m, &es[i], nf);
            to_mont(&r_m, &rs[i], nf);
            fe_mul(&t, &e_m, &w[i], nf); from_mont(&u1[i], &t, nf);
            fe_mul(&t, &r_m, &w[i], nf); from_mont(&u2[i], &t, nf);
        }
        if (!rc) rc = batch_fpmul(c, m, u1, A, lanes);
        if (!rc) rc = batch_upmul(c, m, u2, pubs, B, lanes);
        if (!rc) rc = batch_padd(c, m, A, B, R, lanes);
        for (size_t i = 0; !rc && i < m; ++i) {
            if (R[i].inf) continue;
            u256 x, xr;
            from_mont(&x, &R[i].x, &c->fp);
            xr = reduce_once(&x, &nf->q);
            results[live[i]] = equal(&xr, &rs[i]) ? 1 : 0;
        }
    }
    free(live); free(es); free(rs); free(sm); free(w); free(u1); free(u2);
    free(pubs); free(A); free(B); free(R);
    return rc ? ST_INTERNAL : ST_OK;
}

/* capi.cpp:230-261 + protocol.cpp:224-263 */
int go_ecdh(int curve, size_t count, const uint8_t* secrets, const uint8_t* peers,
            uint8_t* shared, int32_t* lane_status, size_t lanes_cfg) {
    const curve_t* c = curve_of(curve);
    if (!c || (count && (!secrets || !peers || !shared))) return ST_INVALID_ARG;
    size_t cap = count ? count : 1;
    size_t* live = (size_t*)malloc(cap * sizeof(size_t));
    u256* ds = (u256*)malloc(cap * sizeof(u256));
    aff_t *ps = (aff_t*)malloc(cap * sizeof(aff_t)), *prod = (aff_t*)malloc(cap * sizeof(aff_t));
    int* st = (int*)calloc(cap, sizeof(int));
    size_t m = 0;
    int rc = ST_OK;
    for (size_t i = 0; i < count; ++i) {
        u256 d;
        from_be(&d, secrets + 32 * i);
        if (cmp(&d, &c->fn.q) >= 0) { rc = ST_MALFORMED; break; } /* Scalar::checked, zero allowed */
        aff_t p;
        if (decode_point(&p, c, peers + 65 * i)) { st[i] = ST_INVALID_PEER; continue; }
        live[m] = i; ds[m] = d; ps[m] = p; ++m;
    }
    if (rc == ST_OK) {
        memset(shared, 0, 32 * count);
        if (m && batch_upmul(c, m, ds, ps, prod, effective_lanes(m, lanes_cfg))) rc = ST_INTERNAL;
    }
    if (rc == ST_OK) {
        for (size_t i = 0; i < m; ++i) {
            if (prod[i].inf) { st[live[i]] = ST_DEGENERATE; continue; }
            u256 x;
            from_mont(&x, &prod[i].x, &c->fp);
            to_be(shared + 32 * live[i], &x);
        }
        int first = ST_OK;
        for (size_t i = 0; i < count; ++i) {
            if (lane_status) lane_status[i] = st[i];
            if (st[i] && first == ST_OK) first = st[i];
        }
        rc = lane_status ? ST_OK : first;
    }
    free(live); free(ds); free(ps); free(prod); free(st);
    return rc;
}
