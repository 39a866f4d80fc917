/*
 * oracle.c -- plain, slow, obviously-correct CPU oracle for Z_p-RAID
 *             (arxiv cs/0611109, "An approach to RAID-6 based on cyclic groups").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load this library.  The product path
 * (paper_cs_0611109_b200/) never links, imports or calls it, and this file shares
 * no code, header, table or constant generator with the CUDA path.
 *
 * Representation (deliberately naive): a ring element of R_p = F2[x]/(1+x+...+x^{p-1})
 * is an array of n = p-1 bytes, one byte per bit, bits[j] = coefficient of x^j
 * (Sec. 4.5: "x + x" multiplies by x, "x < 0" tests x_15,
 * so bit j of the machine word is the coefficient of x^j).
 *
 * Strip layout (reading R2): a strip of `bytes` bytes is an LSB-first
 * bit stream, stream bit b = (byte[b>>3] >> (b&7)) & 1; word w = stream bits
 * [w*n, (w+1)*n), zero-extended past 8*bytes.  W = ceil(8*bytes/n) words.  P and Q
 * hold W*n bits, i.e. parity_bytes = ceil(W*n/8) bytes, zero past W*n.
 *
 * Every function cites the passage it follows.  Nothing here is blocked, fused or
 * reordered beyond what the cited definition or algorithm states.
 *
 * Parity pins: see tests/test_oracle_pins.py (all functions are pinned; the byte
 * layout for n != 16 is a convention, pinned by hand-derived vectors only -- see
 * DESIGN.md "parity of the layout").
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_MAX_N 256 /* p <= 257 */

/* ---------------------------------------------------------------- basics */

/* n = p - 1 word bits (Lemma 26.1: S_N is (N-1)x(N-1)). */
int oracle_n(int p) { return p - 1; }

/* W = ceil(8*bytes / n) words per strip (reading R5). */
size_t oracle_word_count(int p, size_t bytes) {
    size_t n = (size_t)(p - 1);
    return (8 * bytes + n - 1) / n;
}

/* parity strip length = ceil(W*n / 8) bytes (reading R5). */
size_t oracle_parity_bytes(int p, size_t bytes) {
    size_t n = (size_t)(p - 1);
    return (oracle_word_count(p, bytes) * n + 7) / 8;
}

/* odd prime 3 <= p <= 257 ("Given that N is an odd prime"). */
int oracle_valid_p(int p) {
    if (p < 3 || p > 257 || (p % 2) == 0) return 0;
    for (int d = 3; d * d <= p; d += 2)
        if (p % d == 0) return 0;
    return 1;
}

/* Read word w of a strip (LSB-first stream, zero past 8*len bits). */
static void get_word(const uint8_t *strip, size_t len, size_t w, int n, uint8_t *bits) {
    for (int j = 0; j < n; j++) {
        size_t b = w * (size_t)n + (size_t)j;
        size_t byte = b >> 3;
        bits[j] = (byte < len) ? (uint8_t)((strip[byte] >> (b & 7)) & 1u) : 0u;
    }
}

/* Write word w into a strip buffer of `len` bytes (bits past 8*len are dropped). */
static void put_word(uint8_t *strip, size_t len, size_t w, int n, const uint8_t *bits) {
    for (int j = 0; j < n; j++) {
        size_t b = w * (size_t)n + (size_t)j;
        size_t byte = b >> 3;
        if (byte >= len) continue;
        uint8_t m = (uint8_t)(1u << (b & 7));
        if (bits[j]) strip[byte] |= m;
        else strip[byte] &= (uint8_t)~m;
    }
}

static void xor_into(uint8_t *acc, const uint8_t *v, int n) {
    for (int j = 0; j < n; j++) acc[j] ^= v[j];
}

/* ------------------------------------------------- multiplication by x = S_p */

/*
 * One Sylvester step y = S_p a (Lemma 26.1 matrix; the Z_17 instance
 * PAPER.md:1043-1075, Sec. 4.5):  y_0 = a_{n-1},  y_j = a_{j-1} XOR a_{n-1}  (1 <= j < n).
 * This is the paper's "y = (x + x) ^ ((x < 0) ? 0xffff : 0)" for n bits.
 */
void oracle_mul_x(int p, const uint8_t *a, uint8_t *y) {
    int n = p - 1;
    uint8_t top = a[n - 1];
    uint8_t tmp[ORACLE_MAX_N];
    tmp[0] = top;
    for (int j = 1; j < n; j++) tmp[j] = (uint8_t)(a[j - 1] ^ top);
    memcpy(y, tmp, (size_t)n);
}

/* y = x^k a: k single Sylvester steps (k reduced mod p, since S_p^p = Id, Lemma 26.1(i)). */
void oracle_mul_xk(int p, int k, const uint8_t *a, uint8_t *y) {
    int n = p - 1;
    uint8_t t[ORACLE_MAX_N];
    memcpy(t, a, (size_t)n);
    k %= p;
    if (k < 0) k += p;
    for (int s = 0; s < k; s++) oracle_mul_x(p, t, t);
    memcpy(y, t, (size_t)n);
}

/* ----------------------------------------------- GF(2) matrices (tier A) */

/* Explicit Sylvester matrix S_p, row-major n*n bytes:
 * row 0 = (0 ... 0 1), row r = e_{r-1} + e_{n-1} for r >= 1. */
void oracle_sylvester(int p, uint8_t *S) {
    int n = p - 1;
    memset(S, 0, (size_t)n * (size_t)n);
    S[0 * n + (n - 1)] = 1;
    for (int r = 1; r < n; r++) {
        S[r * n + (r - 1)] = 1;
        S[r * n + (n - 1)] = 1;
    }
}

/* C = A B over GF(2), n x n row-major. */
void oracle_gf2_matmul(int n, const uint8_t *A, const uint8_t *B, uint8_t *C) {
    uint8_t *T = (uint8_t *)calloc((size_t)n * (size_t)n, 1);
    for (int r = 0; r < n; r++)
        for (int c = 0; c < n; c++) {
            uint8_t s = 0;
            for (int k = 0; k < n; k++) s ^= (uint8_t)(A[r * n + k] & B[k * n + c]);
            T[r * n + c] = s;
        }
    memcpy(C, T, (size_t)n * (size_t)n);
    free(T);
}

/* y = M v over GF(2). */
void oracle_gf2_matvec(int n, const uint8_t *M, const uint8_t *v, uint8_t *y) {
    uint8_t t[ORACLE_MAX_N];
    for (int r = 0; r < n; r++) {
        uint8_t s = 0;
        for (int c = 0; c < n; c++) s ^= (uint8_t)(M[r * n + c] & v[c]);
        t[r] = s;
    }
    memcpy(y, t, (size_t)n);
}

/* S_p^k by repeated GF(2) matrix multiplication of the explicit matrix (k >= 0). */
void oracle_sylvester_power(int p, int k, uint8_t *out) {
    int n = p - 1;
    uint8_t *S = (uint8_t *)malloc((size_t)n * (size_t)n);
    oracle_sylvester(p, S);
    memset(out, 0, (size_t)n * (size_t)n);
    for (int i = 0; i < n; i++) out[i * n + i] = 1;
    for (int s = 0; s < k; s++) oracle_gf2_matmul(n, S, out, out);
    free(S);
}

/*
 * Gauss-Jordan inverse over GF(2) (the method SPEC.md:74 names for mat_inverse).
 * Returns 1 and writes Minv if M is invertible, else returns 0.
 */
int oracle_gf2_inverse(int n, const uint8_t *M, uint8_t *Minv) {
    int w = 2 * n;
    uint8_t *A = (uint8_t *)calloc((size_t)n * (size_t)w, 1);
    for (int r = 0; r < n; r++) {
        memcpy(A + (size_t)r * w, M + (size_t)r * n, (size_t)n);
        A[(size_t)r * w + n + r] = 1;
    }
    for (int col = 0; col < n; col++) {
        int piv = -1;
        for (int r = col; r < n; r++)
            if (A[(size_t)r * w + col]) { piv = r; break; }
        if (piv < 0) { free(A); return 0; }
        if (piv != col)
            for (int c = 0; c < w; c++) {
                uint8_t t = A[(size_t)piv * w + c];
                A[(size_t)piv * w + c] = A[(size_t)col * w + c];
                A[(size_t)col * w + c] = t;
            }
        for (int r = 0; r < n; r++)
            if (r != col && A[(size_t)r * w + col])
                for (int c = 0; c < w; c++) A[(size_t)r * w + c] ^= A[(size_t)col * w + c];
    }
    for (int r = 0; r < n; r++) memcpy(Minv + (size_t)r * n, A + (size_t)r * w + n, (size_t)n);
    free(A);
    return 1;
}

/* ------------------------------------------------------------------ encode */

/*
 * Encode one stripe (Eq. (znparity), Corollary 24.4; 0-based as in
 * Eq. (rsparity), disk i <-> g^i):
 *     P = D_0 + D_1 + ... + D_{N-1},     Q = D_0 + g D_1 + ... + g^{N-1} D_{N-1},
 * with g = S_p.  Q is evaluated by Horner's rule exactly as the paper's syndrome loop
 * (Sec. 4.2: Q = D_0 + g(D_1 + g(... + g D_{N-1}))), one
 * multiplication by g per step (Sec. 4.5).
 * strips: N host pointers of `bytes` bytes.  P, Q: parity_bytes each.
 * Returns 0 on success, -1 on invalid arguments.
 */
int oracle_encode(int p, int N, const uint8_t *const *strips, size_t bytes, uint8_t *P, uint8_t *Q) {
    if (!oracle_valid_p(p) || N < 1 || N > p) return -1;
    int n = p - 1;
    size_t W = oracle_word_count(p, bytes);
    size_t pb = oracle_parity_bytes(p, bytes);
    uint8_t d[ORACLE_MAX_N], pw[ORACLE_MAX_N], qw[ORACLE_MAX_N];
    memset(P, 0, pb);
    memset(Q, 0, pb);
    for (size_t w = 0; w < W; w++) {
        memset(pw, 0, (size_t)n);
        for (int i = 0; i < N; i++) {            /* P = sum D_i */
            get_word(strips[i], bytes, w, n, d);
            xor_into(pw, d, n);
        }
        get_word(strips[N - 1], bytes, w, n, qw); /* Q = D_{N-1} */
        for (int i = N - 2; i >= 0; i--) {        /* Q = D_i + g Q */
            oracle_mul_x(p, qw, qw);
            get_word(strips[i], bytes, w, n, d);
            xor_into(qw, d, n);
        }
        put_word(P, pb, w, n, pw);
        put_word(Q, pb, w, n, qw);
    }
    return 0;
}

/*
 * Tier-A encode, definition level: Q = sum_i S_p^i d_i by explicit matrix powers and
 * bit mat-vec (the parity check matrix of Corollary 24.4).
 * Small inputs only (cost O(N n^3 + W N n^2)).
 */
int oracle_encode_matrix(int p, int N, const uint8_t *const *strips, size_t bytes, uint8_t *P, uint8_t *Q) {
    if (!oracle_valid_p(p) || N < 1 || N > p) return -1;
    int n = p - 1;
    size_t W = oracle_word_count(p, bytes);
    size_t pb = oracle_parity_bytes(p, bytes);
    uint8_t *pw_mats = (uint8_t *)malloc((size_t)N * n * n);
    for (int i = 0; i < N; i++) oracle_sylvester_power(p, i, pw_mats + (size_t)i * n * n);
    uint8_t d[ORACLE_MAX_N], t[ORACLE_MAX_N], pw[ORACLE_MAX_N], qw[ORACLE_MAX_N];
    memset(P, 0, pb);
    memset(Q, 0, pb);
    for (size_t w = 0; w < W; w++) {
        memset(pw, 0, (size_t)n);
        memset(qw, 0, (size_t)n);
        for (int i = 0; i < N; i++) {
            get_word(strips[i], bytes, w, n, d);
            xor_into(pw, d, n);
            oracle_gf2_matvec(n, pw_mats + (size_t)i * n * n, d, t);
            xor_into(qw, t, n);
        }
        put_word(P, pb, w, n, pw);
        put_word(Q, pb, w, n, qw);
    }
    free(pw_mats);
    return 0;
}

/* ----------------------------------------------------------------- recover */

/*
 * Double-erasure recovery (Lemma 23.2 proof; Sec. 4.3 and 4.6,
 * PAPER.md:965-992 and 1124-1160).  Strip indices: 0..N-1 data, N = P, N+1 = Q
 * (reading R4).  strips: N+2 host pointers; data strips are `bytes` long,
 * P and Q parity_bytes long.  The two lost strips are outputs (their contents are
 * never read); all others are inputs.  lost_i/lost_j in either order.
 * Returns 0 on success, -1 on invalid arguments, -2 if a required inverse is singular
 * (never happens for a valid p: Theorem 24.1 / Lemma 26.1(ii)).
 */
int oracle_recover(int p, int N, int lost_i, int lost_j, uint8_t *const *strips, size_t bytes) {
    if (!oracle_valid_p(p) || N < 1 || N > p) return -1;
    if (lost_i == lost_j || lost_i < 0 || lost_j < 0 || lost_i >= N + 2 || lost_j >= N + 2) return -1;
    int x = lost_i < lost_j ? lost_i : lost_j; /* canonical x < y (reading R8) */
    int y = lost_i < lost_j ? lost_j : lost_i;
    int n = p - 1;
    size_t W = oracle_word_count(p, bytes);
    size_t pb = oracle_parity_bytes(p, bytes);
    const int iP = N, iQ = N + 1;
    uint8_t d[ORACLE_MAX_N], acc[ORACLE_MAX_N], pw[ORACLE_MAX_N], qw[ORACLE_MAX_N];

    if (x == iP && y == iQ) {
        /* (P, Q) lost: "compute parity bits in terms of information bits". */
        return oracle_encode(p, N, (const uint8_t *const *)strips, bytes, strips[iP], strips[iQ]);
    }

    if (y == iQ) {
        /* (d_j, Q) lost, j = x < N: d_j = P + sum_{k != j} d_k "as in RAID-5", then Q from the
         * second equation. */
        int j = x;
        for (size_t w = 0; w < W; w++) {
            get_word(strips[iP], pb, w, n, acc);
            for (int k = 0; k < N; k++) {
                if (k == j) continue;
                get_word(strips[k], bytes, w, n, d);
                xor_into(acc, d, n);
            }
            put_word(strips[j], bytes, w, n, acc);
        }
        uint8_t *Pd = (uint8_t *)malloc(pb);
        int rc = oracle_encode(p, N, (const uint8_t *const *)strips, bytes, Pd, strips[iQ]);
        free(Pd);
        return rc;
    }

    if (y == iP) {
        /* (d_j, P) lost: d_j = g_j^{-1}(Q + sum_{k != j} g_k d_k) with
         * g_j = S^j and g^{-j} = g^{p-j}; then P = sum_k d_k. */
        int j = x;
        memset(strips[iP], 0, pb); /* parity pad bits past W*n are zero (reading R5) */
        for (size_t w = 0; w < W; w++) {
            /* Horner over the survivors with d_j taken as zero. */
            memset(qw, 0, (size_t)n);
            for (int k = N - 1; k >= 0; k--) {
                oracle_mul_x(p, qw, qw);
                if (k != j) {
                    get_word(strips[k], bytes, w, n, d);
                    xor_into(qw, d, n);
                }
            }
            get_word(strips[iQ], pb, w, n, acc);
            xor_into(acc, qw, n);                     /* Q + sum_{k!=j} g^k d_k */
            oracle_mul_xk(p, (p - j) % p, acc, acc);  /* times g^{p-j} */
            put_word(strips[j], bytes, w, n, acc);
            memset(pw, 0, (size_t)n);                 /* P = sum_k d_k */
            for (int k = 0; k < N; k++) {
                if (k == j) xor_into(pw, acc, n);
                else { get_word(strips[k], bytes, w, n, d); xor_into(pw, d, n); }
            }
            put_word(strips[iP], pb, w, n, pw);
        }
        return 0;
    }

    /* (d_x, d_y) lost, x < y < N (Sec. 4.3 / 4.6):
     *   P_xy = sum_{i != x,y} D_i,  Q_xy = sum_{i != x,y} g^i D_i          (Eq. (PQxy))
     *   dP = P + P_xy,  dQ = Q + Q_xy,  z = y - x
     *   A = (1 + g^z)^{-1},  B = g^{-x} (1 + g^z)^{-1} = g^{p-x} A
     *   D_y = A dP + B dQ,  D_x = D_y + dP.
     * A and B are computed once per pair: A by Gauss-Jordan of the
     * explicit matrix Id + S^z, B = S^{p-x} A by explicit matrix product. */
    {
        int z = y - x;
        size_t nn = (size_t)n * (size_t)n;
        uint8_t *Sz = (uint8_t *)malloc(nn), *A = (uint8_t *)malloc(nn);
        uint8_t *Sb = (uint8_t *)malloc(nn), *B = (uint8_t *)malloc(nn);
        oracle_sylvester_power(p, z, Sz);
        for (int i = 0; i < n; i++) Sz[i * n + i] ^= 1;          /* Id + S^z */
        if (!oracle_gf2_inverse(n, Sz, A)) { free(Sz); free(A); free(Sb); free(B); return -2; }
        oracle_sylvester_power(p, (p - x) % p, Sb);
        oracle_gf2_matmul(n, Sb, A, B);
        uint8_t dP[ORACLE_MAX_N], dQ[ORACLE_MAX_N], t1[ORACLE_MAX_N], t2[ORACLE_MAX_N];
        for (size_t w = 0; w < W; w++) {
            get_word(strips[iP], pb, w, n, dP);
            get_word(strips[iQ], pb, w, n, dQ);
            memset(qw, 0, (size_t)n);                 /* Q_xy by Horner, lost disks zero */
            for (int k = N - 1; k >= 0; k--) {
                oracle_mul_x(p, qw, qw);
                if (k != x && k != y) {
                    get_word(strips[k], bytes, w, n, d);
                    xor_into(qw, d, n);
                    xor_into(dP, d, n);               /* dP = P + P_xy */
                }
            }
            xor_into(dQ, qw, n);                      /* dQ = Q + Q_xy */
            oracle_gf2_matvec(n, A, dP, t1);
            oracle_gf2_matvec(n, B, dQ, t2);
            xor_into(t1, t2, n);                      /* D_y */
            put_word(strips[y], bytes, w, n, t1);
            xor_into(t1, dP, n);                      /* D_x = D_y + dP */
            put_word(strips[x], bytes, w, n, t1);
        }
        free(Sz); free(A); free(Sb); free(B);
    }
    return 0;
}

/*
 * Syndrome check of a complete stripe (both parity equations of Eq. (znparity)):
 * returns the number of words w for which P_w != sum d or Q_w != sum g^i d.
 */
int oracle_encode_ext(int p, int D, const uint8_t *const *strips, size_t bytes, uint8_t *P, uint8_t *Q);

size_t oracle_count_bad_words(int p, int N, const uint8_t *const *strips, size_t bytes) {
    if (!oracle_valid_p(p) || N < 1 || N > 2 * p - 1) return (size_t)-1;
    int n = p - 1;
    if (n < 1 || n > ORACLE_MAX_N) return (size_t)-1;
    size_t W = oracle_word_count(p, bytes);
    size_t pb = oracle_parity_bytes(p, bytes);
    uint8_t *Pc = (uint8_t *)malloc(pb), *Qc = (uint8_t *)malloc(pb);
    /* the parity equations: Eq. (znparity) for N <= p, Eq. (qext) beyond (NEXT-2) */
    if (N <= p) oracle_encode(p, N, strips, bytes, Pc, Qc);
    else if (oracle_encode_ext(p, N, strips, bytes, Pc, Qc) != 0) { free(Pc); free(Qc); return (size_t)-1; }
    uint8_t a[ORACLE_MAX_N], b[ORACLE_MAX_N];
    size_t bad = 0;
    for (size_t w = 0; w < W; w++) {
        int ok = 1;
        get_word(Pc, pb, w, n, a); get_word(strips[N], pb, w, n, b);
        if (memcmp(a, b, (size_t)n)) ok = 0;
        get_word(Qc, pb, w, n, a); get_word(strips[N + 1], pb, w, n, b);
        if (memcmp(a, b, (size_t)n)) ok = 0;
        bad += (size_t)(!ok);
    }
    free(Pc); free(Qc);
    return bad;
}

/* =====================================================================================
 * Extended Q-parity (NEXT-2): Sec. 3.3, Theorem 25.3 and Eq. (qext).
 * ===================================================================================== */

/* Polynomials over F2 as coefficient arrays (one byte per coefficient), degree tracked. */
static int poly_deg(const uint8_t *a, int len) {
    for (int i = len - 1; i >= 0; i--)
        if (a[i]) return i;
    return -1;
}

/* gcd(a, b) over F2 by Euclid's algorithm with plain long division; returns its degree. */
static int poly_gcd_deg(const uint8_t *a0, const uint8_t *b0, int len) {
    uint8_t *a = (uint8_t *)malloc((size_t)len), *b = (uint8_t *)malloc((size_t)len);
    memcpy(a, a0, (size_t)len);
    memcpy(b, b0, (size_t)len);
    for (;;) {
        int db = poly_deg(b, len);
        if (db < 0) break;
        int da;
        while ((da = poly_deg(a, len)) >= db) {      /* a = a mod b */
            for (int i = 0; i <= db; i++) a[da - db + i] ^= b[i];
        }
        uint8_t *t = a; a = b; b = t;                  /* (a, b) = (b, a mod b) */
    }
    int d = poly_deg(a, len);
    free(a); free(b);
    return d;
}

/*
 * Theorem 25.3, condition (3): for every 0 < m < p the polynomials
 * X^p + 1 and X^m + X + 1 are relatively prime.  Returns 1 if p satisfies it (so that
 * {Id, g, ..., g^{p-1}, Id+g, ..., Id+g^{p-1}} is a cone, condition (1)), else 0.
 */
int oracle_ext_condition(int p) {
    if (!oracle_valid_p(p)) return 0;
    int len = p + 1;
    uint8_t *a = (uint8_t *)calloc((size_t)len, 1), *b = (uint8_t *)calloc((size_t)len, 1);
    int ok = 1;
    for (int m = 1; m < p && ok; m++) {
        memset(a, 0, (size_t)len);
        memset(b, 0, (size_t)len);
        a[p] = 1; a[0] = 1;                 /* X^p + 1 */
        b[m] ^= 1; b[1] ^= 1; b[0] ^= 1;    /* X^m + X + 1 (m = 1 gives 1) */
        if (poly_gcd_deg(a, b, len) != 0) ok = 0;
    }
    free(a); free(b);
    return ok;
}

/* Matrix g_k of disk k in Eq. (qext): g^k for 0 <= k < p,
 * Id + g^{k-p+1} for p <= k <= 2p-2; g = S_p. */
/* Column j of S^e is S^e applied to the unit vector e_j: e single Sylvester steps. */
static void sylvester_power_cols(int p, int e, uint8_t *G) {
    int n = p - 1;
    uint8_t v[ORACLE_MAX_N];
    for (int j = 0; j < n; j++) {
        memset(v, 0, (size_t)n);
        v[j] = 1;
        oracle_mul_xk(p, e, v, v);
        for (int r = 0; r < n; r++) G[r * n + j] = v[r];
    }
}

void oracle_ext_coeff(int p, int k, uint8_t *G) {
    int n = p - 1;
    if (k < p) {
        sylvester_power_cols(p, k, G);
    } else {
        sylvester_power_cols(p, k - p + 1, G);
        for (int i = 0; i < n; i++) G[i * n + i] ^= 1;
    }
}

static int ext_args_ok(int p, int D) {
    if (!oracle_valid_p(p) || D < 1 || D > 2 * p - 1) return 0;
    if (D > p && !oracle_ext_condition(p)) return 0;
    return 1;
}

/*
 * Encode with the extended Q-parity, Eq. (qext), D data disks
 * (1 <= D <= 2p-1; D > p requires Theorem 25.3):
 *     P = sum_k d_k,   Q = sum_{k<p} g^k d_k + sum_{k=p}^{D-1} (Id + g^{k-p+1}) d_k,
 * evaluated per word with the explicit matrices g_k (bit mat-vec).  For D <= p this is the
 * basic code of Eq. (znparity).
 */
int oracle_encode_ext(int p, int D, const uint8_t *const *strips, size_t bytes, uint8_t *P, uint8_t *Q) {
    if (!ext_args_ok(p, D)) return -1;
    int n = p - 1;
    size_t nn = (size_t)n * (size_t)n;
    size_t W = oracle_word_count(p, bytes);
    size_t pb = oracle_parity_bytes(p, bytes);
    uint8_t *G = (uint8_t *)malloc((size_t)D * nn);
    for (int k = 0; k < D; k++) oracle_ext_coeff(p, k, G + (size_t)k * nn);
    uint8_t d[ORACLE_MAX_N], t[ORACLE_MAX_N], pw[ORACLE_MAX_N], qw[ORACLE_MAX_N];
    memset(P, 0, pb);
    memset(Q, 0, pb);
    for (size_t w = 0; w < W; w++) {
        memset(pw, 0, (size_t)n);
        memset(qw, 0, (size_t)n);
        for (int k = 0; k < D; k++) {
            get_word(strips[k], bytes, w, n, d);
            xor_into(pw, d, n);
            oracle_gf2_matvec(n, G + (size_t)k * nn, d, t);
            xor_into(qw, t, n);
        }
        put_word(P, pb, w, n, pw);
        put_word(Q, pb, w, n, qw);
    }
    free(G);
    return 0;
}

/*
 * Recovery for the code with coefficients g_k of Eq. (qext), following the constructive
 * proof of Lemma 23.2 literally, with 0-based indices (data 0..D-1,
 * P = D, Q = D+1) and inverses by Gauss-Jordan:
 *   (P, Q):     re-encode;
 *   (d_j, Q):   d_j = P + sum_{k!=j} d_k, then Q from the second equation;
 *   (d_j, P):   d_j = g_j^{-1}(Q + sum_{k!=j} g_k d_k), then P = sum_k d_k;
 *   (d_i, d_j): d_j = (g_i + g_j)^{-1}(g_i P + Q + sum_{k!=i,j} (g_k + g_i) d_k),
 *               then d_i from the first equation, d_i = P + sum_{k!=i} d_k.
 * Returns 0, -1 (bad arguments) or -2 (a required matrix is singular).
 */
int oracle_recover_ext(int p, int D, int lost_i, int lost_j, uint8_t *const *strips, size_t bytes) {
    if (!ext_args_ok(p, D)) return -1;
    if (lost_i == lost_j || lost_i < 0 || lost_j < 0 || lost_i >= D + 2 || lost_j >= D + 2) return -1;
    int i = lost_i < lost_j ? lost_i : lost_j, j = lost_i < lost_j ? lost_j : lost_i;
    int n = p - 1;
    size_t nn = (size_t)n * (size_t)n;
    size_t W = oracle_word_count(p, bytes);
    size_t pb = oracle_parity_bytes(p, bytes);
    const int iP = D, iQ = D + 1;
    if (i == iP && j == iQ)
        return oracle_encode_ext(p, D, (const uint8_t *const *)strips, bytes, strips[iP], strips[iQ]);
    uint8_t *G = (uint8_t *)malloc((size_t)D * nn);
    for (int k = 0; k < D; k++) oracle_ext_coeff(p, k, G + (size_t)k * nn);
    uint8_t *A = (uint8_t *)malloc(nn), *M = (uint8_t *)malloc(nn);
    uint8_t d[ORACLE_MAX_N], t[ORACLE_MAX_N], acc[ORACLE_MAX_N], pw[ORACLE_MAX_N];
    int rc = 0;
    if (j == iQ) {                                   /* (d_i, Q) */
        for (size_t w = 0; w < W; w++) {
            get_word(strips[iP], pb, w, n, acc);
            for (int k = 0; k < D; k++) {
                if (k == i) continue;
                get_word(strips[k], bytes, w, n, d);
                xor_into(acc, d, n);
            }
            put_word(strips[i], bytes, w, n, acc);
        }
        uint8_t *Pd = (uint8_t *)malloc(pb);
        rc = oracle_encode_ext(p, D, (const uint8_t *const *)strips, bytes, Pd, strips[iQ]);
        free(Pd);
    } else if (j == iP) {                            /* (d_i, P) */
        if (!oracle_gf2_inverse(n, G + (size_t)i * nn, A)) rc = -2;
        if (rc == 0) {
            memset(strips[iP], 0, pb);
            for (size_t w = 0; w < W; w++) {
                get_word(strips[iQ], pb, w, n, acc);
                for (int k = 0; k < D; k++) {
                    if (k == i) continue;
                    get_word(strips[k], bytes, w, n, d);
                    oracle_gf2_matvec(n, G + (size_t)k * nn, d, t);
                    xor_into(acc, t, n);
                }
                oracle_gf2_matvec(n, A, acc, t);           /* d_i */
                put_word(strips[i], bytes, w, n, t);
                memcpy(pw, t, (size_t)n);
                for (int k = 0; k < D; k++) {
                    if (k == i) continue;
                    get_word(strips[k], bytes, w, n, d);
                    xor_into(pw, d, n);
                }
                put_word(strips[iP], pb, w, n, pw);
            }
        }
    } else {                                         /* (d_i, d_j), both data */
        for (size_t e = 0; e < nn; e++) M[e] = G[(size_t)i * nn + e] ^ G[(size_t)j * nn + e];
        if (!oracle_gf2_inverse(n, M, A)) rc = -2;   /* A = (g_i + g_j)^{-1} */
        uint8_t *Gs = (uint8_t *)malloc((size_t)D * nn);          /* g_k + g_i, once per pair */
        for (int k = 0; k < D; k++)
            for (size_t e = 0; e < nn; e++) Gs[(size_t)k * nn + e] = G[(size_t)k * nn + e] ^ G[(size_t)i * nn + e];
        for (size_t w = 0; rc == 0 && w < W; w++) {
            get_word(strips[iP], pb, w, n, d);
            oracle_gf2_matvec(n, G + (size_t)i * nn, d, acc);   /* g_i P */
            get_word(strips[iQ], pb, w, n, d);
            xor_into(acc, d, n);                                  /* + Q */
            for (int k = 0; k < D; k++) {
                if (k == i || k == j) continue;
                get_word(strips[k], bytes, w, n, d);
                oracle_gf2_matvec(n, Gs + (size_t)k * nn, d, t);  /* + (g_k + g_i) d_k */
                xor_into(acc, t, n);
            }
            oracle_gf2_matvec(n, A, acc, t);                      /* d_j */
            put_word(strips[j], bytes, w, n, t);
            get_word(strips[iP], pb, w, n, pw);                   /* d_i = P + sum_{k!=i} d_k */
            xor_into(pw, t, n);
            for (int k = 0; k < D; k++) {
                if (k == i || k == j) continue;
                get_word(strips[k], bytes, w, n, d);
                xor_into(pw, d, n);
            }
            put_word(strips[i], bytes, w, n, pw);
        }
        free(Gs);
    }
    free(G); free(A); free(M);
    return rc;
}

/* =====================================================================================
 * NEXT-3: the paper's comparison system, Reed-Solomon RAID-6 over GF(2^8) ("DP-RAID"),
 * Sec. 4.1-4.4: g = {02}, reduction polynomial x^8+x^4+x^3+x^2+1.
 * Bytes are field elements (bit i = coefficient of x^i).
 * ===================================================================================== */

/* Multiplication by g = {02}: y = (x << 1) ^ ((x & 0x80) ? 0x1d : 0x00). */
uint8_t oracle_rs_mul2(uint8_t x) { return (uint8_t)((uint8_t)(x << 1) ^ ((x & 0x80) ? 0x1d : 0x00)); }

/* a * b in GF(2^8): b = sum_i b_i x^i, so a*b = sum_i b_i (g^i a) -- shift and add with mul2. */
uint8_t oracle_rs_mul(uint8_t a, uint8_t b) {
    uint8_t r = 0;
    for (int i = 0; i < 8; i++) {
        if ((b >> i) & 1) r ^= a;
        a = oracle_rs_mul2(a);
    }
    return r;
}

/* g^k (k >= 0) by k multiplications by g. */
uint8_t oracle_rs_exp(int k) {
    uint8_t r = 1;
    for (int i = 0; i < k; i++) r = oracle_rs_mul2(r);
    return r;
}

/* a^{-1} by exhaustive search over the 255 nonzero field elements; 0 for a = 0. */
uint8_t oracle_rs_inv(uint8_t a) {
    for (int b = 1; b < 256; b++)
        if (oracle_rs_mul(a, (uint8_t)b) == 1) return (uint8_t)b;
    return 0;
}

/*
 * Eq. (rsparity): P = D_0 + ... + D_{N-1}, Q = D_0 + g D_1 + ... + g^{N-1} D_{N-1},
 * byte by byte, Q by Horner's rule Q = D_0 + g(D_1 + g(... + g D_{N-1})).
 * 1 <= N <= 255 (g has order 255).  All strips `bytes` long (P, Q too).
 */
int oracle_rs_encode(int N, const uint8_t *const *strips, size_t bytes, uint8_t *P, uint8_t *Q) {
    if (N < 1 || N > 255) return -1;
    for (size_t b = 0; b < bytes; b++) {
        uint8_t p = 0, q = strips[N - 1][b];
        for (int i = 0; i < N; i++) p ^= strips[i][b];
        for (int i = N - 2; i >= 0; i--) q = (uint8_t)(oracle_rs_mul2(q) ^ strips[i][b]);
        P[b] = p;
        Q[b] = q;
    }
    return 0;
}

/*
 * Two-erasure recovery (strip indices 0..N-1 data, N = P, N+1 = Q):
 *   (P, Q): re-encode;  (D_j, Q): D_j = P + sum_{k!=j} D_k, then Q;
 *   (D_j, P): D_j = g^{-j}(Q + Q_j), Q_j = sum_{k!=j} g^k D_k (Lemma 23.2), then P;
 *   (D_x, D_y): Sec. 4.3: P_xy, Q_xy with the lost disks zero,
 *     A = (1 + g^{y-x})^{-1}, B = g^{-x}(1 + g^{y-x})^{-1}, D_y = A(P + P_xy) + B(Q + Q_xy),
 *     D_x = D_y + (P + P_xy).  A and B are computed once per pair.
 */
int oracle_rs_recover(int N, int lost_i, int lost_j, uint8_t *const *strips, size_t bytes) {
    if (N < 1 || N > 255) return -1;
    if (lost_i == lost_j || lost_i < 0 || lost_j < 0 || lost_i >= N + 2 || lost_j >= N + 2) return -1;
    int x = lost_i < lost_j ? lost_i : lost_j, y = lost_i < lost_j ? lost_j : lost_i;
    const int iP = N, iQ = N + 1;
    if (x == iP && y == iQ) return oracle_rs_encode(N, (const uint8_t *const *)strips, bytes, strips[iP], strips[iQ]);
    if (y == iQ) {
        for (size_t b = 0; b < bytes; b++) {
            uint8_t v = strips[iP][b];
            for (int k = 0; k < N; k++)
                if (k != x) v ^= strips[k][b];
            strips[x][b] = v;
        }
        uint8_t *Pd = (uint8_t *)malloc(bytes ? bytes : 1);
        int rc = oracle_rs_encode(N, (const uint8_t *const *)strips, bytes, Pd, strips[iQ]);
        free(Pd);
        return rc;
    }
    if (y == iP) {
        uint8_t ginv = oracle_rs_inv(oracle_rs_exp(x));
        for (size_t b = 0; b < bytes; b++) {
            uint8_t q = strips[iQ][b];
            for (int k = 0; k < N; k++)
                if (k != x) q ^= oracle_rs_mul(oracle_rs_exp(k), strips[k][b]);
            uint8_t d = oracle_rs_mul(ginv, q);
            strips[x][b] = d;
            uint8_t p = d;
            for (int k = 0; k < N; k++)
                if (k != x) p ^= strips[k][b];
            strips[iP][b] = p;
        }
        return 0;
    }
    uint8_t A = oracle_rs_inv((uint8_t)(1 ^ oracle_rs_exp(y - x)));
    uint8_t B = oracle_rs_mul(oracle_rs_inv(oracle_rs_exp(x)), A);
    for (size_t b = 0; b < bytes; b++) {
        uint8_t dp = strips[iP][b], dq = strips[iQ][b];
        for (int k = 0; k < N; k++) {
            if (k == x || k == y) continue;
            dp ^= strips[k][b];
            dq ^= oracle_rs_mul(oracle_rs_exp(k), strips[k][b]);
        }
        uint8_t dy = (uint8_t)(oracle_rs_mul(A, dp) ^ oracle_rs_mul(B, dq));
        strips[y][b] = dy;
        strips[x][b] = (uint8_t)(dy ^ dp);
    }
    return 0;
}
