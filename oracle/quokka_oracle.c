/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle.  Never linked into, loaded by,
 * or called from the product path; only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg use it, and only as the checker.
 *
 * Plain-C restatement of the reference's (Quokka / Queen, /root/reference/proj)
 * hot-path arithmetic.  Every function keeps the reference's operation order
 * and is compiled with -ffp-contract=off, so it is BIT-EXACT against the
 * reference build (oracle/_ref/libquokka_ref.so) — tests/test_oracle.py pins
 * it that way, plus against the golden vectors in tests/golden/.
 *
 * Amplitudes are interleaved (re, im) doubles; qubit 0 is the index LSB
 * (SPEC.md:83).  Multi-qubit matrices use "first listed qubit = MSB of the
 * sub-index" (proj/include/quokka/gates.hpp:36-39).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* GateKind order of proj/include/quokka/gates.hpp:10-23. */
enum { QO_H, QO_U, QO_X, QO_CX, QO_CP, QO_SWAP, QO_RX, QO_RY, QO_RZ, QO_RZZ, QO_D, QO_UK };

typedef struct {
    int kind;
    int nq;          /* qubit count (controls first, as Gate::qubits()) */
    int q[16];
    double p[3];     /* params */
    const double* payload; /* fused kinds: interleaved 2^k (D) or 4^k (U) entries */
} qo_gate;

/* ---- coefficients: proj/src/gates.cpp:90-164 ------------------------------ */

/* 2x2 matrix, row-major interleaved m[8]  (gates.cpp:115-146). */
static void qo_mat1(const qo_gate* g, double m[8]) {
    const double s2 = 1.0 / sqrt(2.0);
    memset(m, 0, 8 * sizeof(double));
    switch (g->kind) {
    case QO_H: m[0] = s2; m[2] = s2; m[4] = s2; m[6] = -s2; break;
    case QO_X: m[2] = 1; m[4] = 1; break;
    case QO_U: {
        double th = g->p[0], ph = g->p[1], la = g->p[2];
        double c = cos(th / 2.0), s = sin(th / 2.0);
        /* gates.cpp:122-127: entries c, -e^{i la} s, e^{i ph} s, e^{i(ph+la)} c.
           std::complex * double multiplies each component. */
        m[0] = c; m[1] = 0.0;
        m[2] = -cos(la) * s; m[3] = -sin(la) * s;
        m[4] = cos(ph) * s; m[5] = sin(ph) * s;
        m[6] = cos(ph + la) * c; m[7] = sin(ph + la) * c;
        break;
    }
    case QO_RX: {
        double t = g->p[0] / 2.0, c = cos(t), s = sin(t);
        m[0] = c; m[3] = -s; m[5] = -s; m[6] = c;
        break;
    }
    case QO_RY: {
        double t = g->p[0] / 2.0, c = cos(t), s = sin(t);
        m[0] = c; m[2] = -s; m[4] = s; m[6] = c;
        break;
    }
    default: break;
    }
}

/* Diagonal entries, interleaved (gates.cpp:90-113). Returns entry count. */
static int qo_diag(const qo_gate* g, double d[8]) {
    switch (g->kind) {
    case QO_RZ: {
        double t = g->p[0] / 2.0;
        d[0] = cos(t); d[1] = -sin(t); d[2] = cos(t); d[3] = sin(t);
        return 2;
    }
    case QO_RZZ: {
        double t = g->p[0] / 2.0;
        double mr = cos(t), mi = -sin(t), pr = cos(t), pi = sin(t);
        d[0] = mr; d[1] = mi; d[2] = pr; d[3] = pi; d[4] = pr; d[5] = pi; d[6] = mr; d[7] = mi;
        return 4;
    }
    case QO_CP: {
        double t = g->p[0];
        d[0] = 1; d[1] = 0; d[2] = 1; d[3] = 0; d[4] = 1; d[5] = 0; d[6] = cos(t); d[7] = sin(t);
        return 4;
    }
    default: return 0;
    }
}

/* ---- amplitude kernels: proj/src/kernels.cpp:16-48 ------------------------ */

void qo_apply1(double* a, uint64_t n, int q, const double m[8]) {
    uint64_t step = (uint64_t)1 << q;
    for (uint64_t base = 0; base < n; base += 2 * step)
        for (uint64_t i = base; i < base + step; i++) {
            double* lo = a + 2 * i;
            double* hi = a + 2 * (i + step);
            double x = lo[0], y = lo[1], u = hi[0], v = hi[1];
            lo[0] = (x * m[0] - y * m[1]) + (u * m[2] - v * m[3]);
            lo[1] = (y * m[0] + x * m[1]) + (v * m[2] + u * m[3]);
            hi[0] = (x * m[4] - y * m[5]) + (u * m[6] - v * m[7]);
            hi[1] = (y * m[4] + x * m[5]) + (v * m[6] + u * m[7]);
        }
}

void qo_diag1(double* a, uint64_t n, int q, const double d[4]) {
    for (uint64_t i = 0; i < n; i++) {
        const double* c = d + 2 * ((i >> q) & 1);
        double x = a[2 * i], y = a[2 * i + 1];
        a[2 * i] = x * c[0] - y * c[1];
        a[2 * i + 1] = y * c[0] + x * c[1];
    }
}

void qo_diag2(double* a, uint64_t n, int qa, int qb, const double d[8]) {
    for (uint64_t i = 0; i < n; i++) {
        uint64_t e = ((i >> qa) & 1) * 2 + ((i >> qb) & 1);
        const double* c = d + 2 * e;
        double x = a[2 * i], y = a[2 * i + 1];
        a[2 * i] = x * c[0] - y * c[1];
        a[2 * i + 1] = y * c[0] + x * c[1];
    }
}

static void swap_amp(double* a, uint64_t i, uint64_t j) {
    double r = a[2 * i], m = a[2 * i + 1];
    a[2 * i] = a[2 * j]; a[2 * i + 1] = a[2 * j + 1];
    a[2 * j] = r; a[2 * j + 1] = m;
}

/* One gate over n amplitudes: proj/src/engine.cpp:189-254 (applyPrepared). */
void qo_apply_gate(double* a, uint64_t n, const qo_gate* g) {
    double m[8], d[8];
    switch (g->kind) {
    case QO_H: case QO_U: case QO_X: case QO_RX: case QO_RY:
        qo_mat1(g, m);
        qo_apply1(a, n, g->q[0], m);
        return;
    case QO_RZ:
        qo_diag(g, d);
        qo_diag1(a, n, g->q[0], d);
        return;
    case QO_CP: case QO_RZZ:
        qo_diag(g, d);
        qo_diag2(a, n, g->q[0], g->q[1], d);
        return;
    case QO_CX: { /* engine.cpp:206-209; q[0] = control */
        uint64_t A = (uint64_t)1 << g->q[0], B = (uint64_t)1 << g->q[1];
        for (uint64_t i = 0; i < n; i++)
            if ((i & A) && !(i & B)) swap_amp(a, i, i | B);
        return;
    }
    case QO_SWAP: { /* engine.cpp:210-213 */
        uint64_t A = (uint64_t)1 << g->q[0], B = (uint64_t)1 << g->q[1];
        for (uint64_t i = 0; i < n; i++)
            if ((i & A) && !(i & B)) swap_amp(a, i, i ^ A ^ B);
        return;
    }
    case QO_D: { /* engine.cpp:214-227: first target = MSB of the table index */
        int k = g->nq;
        for (uint64_t i = 0; i < n; i++) {
            uint64_t sub = 0;
            for (int j = 0; j < k; j++) sub |= ((i >> g->q[j]) & 1) << (k - 1 - j);
            double cr = g->payload[2 * sub], ci = g->payload[2 * sub + 1];
            double x = a[2 * i], y = a[2 * i + 1];
            a[2 * i] = x * cr - y * ci;
            a[2 * i + 1] = y * cr + x * ci;
        }
        return;
    }
    case QO_UK: { /* engine.cpp:228-251 + prepareGate subOff (:170-185) */
        int k = g->nq;
        uint64_t dim = (uint64_t)1 << k, qmask = 0;
        for (int j = 0; j < k; j++) qmask |= (uint64_t)1 << g->q[j];
        uint64_t* off = (uint64_t*)malloc(dim * sizeof(uint64_t));
        double* tmp = (double*)malloc(2 * dim * sizeof(double));
        double* res = (double*)malloc(2 * dim * sizeof(double));
        for (uint64_t s = 0; s < dim; s++) {
            uint64_t o = 0;
            for (int j = 0; j < k; j++) o |= ((s >> (k - 1 - j)) & 1) << g->q[j];
            off[s] = o;
        }
        for (uint64_t base = 0; base < n; base++) {
            if (base & qmask) continue;
            for (uint64_t s = 0; s < dim; s++) {
                tmp[2 * s] = a[2 * (base | off[s])];
                tmp[2 * s + 1] = a[2 * (base | off[s]) + 1];
            }
            for (uint64_t r = 0; r < dim; r++) {
                double sr = 0.0, si = 0.0;
                const double* row = g->payload + 2 * r * dim;
                for (uint64_t s = 0; s < dim; s++) {
                    double x = tmp[2 * s], y = tmp[2 * s + 1];
                    sr += x * row[2 * s] - y * row[2 * s + 1];
                    si += y * row[2 * s] + x * row[2 * s + 1];
                }
                res[2 * r] = sr;
                res[2 * r + 1] = si;
            }
            for (uint64_t r = 0; r < dim; r++) {
                a[2 * (base | off[r])] = res[2 * r];
                a[2 * (base | off[r]) + 1] = res[2 * r + 1];
            }
        }
        free(off); free(tmp); free(res);
        return;
    }
    }
}

/* applyBlock: chunks x gates (engine.cpp:262-281). Returns -1 if a gate
   reaches outside the chunk (engine.cpp:264-268). */
int qo_apply_block(double* a, int nQubits, const qo_gate* gates, int ngates, int chunkQubits) {
    for (int g = 0; g < ngates; g++)
        for (int j = 0; j < gates[g].nq; j++)
            if (gates[g].q[j] >= chunkQubits) return -1;
    uint64_t len = (uint64_t)1 << chunkQubits;
    uint64_t chunks = ((uint64_t)1 << nQubits) >> chunkQubits;
    for (uint64_t c = 0; c < chunks; c++)
        for (int g = 0; g < ngates; g++) qo_apply_gate(a + 2 * c * len, len, &gates[g]);
    return 0;
}

/* ---- permutations: engine.cpp:30-36, 86-101 -------------------------------- */

uint64_t qo_bitswap(uint64_t x, const int* outs, const int* ins, int s) {
    for (int j = 0; j < s; j++) {
        uint64_t b1 = (x >> outs[j]) & 1, b2 = (x >> ins[j]) & 1;
        if (b1 != b2) x ^= ((uint64_t)1 << outs[j]) | ((uint64_t)1 << ins[j]);
    }
    return x;
}

/* imsSwap result: a[bitswap(i)] <- a[i], in place.  The reference's
   cache-line traversal (shiftPairs) only reorders visits; the permutation is
   the same, so the restatement walks indices directly (engine.cpp:93-99
   swaps each orbit once, from its larger member). */
void qo_ims_swap(double* a, int nQubits, const int* outs, const int* ins, int s) {
    uint64_t n = (uint64_t)1 << nQubits;
    for (uint64_t t = 0; t < n; t++) {
        uint64_t u = qo_bitswap(t, outs, ins, s);
        if (t > u) swap_amp(a, t, u);
    }
}

/* ---- cross-rank swap: distributed.cpp:25-138 ------------------------------
   state: all 2^r slices back to back (rank-major).  stats: 4 u64 per rank
   {bytesSent, bytesReceived, peakBufferBytes, rounds}.  Returns -1 on the
   reference's validation errors (distributed.cpp:36-48). */
int qo_xrs_swap(double* state, int n, int r, int bufferQubits, const int* outs, const int* ins,
                int s, uint64_t* stats) {
    int region = n - r;
    if (bufferQubits < s) return -1;
    int offPos[64], nOff = 0, insRel[64];
    for (int j = 0; j < s; j++) {
        if (outs[j] < 0 || outs[j] >= region || ins[j] < region || ins[j] >= n) return -1;
        insRel[j] = ins[j] - region;
    }
    for (int p = 0; p < region; p++) {
        int used = 0;
        for (int j = 0; j < s; j++) used |= outs[j] == p;
        if (!used) offPos[nOff++] = p;
    }
    uint64_t slabOffsets = (uint64_t)1 << (region - s);
    uint64_t window = (uint64_t)1 << (bufferQubits - s);
    if (window > slabOffsets) window = slabOffsets;
    int ranks = 1 << r, slabs = 1 << s;
    uint64_t per = (uint64_t)1 << region;
    if (stats) memset(stats, 0, 4 * sizeof(uint64_t) * ranks);
    if (s == 0) return 0;
    double** buf = (double**)calloc(ranks, sizeof(double*));
    for (int k = 0; k < ranks; k++) buf[k] = (double*)malloc(2 * (slabs - 1) * window * sizeof(double));
    for (uint64_t w0 = 0; w0 < slabOffsets; w0 += window) {
        uint64_t cnt = window < slabOffsets - w0 ? window : slabOffsets - w0;
        /* xrsFill (distributed.cpp:76-94) */
        for (int k = 0; k < ranks; k++) {
            int own = 0;
            for (int j = 0; j < s; j++) own |= ((k >> insRel[j]) & 1) << j;
            uint64_t at = 0;
            double* slice = state + 2 * per * k;
            for (int p = 0; p < slabs; p++) {
                if (p == own) continue;
                for (uint64_t o = w0; o < w0 + cnt; o++) {
                    uint64_t l = 0;
                    for (int j = 0; j < s; j++) l |= (uint64_t)((p >> j) & 1) << outs[j];
                    for (int i = 0; i < nOff; i++) l |= ((o >> i) & 1) << offPos[i];
                    buf[k][2 * at] = slice[2 * l];
                    buf[k][2 * at + 1] = slice[2 * l + 1];
                    at++;
                }
            }
            if (stats) {
                uint64_t bytes = at * 16;
                stats[4 * k + 0] += bytes;
                uint64_t cap = (uint64_t)(slabs - 1) * cnt * 16;
                if (cap > stats[4 * k + 2]) stats[4 * k + 2] = cap;
                stats[4 * k + 3] += 1;
            }
        }
        /* xrsDeliver (distributed.cpp:97-120) */
        for (int k = 0; k < ranks; k++) {
            int own = 0;
            for (int j = 0; j < s; j++) own |= ((k >> insRel[j]) & 1) << j;
            double* slice = state + 2 * per * k;
            for (int pa = 0; pa < slabs; pa++) {
                if (pa == own) continue;
                int partner = k;
                for (int j = 0; j < s; j++) {
                    partner &= ~(1 << insRel[j]);
                    partner |= ((pa >> j) & 1) << insRel[j];
                }
                uint64_t section = (uint64_t)(own - (own > pa ? 1 : 0)) * cnt;
                const double* src = buf[partner] + 2 * section;
                for (uint64_t o = w0; o < w0 + cnt; o++) {
                    uint64_t l = 0;
                    for (int j = 0; j < s; j++) l |= (uint64_t)((pa >> j) & 1) << outs[j];
                    for (int i = 0; i < nOff; i++) l |= ((o >> i) & 1) << offPos[i];
                    slice[2 * l] = src[2 * (o - w0)];
                    slice[2 * l + 1] = src[2 * (o - w0) + 1];
                }
                if (stats) stats[4 * k + 1] += cnt * 16;
            }
        }
    }
    for (int k = 0; k < ranks; k++) free(buf[k]);
    free(buf);
    return 0;
}

/* ---- state helpers: engine.cpp:12-28 -------------------------------------- */

void qo_init(double* a, int nQubits, uint64_t initial) {
    uint64_t n = (uint64_t)1 << nQubits;
    memset(a, 0, 2 * n * sizeof(double));
    a[2 * initial] = 1.0;
}

double qo_norm(const double* a, uint64_t n) {
    double s = 0.0;
    for (uint64_t i = 0; i < n; i++) s += a[2 * i] * a[2 * i] + a[2 * i + 1] * a[2 * i + 1];
    return s;
}

/* Matrix-based gate application used by the brute-force oracle
   (tools.cpp:10-40): gather/scatter through the full embedded matrix. */
void qo_gate_matrix(const qo_gate* g, double* out /* 4^nq interleaved */) {
    int k = g->nq;
    uint64_t dim = (uint64_t)1 << k;
    memset(out, 0, 2 * dim * dim * sizeof(double));
    double m[8], d[8];
    switch (g->kind) {
    case QO_H: case QO_U: case QO_X: case QO_RX: case QO_RY:
        qo_mat1(g, m);
        memcpy(out, m, sizeof m);
        return;
    case QO_RZ: case QO_RZZ: case QO_CP: {
        int e = qo_diag(g, d);
        for (int i = 0; i < e; i++) {
            out[2 * (i * e + i)] = d[2 * i];
            out[2 * (i * e + i) + 1] = d[2 * i + 1];
        }
        return;
    }
    case QO_CX:
        out[0] = 1; out[2 * 5] = 1; out[2 * 11] = 1; out[2 * 14] = 1;
        return;
    case QO_SWAP:
        out[0] = 1; out[2 * 6] = 1; out[2 * 9] = 1; out[2 * 15] = 1;
        return;
    case QO_D:
        for (uint64_t i = 0; i < dim; i++) {
            out[2 * (i * dim + i)] = g->payload[2 * i];
            out[2 * (i * dim + i) + 1] = g->payload[2 * i + 1];
        }
        return;
    case QO_UK:
        memcpy(out, g->payload, 2 * dim * dim * sizeof(double));
        return;
    }
}
