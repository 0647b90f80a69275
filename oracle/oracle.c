/*
 * oracle.c -- fp64 CPU oracle (TEST INFRASTRUCTURE ONLY; see oracle.h).
 *
 * Plain, slow, obviously correct: 4x4 homogeneous matrices, the paper's
 * sequential transform chain, and the paper's O(L^2) backward sums.  No
 * blocking, no fusion, no reordering beyond what the paper states.  Built
 * with -O2 -ffp-contract=off (reading Q17: round-to-nearest, no FMA
 * contraction); OpenMP only distributes independent chains.
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ---- PAPER §3: the backbone transform table ----------------
 * atom index i = 3j   : C-N peptide bond,  R(omega, pi - 2.1186, 1.330)
 * atom index i = 3j+1 : N-CA bond,         R(phi_j, pi - 1.9391, 1.460)
 * atom index i = 3j+2 : CA-C bond,         R(psi_j, pi - 2.0610, 1.525)
 * Reading Q1: R_0 = identity (N_0 at the origin).  Reading Q2: transform 3j
 * (j >= 1) carries omega_{j-1} = angles[j-1][2] (IUPAC: omega_j is the
 * C_j-N_{j+1} torsion), so omega_{L-1} drives nothing. */
static double bb_theta(int k) {
    if (k == 0) return M_PI - 2.1186;
    if (k == 1) return M_PI - 1.9391;
    return M_PI - 2.0610;
}
static double bb_d(int k) {
    if (k == 0) return 1.330;
    if (k == 1) return 1.460;
    return 1.525;
}

/* ---- 4x4 algebra (row-major) ------------------------------------------- */
static void mat_identity(double m[16]) {
    memset(m, 0, 16 * sizeof(double));
    m[0] = m[5] = m[10] = m[15] = 1.0;
}
static void mat_mul(const double a[16], const double b[16], double out[16]) {
    double t[16];
    for (int r = 0; r < 4; ++r)
        for (int c = 0; c < 4; ++c) {
            double s = 0.0;
            for (int k = 0; k < 4; ++k) s += a[4 * r + k] * b[4 * k + c];
            t[4 * r + c] = s;
        }
    memcpy(out, t, sizeof(t));
}
/* Rigid inverse [R^T | -R^T t] ("the inverses ... have simple forms"). */
static void mat_rigid_inverse(const double m[16], double out[16]) {
    double t[16];
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) t[4 * r + c] = m[4 * c + r];
    for (int r = 0; r < 3; ++r)
        t[4 * r + 3] = -(t[4 * r + 0] * m[3] + t[4 * r + 1] * m[7] + t[4 * r + 2] * m[11]);
    t[12] = t[13] = t[14] = 0.0;
    t[15] = 1.0;
    memcpy(out, t, sizeof(t));
}
static void mat_apply(const double m[16], const double p[3], double out[3]) {
    for (int r = 0; r < 3; ++r) out[r] = m[4 * r + 0] * p[0] + m[4 * r + 1] * p[1] + m[4 * r + 2] * p[2] + m[4 * r + 3];
}
/* R_x(beta), right-handed (reading Q4), used for the out-of-plane R'. */
static void mat_rot_x(double beta, double m[16]) {
    mat_identity(m);
    m[5] = cos(beta);
    m[6] = -sin(beta);
    m[9] = sin(beta);
    m[10] = cos(beta);
}

/* P:149-155, entries exactly as printed. */
void tplref_bond_transform(double alpha, double theta, double d, double m[16]) {
    double ca = cos(alpha), sa = sin(alpha), ct = cos(theta), st = sin(theta);
    m[0] = ct;   m[1] = sa * st;  m[2] = ca * st;  m[3] = d * ct;
    m[4] = 0.0;  m[5] = ca;       m[6] = -sa;      m[7] = 0.0;
    m[8] = -st;  m[9] = sa * ct;  m[10] = ca * ct; m[11] = -d * st;
    m[12] = 0.0; m[13] = 0.0;     m[14] = 0.0;     m[15] = 1.0;
}
/* Entrywise d/dalpha of the printed matrix. */
void tplref_bond_transform_dalpha(double alpha, double theta, double d, double m[16]) {
    double ca = cos(alpha), sa = sin(alpha), ct = cos(theta), st = sin(theta);
    (void)d;
    m[0] = 0.0;  m[1] = ca * st;  m[2] = -sa * st; m[3] = 0.0;
    m[4] = 0.0;  m[5] = -sa;      m[6] = -ca;      m[7] = 0.0;
    m[8] = 0.0;  m[9] = ca * ct;  m[10] = -sa * ct; m[11] = 0.0;
    m[12] = 0.0; m[13] = 0.0;     m[14] = 0.0;     m[15] = 0.0;
}

int tplref_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* Threads of the OpenMP loops over chains (timing the 1-thread rate). */
void tplref_set_num_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

/* ======================================================================= *
 * Backbone model, PAPER §3                                                *
 * ======================================================================= */

/* Alpha carried by transform i of a chain (table above, readings Q1/Q2);
 * *slot receives the flat index into angles[j][.] or -1 for R_0. */
static double bb_alpha(const double* ang, int i, int* slot) {
    int j = i / 3, k = i % 3;
    if (i == 0) { *slot = -1; return 0.0; }
    if (k == 0) { *slot = 3 * (j - 1) + 2; return ang[*slot]; }  /* omega_{j-1} */
    *slot = 3 * j + (k - 1);                                      /* phi_j / psi_j */
    return ang[*slot];
}

/* Forward: M_i = R_0 R_1 ... R_i, r_i = M_i 0. */
static void bb_chain(const double* ang, int L, double* M /*[3L][16]*/) {
    double Mi[16], R[16];
    mat_identity(Mi);
    for (int i = 0; i < 3 * L; ++i) {
        int slot;
        double a = bb_alpha(ang, i, &slot);
        if (i == 0) mat_identity(R);
        else tplref_bond_transform(a, bb_theta(i % 3), bb_d(i % 3), R);
        mat_mul(Mi, R, Mi);
        memcpy(M + 16 * (size_t)i, Mi, sizeof(Mi));
    }
}

int tplref_backbone_forward(const double* angles, const int32_t* lengths, int32_t B, int32_t Lmax,
                            double* coords) {
    if (!angles || !lengths || !coords || B < 1 || Lmax < 1) return 1;
    for (int b = 0; b < B; ++b)
        if (lengths[b] < 1 || lengths[b] > Lmax) return 2;
#pragma omp parallel for schedule(dynamic)
    for (int b = 0; b < B; ++b) {
        int L = lengths[b];
        double* M = (double*)malloc(sizeof(double) * 16 * 3 * (size_t)L);
        bb_chain(angles + (size_t)b * Lmax * 3, L, M);
        double* out = coords + (size_t)b * 3 * Lmax * 3;
        for (int i = 0; i < 3 * L; ++i) {
            const double zero[3] = {0.0, 0.0, 0.0};
            mat_apply(M + 16 * (size_t)i, zero, out + 3 * i); /* r_i = M_i 0 */
        }
        free(M);
    }
    return 0;
}

/* Eq. 2: for transform a carrying angle alpha_a,
 *   dr_i/dalpha_a = M_{a-1} dR_a M_a^{-1} M_i 0   for i >= a   (0 for i < a)
 *   dL/dalpha_a  = sum_i dL/dr_i . dr_i/dalpha_a
 * computed per angle independently, O(L^2) per chain, as the paper does.
 * Structural zeros (reading Q2): psi_{L-1} moves no atom but its own origin
 * and omega_{L-1} drives no transform; both are written as exactly 0. */
int tplref_backbone_backward(const double* angles, const int32_t* lengths, int32_t B, int32_t Lmax,
                             const double* grad_coords, double* grad_angles) {
    if (!angles || !lengths || !grad_coords || !grad_angles || B < 1 || Lmax < 1) return 1;
    for (int b = 0; b < B; ++b)
        if (lengths[b] < 1 || lengths[b] > Lmax) return 2;
#pragma omp parallel for schedule(dynamic)
    for (int b = 0; b < B; ++b) {
        int L = lengths[b];
        const double* ang = angles + (size_t)b * Lmax * 3;
        const double* g = grad_coords + (size_t)b * 3 * Lmax * 3;
        double* ga = grad_angles + (size_t)b * Lmax * 3;
        double* M = (double*)malloc(sizeof(double) * 16 * 3 * (size_t)L);
        double* r = (double*)malloc(sizeof(double) * 3 * 3 * (size_t)L);
        bb_chain(ang, L, M);
        for (int i = 0; i < 3 * L; ++i) {
            const double zero[3] = {0.0, 0.0, 0.0};
            mat_apply(M + 16 * (size_t)i, zero, r + 3 * i);
        }
        for (int s = 0; s < 3 * L; ++s) ga[s] = 0.0;
        for (int a = 1; a < 3 * L; ++a) {
            int slot;
            double alpha = bb_alpha(ang, a, &slot);
            double dR[16], Minv[16], D[16];
            tplref_bond_transform_dalpha(alpha, bb_theta(a % 3), bb_d(a % 3), dR);
            mat_mul(M + 16 * (size_t)(a - 1), dR, D);
            mat_rigid_inverse(M + 16 * (size_t)a, Minv);
            mat_mul(D, Minv, D);
            double sum = 0.0;
            for (int i = a; i < 3 * L; ++i) {
                double dr[3];
                mat_apply(D, r + 3 * i, dr);
                sum += g[3 * i + 0] * dr[0] + g[3 * i + 1] * dr[1] + g[3 * i + 2] * dr[2];
            }
            ga[slot] = sum;
        }
        ga[3 * (L - 1) + 1] = 0.0; /* psi_{L-1} */
        ga[3 * (L - 1) + 2] = 0.0; /* omega_{L-1} */
        free(M);
        free(r);
    }
    return 0;
}

/* ======================================================================= *
 * Full-atom model, PAPER §2                                               *
 * ======================================================================= */

typedef struct {
    int parent;          /* node index, -1 for the chain root N_0 */
    int grad;            /* flat index into grad_angles[b][.][.] or -1 */
    double alpha, theta, d;
    double P[16];        /* M_parent (times R' where the table has one) */
    double M[16];        /* cumulative transform of this node */
    int first_child, next_sibling;
    int first_atom;      /* atoms attached to this node (linked list) */
} fa_node;

typedef struct {
    int node;
    int next;            /* next atom on the same node */
    double r[3];
} fa_atom;

typedef struct {
    fa_node* nodes;
    fa_atom* atoms;
    int n_nodes, n_atoms;
} fa_graph;

static int fa_new_node(fa_graph* G, int parent) {
    int n = G->n_nodes++;
    fa_node* x = &G->nodes[n];
    x->parent = parent;
    x->grad = -1;
    x->alpha = x->theta = x->d = 0.0;
    x->first_child = -1;
    x->first_atom = -1;
    if (parent >= 0) {
        x->next_sibling = G->nodes[parent].first_child;
        G->nodes[parent].first_child = n;
    } else {
        x->next_sibling = -1;
    }
    return n;
}

/* M_node = P R(alpha, theta, d) with P = M_parent. */
static void fa_set_transform(fa_graph* G, int n, const double P[16], double alpha, double theta, double d, int grad) {
    fa_node* x = &G->nodes[n];
    double R[16];
    memcpy(x->P, P, sizeof(x->P));
    x->alpha = alpha;
    x->theta = theta;
    x->d = d;
    x->grad = grad;
    tplref_bond_transform(alpha, theta, d, R);
    mat_mul(P, R, x->M);
}

/* Builds the transform graph of one chain and places every atom
 * (r = M_owner r°).  Atoms are stored in output order. */
static int fa_build(const tplref_restype* types, int n_types, const double* ang /*[Lmax][8]*/,
                    const uint8_t* rt, int L, fa_graph* G) {
    int prevC = -1;
    G->n_nodes = 0;
    G->n_atoms = 0;
    for (int j = 0; j < L; ++j) {
        if (rt[j] >= n_types) return 2;
        const tplref_restype* T = &types[rt[j]];
        const double* a = ang + (size_t)j * TPLREF_SLOTS;
        int gnode[TPLREF_MAX_GROUPS];
        /* N_j: reached from C_{j-1} by R(omega_{j-1}, pi-2.1186, 1.330) (Q2);
         * N_0 is the root with M = identity (Q1). */
        int nN = fa_new_node(G, prevC);
        if (prevC < 0) {
            mat_identity(G->nodes[nN].P);
            mat_identity(G->nodes[nN].M);
        } else {
            const double* ap = ang + (size_t)(j - 1) * TPLREF_SLOTS;
            fa_set_transform(G, nN, G->nodes[prevC].M, ap[2], M_PI - 2.1186, 1.330, (j - 1) * TPLREF_SLOTS + 2);
        }
        /* CA_j: R(phi_j, pi-1.9391, 1.460)  (threonine M_1 = M_0 R_1(phi)) */
        int nCA = fa_new_node(G, nN);
        fa_set_transform(G, nCA, G->nodes[nN].M, a[0], M_PI - 1.9391, 1.460, j * TPLREF_SLOTS + 0);
        /* side-chain groups (threonine M_2 = M_0 R_1 R' R_2(chi)) */
        for (int g = 0; g < T->n_groups; ++g) {
            int par = T->g_parent[g] < 0 ? nCA : gnode[T->g_parent[g]];
            double P[16], Rx[16];
            memcpy(P, G->nodes[par].M, sizeof(P));
            if (T->g_prerx[g] != 0.0) {
                mat_rot_x(T->g_prerx[g], Rx);
                mat_mul(P, Rx, P);
            }
            int slot = T->g_slot[g];
            double alpha = slot >= 0 ? a[slot] : T->g_alpha[g];
            gnode[g] = fa_new_node(G, par);
            fa_set_transform(G, gnode[g], P, alpha, T->g_theta[g], T->g_d[g], slot >= 0 ? j * TPLREF_SLOTS + slot : -1);
        }
        /* C_j: R(psi_j, pi-2.0610, 1.525)  (threonine M_3 = M_0 R_1 R_3(psi)) */
        int nC = fa_new_node(G, nCA);
        fa_set_transform(G, nC, G->nodes[nCA].M, a[1], M_PI - 2.0610, 1.525, j * TPLREF_SLOTS + 1);
        /* atoms, in the table's (output) order */
        for (int k = 0; k < T->n_atoms; ++k) {
            int o = T->a_owner[k];
            int node = o == TPLREF_OWNER_N ? nN : o == TPLREF_OWNER_CA ? nCA : o == TPLREF_OWNER_C ? nC : gnode[o];
            fa_atom* at = &G->atoms[G->n_atoms];
            at->node = node;
            mat_apply(G->nodes[node].M, T->a_r[k], at->r);
            /* append to the node's atom list */
            at->next = -1;
            if (G->nodes[node].first_atom < 0) {
                G->nodes[node].first_atom = G->n_atoms;
            } else {
                int q = G->nodes[node].first_atom;
                while (G->atoms[q].next >= 0) q = G->atoms[q].next;
                G->atoms[q].next = G->n_atoms;
            }
            G->n_atoms++;
        }
        prevC = nC;
    }
    return 0;
}

static int fa_validate(const tplref_restype* types, int32_t n_types, const uint8_t* restype, const int32_t* lengths,
                       int32_t B, int32_t Lmax, int32_t atom_stride) {
    if (!types || n_types < 1 || !restype || !lengths || B < 1 || Lmax < 1) return 1;
    for (int t = 0; t < n_types; ++t)
        if (types[t].n_groups < 0 || types[t].n_groups > TPLREF_MAX_GROUPS || types[t].n_atoms < 0 ||
            types[t].n_atoms > TPLREF_MAX_ATOMS)
            return 1;
    for (int b = 0; b < B; ++b) {
        if (lengths[b] < 1 || lengths[b] > Lmax) return 2;
        long n = 0;
        for (int j = 0; j < lengths[b]; ++j) {
            uint8_t t = restype[(size_t)b * Lmax + j];
            if (t >= n_types) return 2;
            n += types[t].n_atoms;
        }
        if (n > atom_stride) return 1;
    }
    return 0;
}

static void fa_alloc(fa_graph* G, const tplref_restype* types, const uint8_t* rt, int L) {
    int nn = 0, na = 0;
    for (int j = 0; j < L; ++j) {
        nn += 3 + types[rt[j]].n_groups;
        na += types[rt[j]].n_atoms;
    }
    G->nodes = (fa_node*)malloc(sizeof(fa_node) * (size_t)(nn > 0 ? nn : 1));
    G->atoms = (fa_atom*)malloc(sizeof(fa_atom) * (size_t)(na > 0 ? na : 1));
}

int tplref_fullatom_forward(const tplref_restype* types, int32_t n_types, const double* angles,
                            const uint8_t* restype, const int32_t* lengths, int32_t B, int32_t Lmax,
                            int32_t atom_stride, double* coords, int32_t* n_atoms) {
    int v = fa_validate(types, n_types, restype, lengths, B, Lmax, atom_stride);
    if (v) return v;
    if (!angles || !coords) return 1;
#pragma omp parallel for schedule(dynamic)
    for (int b = 0; b < B; ++b) {
        fa_graph G;
        const uint8_t* rt = restype + (size_t)b * Lmax;
        fa_alloc(&G, types, rt, lengths[b]);
        fa_build(types, n_types, angles + (size_t)b * Lmax * TPLREF_SLOTS, rt, lengths[b], &G);
        double* out = coords + (size_t)b * atom_stride * 3;
        for (int k = 0; k < G.n_atoms; ++k) {
            out[3 * k + 0] = G.atoms[k].r[0];
            out[3 * k + 1] = G.atoms[k].r[1];
            out[3 * k + 2] = G.atoms[k].r[2];
        }
        if (n_atoms) n_atoms[b] = G.n_atoms;
        free(G.nodes);
        free(G.atoms);
    }
    return 0;
}

/* Eq. 1, reading Q6:
 *   dL/dalpha_n = sum_{k in subtree(n)} dL/dr_k . F_n r_k,
 *   F_n = P_n dR(alpha_n)/dalpha M_n^{-1}
 * with the sum accumulated by a depth-first traversal of node n's subtree
 * using an explicit stack ("backward depth-first propagation").
 * Fixed nodes and unused slots get exactly 0. */
int tplref_fullatom_backward(const tplref_restype* types, int32_t n_types, const double* angles,
                             const uint8_t* restype, const int32_t* lengths, int32_t B, int32_t Lmax,
                             int32_t atom_stride, const double* grad_coords, double* grad_angles) {
    int v = fa_validate(types, n_types, restype, lengths, B, Lmax, atom_stride);
    if (v) return v;
    if (!angles || !grad_coords || !grad_angles) return 1;
#pragma omp parallel for schedule(dynamic)
    for (int b = 0; b < B; ++b) {
        fa_graph G;
        const uint8_t* rt = restype + (size_t)b * Lmax;
        const double* g = grad_coords + (size_t)b * atom_stride * 3;
        double* ga = grad_angles + (size_t)b * Lmax * TPLREF_SLOTS;
        fa_alloc(&G, types, rt, lengths[b]);
        fa_build(types, n_types, angles + (size_t)b * Lmax * TPLREF_SLOTS, rt, lengths[b], &G);
        for (int s = 0; s < lengths[b] * TPLREF_SLOTS; ++s) ga[s] = 0.0;
        int* stack = (int*)malloc(sizeof(int) * (size_t)(G.n_nodes > 0 ? G.n_nodes : 1));
        for (int n = 0; n < G.n_nodes; ++n) {
            fa_node* x = &G.nodes[n];
            if (x->grad < 0) continue;
            double dR[16], Minv[16], F[16];
            tplref_bond_transform_dalpha(x->alpha, x->theta, x->d, dR);
            mat_mul(x->P, dR, F);
            mat_rigid_inverse(x->M, Minv);
            mat_mul(F, Minv, F);
            double sum = 0.0;
            int sp = 0;
            stack[sp++] = n;
            while (sp > 0) {
                int u = stack[--sp];
                for (int k = G.nodes[u].first_atom; k >= 0; k = G.atoms[k].next) {
                    double dr[3];
                    mat_apply(F, G.atoms[k].r, dr);
                    sum += g[3 * k + 0] * dr[0] + g[3 * k + 1] * dr[1] + g[3 * k + 2] * dr[2];
                }
                for (int c = G.nodes[u].first_child; c >= 0; c = G.nodes[c].next_sibling) stack[sp++] = c;
            }
            ga[x->grad] = sum;
        }
        free(stack);
        free(G.nodes);
        free(G.atoms);
    }
    return 0;
}
