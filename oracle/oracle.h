/*
 * oracle.h -- fp64 CPU oracle for arXiv 1812.01108 (TorchProteinLibrary).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load liboracle.so.
 * The product (paper_1812_01108_b200/, libtpl.so) never calls it, and this
 * file shares no header, helper or constant with include/tpl.h or the CUDA
 * sources.
 *
 * Everything here is the paper's own sequential algorithm, written out in
 * double precision in the paper's order and notation:
 *   backbone forward  P:143-175  (r_i = R_0 R_1 ... R_i 0, saved M_i)
 *   backbone backward P:176-196  (Eq. 2 with M_{a-1} dR_a M_a^{-1}, O(L^2))
 *   full-atom forward P:41-59    (M_child = M_parent R_child, r = M r°)
 *   full-atom backward P:68-128  (Eq. 1, depth-first over the subtree, O(L^2))
 *   LRMSD             P:198-237  (Coutsias-Seok-Dill quaternion method)
 * Readings of ambiguous passages (Q1..Q22) are listed in DESIGN.md.
 *
 * Inputs are double (tests promote the fp32 GPU inputs exactly); outputs are
 * double.  Return value: 0 = ok, 1 = bad argument, 2 = bad length/restype.
 */
#ifndef TPL_ORACLE_H
#define TPL_ORACLE_H
#include <stdint.h>

#define TPLREF_MAX_GROUPS 8
#define TPLREF_MAX_ATOMS 16
#define TPLREF_SLOTS 8 /* phi, psi, omega, chi1..chi5 (reading Q10) */

/* Owner codes of an atom in a residue-type description. */
#define TPLREF_OWNER_N (-3)
#define TPLREF_OWNER_CA (-2)
#define TPLREF_OWNER_C (-1)

/* One residue type of the full-atom model: side-chain rigid
 * groups (parent = -1: the CA frame, else an earlier group), each reached by
 * R_x(prerx) R(alpha, theta, d) where alpha is angles[slot] or the fixed
 * g_alpha when slot < 0; and atoms with standard coordinates r° in the frame
 * of their owner (N / CA / C node or a side-chain group). */
typedef struct {
    int32_t n_groups, n_atoms;
    int32_t g_parent[TPLREF_MAX_GROUPS];
    int32_t g_slot[TPLREF_MAX_GROUPS];
    double g_alpha[TPLREF_MAX_GROUPS];
    double g_theta[TPLREF_MAX_GROUPS];
    double g_d[TPLREF_MAX_GROUPS];
    double g_prerx[TPLREF_MAX_GROUPS];
    int32_t a_owner[TPLREF_MAX_ATOMS];
    double a_r[TPLREF_MAX_ATOMS][3];
} tplref_restype;

/* P:149-155, the printed R(alpha, theta, d); row-major 4x4. */
void tplref_bond_transform(double alpha, double theta, double d, double out[16]);
/* dR/dalpha of the printed matrix (theta, d fixed). */
void tplref_bond_transform_dalpha(double alpha, double theta, double d, double out[16]);

int tplref_num_threads(void);
void tplref_set_num_threads(int n);

/* Backbone (PAPER §3).  angles [B][Lmax][3] = (phi, psi, omega) per residue,
 * coords [B][3*Lmax][3] (atoms N, CA, C per residue), grad_coords likewise,
 * grad_angles [B][Lmax][3].  Entries past lengths[b] are not touched. */
int tplref_backbone_forward(const double* angles, const int32_t* lengths, int32_t B, int32_t Lmax,
                            double* coords);
int tplref_backbone_backward(const double* angles, const int32_t* lengths, int32_t B, int32_t Lmax,
                             const double* grad_coords, double* grad_angles);

/* Full atom (PAPER §2).  angles [B][Lmax][8], restype [B][Lmax],
 * coords [B][atom_stride][3] packed per chain in residue order, atoms of one
 * residue in the table's order.  n_atoms [B] receives each chain's count. */
int tplref_fullatom_forward(const tplref_restype* types, int32_t n_types, const double* angles,
                            const uint8_t* restype, const int32_t* lengths, int32_t B, int32_t Lmax,
                            int32_t atom_stride, double* coords, int32_t* n_atoms);
int tplref_fullatom_backward(const tplref_restype* types, int32_t n_types, const double* angles,
                             const uint8_t* restype, const int32_t* lengths, int32_t B, int32_t Lmax,
                             int32_t atom_stride, const double* grad_coords, double* grad_angles);

#endif
