/*
 * tpl.h -- C ABI v1 of libtpl.so: batched, differentiable dihedral-angle ->
 * Cartesian-coordinate maps of arXiv 1812.01108 (TorchProteinLibrary) on B200.
 *
 * No CUDA headers: device pointers are plain pointers, streams are passed as
 * void* (a cudaStream_t; NULL = the legacy default stream).
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 * Ownership   The caller owns every buffer.  fwd/bwd calls never allocate;
 *             only tpl_tables_create allocates (device memory for the table).
 * Streams     All device work is enqueued on `stream`; nothing synchronises
 *             except tpl_sync_status.
 * Memory      Every array argument of a fwd/bwd call is DEVICE memory
 *             (lengths included), dense row-major as documented, 4-byte
 *             aligned; 16-byte alignment lets more of it move by TMA bulk
 *             copies but is not required.
 * Padding     Entries of a chain past lengths[b] are neither read nor written.
 * Errors      Host-detectable problems (NULL, B < 1, Lmax < 1, workspace too
 *             small, atom_stride < 1, bad table) return a status BEFORE
 *             any launch and set tpl_last_error().  Device-detectable
 *             problems (lengths[b] outside [1, Lmax], a restype >= n_types,
 *             a chain with more atoms than atom_stride) set a flag in the
 *             workspace, the offending chain is skipped (a full-atom chain
 *             over atom_stride keeps the tiles that fit),
 *             and tpl_sync_status reports TPL_ERR_DEVICE_INPUT.  No C++
 *             exception crosses the ABI.
 * Workspace   Device buffer of tpl_workspace_bytes(model, B, Lmax) bytes,
 *             ZERO-INITIALISED before first use; reusable across calls on
 *             the same stream; one workspace per concurrently used stream.
 *             It holds the error word, a launch epoch and per-(chain, tile)
 *             carry slots: for few long chains the backbone kernels split a
 *             chain over co-resident CTAs that exchange their carries there
 *             (waiting only on earlier work items, so they always finish,
 *             given the grid's CTAs are not starved by a never-ending
 *             concurrent kernel).
 * Determinism Bitwise identical results for identical inputs on one build
 *             and device: no float atomics, fixed association order.
 * Precision   fp32 arithmetic with FMA contraction, accurate sincosf (no
 *             fast-math); fixed theta/d constants are rounded from fp64.
 *             Scan aggregates are re-orthonormalised (one Newton-Schulz
 *             step) unless the environment sets TPL_ORTHO=0.
 */
#ifndef TPL_H
#define TPL_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TPL_ABI_VERSION 1

#if defined(__GNUC__)
#define TPL_API __attribute__((visibility("default")))
#else
#define TPL_API
#endif

typedef enum {
    TPL_OK = 0,
    TPL_ERR_NULL = 1,         /* a required pointer is NULL */
    TPL_ERR_SHAPE = 2,        /* B < 1, Lmax < 1, atom_stride too small, ... */
    TPL_ERR_ALIGN = 3,        /* a pointer is not 4-byte aligned */
    TPL_ERR_TABLE = 4,        /* residue-type table rejected */
    TPL_ERR_CUDA = 5,         /* a CUDA runtime call failed (see tpl_last_error) */
    TPL_ERR_DEVICE_INPUT = 6, /* a kernel flagged a bad length / restype */
    TPL_ERR_WORKSPACE = 7     /* workspace NULL or smaller than tpl_workspace_bytes */
} tpl_status;

#define TPL_MODEL_BACKBONE 0
#define TPL_MODEL_FULLATOM 1

/* Slots of the per-residue angle record.  Backbone records have 3 slots
 * (phi, psi, omega); full-atom records 8 (phi, psi, omega, chi1..chi5),
 * reading Q10 of DESIGN.md ("up to 7 dihedral angles", plus chi5). */
#define TPL_BB_SLOTS 3
#define TPL_FA_SLOTS 8
#define TPL_SLOT_PHI 0
#define TPL_SLOT_PSI 1
#define TPL_SLOT_OMEGA 2
#define TPL_SLOT_CHI1 3

#define TPL_MAX_GROUPS 8   /* side-chain rigid groups per residue type */
#define TPL_MAX_ATOMS 16   /* atoms per residue type (N, CA, side chain, C, O) */
#define TPL_MAX_TYPES 32   /* residue types per table */

/* Owner of an atom in a residue type: the N, CA or C backbone frame, or a
 * side-chain group index >= 0. */
#define TPL_OWNER_N (-3)
#define TPL_OWNER_CA (-2)
#define TPL_OWNER_C (-1)

/* Thread-local text describing the last non-OK status of this thread. */
TPL_API const char* tpl_last_error(void);
TPL_API int tpl_abi_version(void);

/* Device workspace bytes needed by any fwd/bwd call of `model` with these
 * B and Lmax (header words + per-(chain, tile) carry slots). */
TPL_API size_t tpl_workspace_bytes(int32_t model, int32_t B, int32_t Lmax);

/* Synchronise `stream`, then read and clear the device error flags of
 * `workspace`.  TPL_ERR_DEVICE_INPUT if a kernel skipped a chain. */
TPL_API tpl_status tpl_sync_status(void* stream, void* workspace);

/* ======================================================================
 * Backbone model (§3)
 * ====================================================================== */

/* Atoms of a backbone chain of L residues: 3L (N, CA, C). */
TPL_API int64_t tpl_backbone_atoms(int32_t L);

/* Forward.  P:143-175: r_i = R_0 R_1 ... R_i 0 with the transform table of
 * atom 3j (N_j) via R(omega_{j-1}, pi-2.1186, 1.330), atom 3j+1
 * (CA_j) via R(phi_j, pi-1.9391, 1.460), atom 3j+2 (C_j) via
 * R(psi_j, pi-2.0610, 1.525); R_0 = I (N_0 at the origin, reading Q1) and
 * omega_j is the C_j-N_{j+1} torsion (reading Q2).
 *   angles   [B][Lmax][3] fp32, (phi, psi, omega) in radians, any real value
 *   lengths  [B] int32, each in [1, Lmax]
 *   coords   [B][3*Lmax][3] fp32 output, Angstrom, atoms N, CA, C per residue */
TPL_API tpl_status tpl_backbone_forward(const float* angles, const int32_t* lengths, int32_t B, int32_t Lmax,
                                float* coords, void* workspace, size_t ws_bytes, void* stream);

/* Backward: dL/dangles for L with dL/dr = grad_coords (Eq. 2),
 * recomputed from the angles (no saved forward state).
 *   grad_coords [B][3*Lmax][3] fp32
 *   grad_angles [B][Lmax][3]   fp32 output; psi_{L-1} and omega_{L-1} are 0 */
TPL_API tpl_status tpl_backbone_backward(const float* angles, const int32_t* lengths, int32_t B, int32_t Lmax,
                                 const float* grad_coords, float* grad_angles, void* workspace, size_t ws_bytes,
                                 void* stream);

/* Backward from the forward's output: the same dL/dangles computed from
 * coords = tpl_backbone_forward(angles) instead of the angles.  Eq. 2's
 * derivative dr_b/dalpha_a = e_a x (r_b - r_a) (b > a) needs only
 * positions: the rotation axis e_a of transform a is the unit bond vector
 * (r_a - r_{a-1}) / |r_a - r_{a-1}|.  No trig, no scan of
 * transforms: one reverse suffix sum of (sum g, sum r x g) per chain.
 *   coords      [B][3*Lmax][3] fp32, the forward's output for these lengths
 *   grad_coords [B][3*Lmax][3] fp32
 *   grad_angles [B][Lmax][3]   fp32 output; psi_{L-1} and omega_{L-1} are 0 */
TPL_API tpl_status tpl_backbone_backward_from_coords(const float* coords, const int32_t* lengths, int32_t B,
                                             int32_t Lmax, const float* grad_coords, float* grad_angles,
                                             void* workspace, size_t ws_bytes, void* stream);

/* precise mode: the same map as tpl_backbone_forward (P:143-175,
 * Q1/Q2) computed entirely in fp64 (the paper's decimal theta/d, fp64 sincos,
 * transforms and scan), coordinates rounded once to fp32.  For regular chains
 * that span hundreds to thousands of Angstrom, where the fp32 path's rounding
 * crosses 1e-3 A (f2).  Slower: fp64 arithmetic throughout. */
TPL_API tpl_status tpl_backbone_forward_precise(const float* angles, const int32_t* lengths, int32_t B,
                                        int32_t Lmax, float* coords, void* workspace, size_t ws_bytes,
                                        void* stream);

/* SURVEY f1 in one pass (PAPER §3 P:143-196 + §4, reading Q19):
 * angles -> backbone coordinates -> LRMSD to the target y -> dLRMSD/dangles,
 * one kernel, no coordinate round-trip through HBM.  Per chain b (3L atoms):
 *   lrmsd[b]        the LRMSD of P:204 after optimal superposition
 *   state[b][16]    U (9, row-major), barycentre of x (3), of y (3), 1/(3L LRMSD)
 *                   (the layout of tpl_lrmsd_forward)
 *   grad_angles     [B][Lmax][3] dLRMSD/d(phi, psi, omega) (not yet multiplied by
 *                   dL/dLRMSD: see tpl_chain_scale); psi_{L-1}, omega_{L-1} = 0;
 *                   0 for a chain whose LRMSD vanishes (the gradient is undefined)
 *   coords          [B][3*Lmax][3] fp32 or NULL (written only when non-NULL)
 * target [B][3*Lmax][3] fp32.  Lmax <= tpl_backbone_lrmsd_fused_max_L() (one CTA
 * tile per chain), else TPL_ERR_SHAPE (use the two-call pair below).  Entries
 * past lengths[b] are neither read for the sums nor written.  Device input
 * errors as tpl_backbone_forward (chain skipped, error word set). */
TPL_API int32_t tpl_backbone_lrmsd_fused_max_L(void);
TPL_API tpl_status tpl_backbone_lrmsd_fused(const float* angles, const int32_t* lengths, int32_t B, int32_t Lmax,
                                            const float* target, float* coords, float* lrmsd, float* state,
                                            float* grad_angles, void* workspace, size_t ws_bytes, void* stream);

/* y[b * per_chain + i] = x[b * per_chain + i] * scale[b] for b < B, i < per_chain
 * (device pointers): the chain rule dL/dangles = dL/dLRMSD[b] dLRMSD/dangles of
 * the fused pass's autograd backward.  x and y may alias. */
TPL_API tpl_status tpl_chain_scale(const float* x, const float* scale, int32_t B, int32_t per_chain, float* y,
                                   void* stream);

/* the backbone map and the LRMSD loss (PAPER §4)
 * fused: the forward also reduces, per chain, the moments of (r, y) over the
 * chain's 3L atoms against the reference y [B][3*Lmax][3] and returns
 * lrmsd[B] and state[B][16] (as tpl_lrmsd_forward); the backward forms
 * dL/dr_i = grad_lrmsd[b] (r~_i - U^T y~_i) / (3L LRMSD) on the fly inside the
 * coordinate backward (no dL/dr array), giving grad_angles [B][Lmax][3].
 * coords is the forward's output (kept by the caller for the backward). */
TPL_API tpl_status tpl_backbone_lrmsd_forward(const float* angles, const int32_t* lengths, int32_t B, int32_t Lmax,
                                      const float* target, float* coords, float* lrmsd, float* state,
                                      void* workspace, size_t ws_bytes, void* stream);
TPL_API tpl_status tpl_backbone_lrmsd_backward(const float* coords, const int32_t* lengths, int32_t B,
                                       int32_t Lmax, const float* target, const float* state,
                                       const float* grad_lrmsd, float* grad_angles, void* workspace,
                                       size_t ws_bytes, void* stream);

/* one chain split over n_seg ranks (segment s holds residues
 * [j_s, j_{s+1}) of every chain; lengths[b] = its segment length >= 1), one
 * exchange per pass.  Forward: each rank computes its segment in
 * the segment's own frame -- identity at the previous segment's last C, with
 * omega_prev[b] (= omega_{j_s - 1}, NULL for the first segment) driving the
 * bond to its first N -- and exports the aggregate transform A_s [B][12]
 * (row-major 3x4).  The caller all-gathers A into [n_seg][B][12]; _place
 * maps the local coordinates to the chain frame with A_0 ... A_{s-1} composed
 * in that order.  Backward (Eq. 2 as e . (T - r x S)): _totals writes
 * (S = sum g, T = sum (r - c) x g, c = the segment's first atom, 0,0,0) [B][12]
 * of the placed coordinates; after an all-gather into [n_seg][B][12], _backward
 * adds the later segments' sums and closes omega of the segment's last residue
 * with the next segment's first atom.  All arrays are device memory. */
TPL_API tpl_status tpl_backbone_segment_forward(const float* angles, const int32_t* lengths, int32_t B,
                                        int32_t Lmax, const float* omega_prev, float* coords, float* aggregate,
                                        void* workspace, size_t ws_bytes, void* stream);
TPL_API tpl_status tpl_backbone_segment_place(float* coords, const int32_t* lengths, int32_t B, int32_t Lmax,
                                      const float* aggregates, int32_t n_seg, int32_t seg, void* workspace,
                                      size_t ws_bytes, void* stream);
TPL_API tpl_status tpl_backbone_segment_totals(const float* coords, const int32_t* lengths, int32_t B,
                                       int32_t Lmax, const float* grad_coords, float* totals, void* workspace,
                                       size_t ws_bytes, void* stream);
TPL_API tpl_status tpl_backbone_segment_backward(const float* coords, const int32_t* lengths, int32_t B,
                                         int32_t Lmax, const float* grad_coords, const float* totals,
                                         int32_t n_seg, int32_t seg, float* grad_angles, void* workspace,
                                         size_t ws_bytes, void* stream);

/* the paper's own GPU design, built as a measured comparison
 * point (not the product path).  Forward: one thread per chain saves every
 * cumulative transform M_i = R_0...R_i as a row-major 4x4 fp32
 * (64 B/atom) plus r_i.  Backward: one thread per (chain, angle) evaluates
 * sum_{i>=a} g_i . (M_{a-1} dR_a M_a^{-1} M_i 0) (Eq. 2) without a
 * reduction: O(L^2) per chain.  Same readings (Q1, Q2) and outputs as
 * the product pair.
 *   saved_M [B][3*Lmax][16] fp32, 16-byte aligned, written by the forward and
 *           read by the backward; tpl_paper_backbone_saved_floats(B, Lmax) floats */
TPL_API int64_t tpl_paper_backbone_saved_floats(int32_t B, int32_t Lmax);
TPL_API tpl_status tpl_paper_backbone_forward(const float* angles, const int32_t* lengths, int32_t B, int32_t Lmax,
                                      float* coords, float* saved_M, void* workspace, size_t ws_bytes,
                                      void* stream);
TPL_API tpl_status tpl_paper_backbone_backward(const float* angles, const int32_t* lengths, int32_t B,
                                       int32_t Lmax, const float* saved_M, const float* grad_coords,
                                       float* grad_angles, void* workspace, size_t ws_bytes, void* stream);

/* ======================================================================
 * Full-atom model (§2)
 * ====================================================================== */

/* One residue type (host memory, plain data).  The backbone nodes are
 * implicit and use the §3 constants: N_j (from C_{j-1} by omega_{j-1}),
 * CA_j (phi_j), C_j (psi_j).  Side-chain group g is reached from its parent
 * frame P by  M_g = P * R_x(group_pre_rx[g]) * R(alpha, theta, d)  (R' of
 * P:48 when pre_rx != 0) with alpha = angles[slot] for slot in 3..7
 * (chi1..chi5) or the fixed group_alpha[g] when slot < 0.
 * v1 restriction: group_parent[g] is -1 (the CA frame) or g-1.
 * Atoms: r = M_owner r°, owner = TPL_OWNER_N/CA/C or a group;
 * atoms are listed in output order, which must be owner-sorted as
 *   N-owned, CA-owned, group 0, group 1, ..., C-owned
 * (e.g. N, CA, side chain depth-first, C, O: reading Q9). */
typedef struct tpl_residue_desc {
    int32_t n_groups;
    int32_t n_atoms;
    int32_t group_parent[TPL_MAX_GROUPS];
    int32_t group_slot[TPL_MAX_GROUPS];
    double group_alpha[TPL_MAX_GROUPS];
    double group_theta[TPL_MAX_GROUPS];
    double group_d[TPL_MAX_GROUPS];
    double group_pre_rx[TPL_MAX_GROUPS];
    int32_t atom_owner[TPL_MAX_ATOMS];
    double atom_r[TPL_MAX_ATOMS][3];
} tpl_residue_desc;

typedef struct tpl_tables tpl_tables; /* opaque, immutable after create */

/* The residue-type table of the full-atom model: per type the rigid groups
 * ("the rigid groups of atoms ... connected by the dihedral angles",
 * R' of P:48) and their atoms' positions in the group frame (r°);
 * the paper gives only threonine's topology, so the values are data
 * (reading Q8).  Validate and upload `n_types` (1..TPL_MAX_TYPES) types;
 * uses the current CUDA device.  Errors: TPL_ERR_NULL, TPL_ERR_TABLE (a
 * count out of range, a parent that is neither -1 nor g-1, a slot outside
 * 3..7, atoms not owner-sorted), TPL_ERR_CUDA.  *out is NULL on failure;
 * the caller owns the table and frees it with tpl_tables_destroy. */
TPL_API tpl_status tpl_tables_create(const tpl_residue_desc* types, int32_t n_types, tpl_tables** out);
TPL_API void tpl_tables_destroy(tpl_tables* tables);
TPL_API int32_t tpl_tables_n_types(const tpl_tables* tables);

/* Host-side bookkeeping of the packed output layout (each residue
 * contributes its type's heavy atoms, hydrogens omitted -- reading Q14):
 * atoms_per_chain[b] (may be NULL) = sum of the chain's per-type atom counts,
 * and the padded *atom_stride = max_b atoms (rounded up to a multiple of 4)
 * for HOST restype [B][Lmax] and lengths [B].  Errors: TPL_ERR_NULL,
 * TPL_ERR_SHAPE (B or Lmax < 1, a length outside [1, Lmax], a restype >= the
 * table's type count, a stride that overflows int32). */
TPL_API tpl_status tpl_fullatom_atoms(const tpl_tables* tables, const uint8_t* restype_host, const int32_t* lengths_host,
                              int32_t B, int32_t Lmax, int32_t* atoms_per_chain, int32_t* atom_stride);

/* Forward (P:41-59 on the backbone chain of P:143-175): the backbone frames
 * N_j, CA_j, C_j by the same transform product as the backbone model, then per
 * residue the side-chain groups M_g = M_parent R_x(pre) R(chi or fixed, theta,
 * d) and every atom r = M_owner r°.  angles [B][Lmax][8] fp32 (phi, psi, omega,
 * chi1..chi5), restype [B][Lmax] uint8 (device), coords [B][atom_stride][3]
 * fp32 output: each chain's atoms packed from index 0, residue by residue, in
 * the table's atom order; entries past a chain's atoms are not written.  A
 * length outside [1, Lmax], a restype >= n_types or a chain that overflows
 * atom_stride is skipped and flagged in the workspace error word. */
TPL_API tpl_status tpl_fullatom_forward(const tpl_tables* tables, const float* angles, const uint8_t* restype,
                                const int32_t* lengths, int32_t B, int32_t Lmax, int32_t atom_stride,
                                float* coords, void* workspace, size_t ws_bytes, void* stream);

/* Backward (Eq. 1, in O(L) with suffix sums): grad_coords in the
 * coords layout, grad_angles [B][Lmax][8] output; fixed and unused slots
 * and omega_{L-1} are 0. */
TPL_API tpl_status tpl_fullatom_backward(const tpl_tables* tables, const float* angles, const uint8_t* restype,
                                 const int32_t* lengths, int32_t B, int32_t Lmax, int32_t atom_stride,
                                 const float* grad_coords, float* grad_angles, void* workspace, size_t ws_bytes,
                                 void* stream);

/* Backward from the forward's output: the same grad_angles computed from
 * coords = tpl_fullatom_forward(angles) instead of the angles.  Each angle of
 * Eq. 1 rotates a frame about the bond from its parent frame's
 * origin to its own: the axis is the unit vector between those two
 * origin atoms and the rotated subtree is fixed by the atom order.  Needs a
 * table in which every such origin is an atom (r° = 0): N, CA, C and each
 * chi group's first atom -- tpl_tables_backward_from_coords_ok() tells; else
 * TPL_ERR_TABLE.  The bundled table (synth/residue_table.json) qualifies. */
TPL_API tpl_status tpl_fullatom_backward_from_coords(const tpl_tables* tables, const float* coords,
                                             const uint8_t* restype, const int32_t* lengths, int32_t B,
                                             int32_t Lmax, int32_t atom_stride, const float* grad_coords,
                                             float* grad_angles, void* workspace, size_t ws_bytes, void* stream);
TPL_API int32_t tpl_tables_backward_from_coords_ok(const tpl_tables* tables);

/* ======================================================================
 * LRMSD loss (§4): Coutsias-Seok-Dill quaternion method
 * ====================================================================== */

/* Per chain b: barycentres, R = sum x~ y~^T, the 4x4 T as printed, its largest
 * eigenpair (lambda, q), U(q) as printed, LRMSD = sqrt((sum|x~|^2+|y~|^2 - 2 lambda)/N).
 * x is the structure that is differentiated, y the reference (reading Q19).
 *   x, y     [B][stride][3] fp32 device (e.g. packed full-atom or backbone coords)
 *   n_atoms  [B] int32 device, each in [1, stride]; atoms past n_atoms[b] are ignored
 *   lrmsd    [B] fp32 output
 *   state    [B][16] fp32 output for the backward: U row-major, centroid of x,
 *            centroid of y, 1/(N LRMSD) (0 where LRMSD == 0)
 *   workspace: any tpl workspace (its error word flags bad n_atoms). */
TPL_API tpl_status tpl_lrmsd_forward(const float* x, const float* y, const int32_t* n_atoms, int32_t B,
                                     int32_t stride, float* lrmsd, float* state, void* workspace, size_t ws_bytes,
                                     void* stream);

/* grad_x[b][i] = grad_lrmsd[b] * (x~_i - U^T y~_i) / (N LRMSD): the printed
 * gradient with its normalisation; 0 where LRMSD == 0.  Atoms past
 * n_atoms[b] are not written. */
TPL_API tpl_status tpl_lrmsd_backward(const float* x, const float* y, const int32_t* n_atoms, int32_t B,
                                      int32_t stride, const float* state, const float* grad_lrmsd, float* grad_x,
                                      void* workspace, size_t ws_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* TPL_H */
