// kernels.h -- internal launch interface between capi.cu and the kernels.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace tpl {

// Bond-transform constants of one node: cos/sin of the fixed theta and d.
struct BondC {
    float ct, st, d;
};

constexpr int kBBThreads = 128;
constexpr int kMaxGroups = 8;
constexpr int kMaxAtomsPerRes = 16;
constexpr int kMaxTypes = 32;
constexpr int kFASlots = 8;

// Backbone transform constants: theta_k = pi - 2.1186,
// pi - 1.9391, pi - 2.0610 and d_k = 1.330, 1.460, 1.525 for k = 0 (C-N,
// omega), 1 (N-CA, phi), 2 (CA-C, psi).  cos/sin evaluated in fp64 and rounded
// once to fp32 (reading Q20); tests/test_abi_cpu.py re-derives every literal.
// Compile-time literals so the bond products issue as immediate-operand FFMAs.
constexpr float kBBct[3] = {5.208135247e-01f, 3.600333929e-01f, 4.708055854e-01f};
constexpr float kBBst[3] = {8.536704779e-01f, 9.329394102e-01f, 8.822369576e-01f};
constexpr float kBBd[3] = {1.330000043e+00f, 1.460000038e+00f, 1.524999976e+00f};
// 1 / kBBd[k]: the backward's unit bond axes from coordinates (the selects fold in unrolled code)
constexpr float kBBinvd0 = 1.f / kBBd[0], kBBinvd1 = 1.f / kBBd[1], kBBinvd2 = 1.f / kBBd[2];
__host__ __device__ constexpr float bb_invd(int k) { return k == 0 ? kBBinvd0 : k == 1 ? kBBinvd1 : kBBinvd2; }
struct BBConst {
    BondC b[3];
};

struct BBArgs {
    const float* angles;
    const int* lengths;
    int B, Lmax;
    float* coords;
    const float* grad_coords;
    float* grad_angles;
    unsigned* err;
    float* ws_prefix;
    int max_tiles;
    int ns;  // Newton-Schulz policy: 0 none, 1 prefix/total, 2 every combine
    BBConst K;
    // f4 chain segments (nullptr otherwise): see tpl_backbone_segment_*
    const float* seg_omega_prev;  // [B] omega of the residue before the segment
    float* seg_agg_out;           // [B][12] the segment's aggregate transform
    const float* seg_totals;      // [n_seg][B][12] (S, T about c, c, pad) of every segment
    int n_seg, seg;
    // f1 fused LRMSD (nullptr otherwise): see tpl_backbone_lrmsd_*
    const float* loss_target;  // [B][3*Lmax][3] the reference coordinates y
    float* loss_out;           // [B] LRMSD (forward)
    float* loss_state_out;     // [B][16] U, barycentres, 1/(N LRMSD) (forward)
    const float* loss_state;   // [B][16] U, barycentres, 1/(N LRMSD) (backward)
    const float* loss_grad;    // [B] dL/dLRMSD (backward)
};

bool pdl_enabled();  // capi.cu: programmatic dependent launch on (TPL_PDL != 0)

int bb_rpt_for(int Lmax);
int bb_tile_for(int Lmax);
cudaError_t bb_forward_launch(const BBArgs& a, cudaStream_t st);
// packed.cu: two residue runs per thread in f32x2 lanes, one CTA per chain (Lmax <= bbp_forward_max_L())
bool bbp_enabled();
int bbp_forward_max_L();
cudaError_t bbp_forward_launch(const BBArgs& a, cudaStream_t st);
cudaError_t bbp_forward_tiles_launch(const BBArgs& a, cudaStream_t st);  // multi-tile chains, policy 1
bool bbp_backward_xyz_ok(const BBArgs& a);
cudaError_t bbp_backward_xyz_launch(const BBArgs& a, cudaStream_t st);
cudaError_t bbp_backward_xyz_tiles_launch(const BBArgs& a, cudaStream_t st);  // multi-tile chains
// fused_lrmsd.cu: angles -> coords -> LRMSD -> dLRMSD/dangles in one kernel
int bbp_lrmsd_max_L();
cudaError_t bbp_lrmsd_fused_launch(const BBArgs& a, float* grad_angles, cudaStream_t st);
cudaError_t chain_scale_launch(const float* x, const float* s, int B, int per_chain, float* y, cudaStream_t st);
cudaError_t bb_backward_launch(const BBArgs& a, cudaStream_t st);
cudaError_t bb_backward_xyz_launch(const BBArgs& a, cudaStream_t st);  // a.coords is the input
int bb_dl_max_tiles(int Lmax);
cudaError_t bb_forward_precise_launch(const BBArgs& a, cudaStream_t st);  // f2: fp64-internal forward
// f4 across ranks (segment.cu)
cudaError_t segment_totals_launch(const BBArgs& a, float* totals, cudaStream_t st);
cudaError_t segment_place_launch(const BBArgs& a, const float* aggs, int seg, cudaStream_t st);  // per-chain carry slots of the decoupled backbone kernels
// the paper's own GPU design (paper_baseline.cu), a comparison point
cudaError_t paper_bb_forward_launch(const BBArgs& a, float* Msave, cudaStream_t st);
cudaError_t paper_bb_backward_launch(const BBArgs& a, const float* Msave, cudaStream_t st);

// ---- full atom -------------------------------------------------------------
// Device residue-type table (fp32, uploaded once by tpl_tables_create).
// One record per type, 16-byte aligned, copied whole into shared memory.
struct alignas(16) FAGroup {  // 64 bytes: loaded whole with four 16-byte loads
    float ca, sa;      // cos/sin of the fixed alpha (slot < 0)
    float ct, st, d;   // bond constants
    float cb, sb;      // R' = R_x(pre_rx); (1, 0) when absent
    int parent;        // -1 = CA frame, else g-1 (v1 restriction, see tpl.h)
    int slot;          // 3..7 = chi1..chi5, -1 fixed
    int has_pre;       // pre_rx != 0
    int first_atom;    // index of the group's first atom in the type's atom list
    int end_atom;      // one past the group's last atom
    int origin;        // atom at the group frame's origin (owned by g, r° = 0), -1 if none
    int porigin;       // atom at the parent frame's origin (CA for parent -1), -1 if none
    int pad_[2];
};
static_assert(sizeof(FAGroup) == 64, "FAGroup is loaded as four 16-byte vectors");
struct alignas(16) FAType {
    int n_groups, n_atoms;
    int n_N, n_CA;            // atoms owned by the N / CA frames (first n_N, then n_CA)
    int first_C;              // first atom owned by the C frame; C-owned atoms run to n_atoms
    int iN, iCA, iC;          // atoms at the N / CA / C frame origins (r° = 0), -1 if none
    FAGroup g[kMaxGroups];
    float r[kMaxAtomsPerRes][4];  // r° xyz (w unused)
};

struct FAArgs {
    const FAType* types;
    int n_types;
    const float* angles;
    const unsigned char* restype;
    const int* lengths;
    int B, Lmax, atom_stride;
    float* coords;
    const float* grad_coords;
    float* grad_angles;
    unsigned* err;
    float* ws_prefix;  // per chain per tile: 12 floats prefix + 1 int atom offset (stride 16)
    int max_tiles;
    int ns;
    int max_atoms;  // largest atom count of a residue type in the table
    BBConst K;
};

// ---- LRMSD (PAPER §4) ------------------------------------------------------
struct LRArgs {
    const float* x;  // [B][stride][3], differentiated structure
    const float* y;  // [B][stride][3], reference
    const int* n_atoms;
    int B, stride;
    float* out;    // [B] LRMSD
    float* state;  // [B][16]: U (9), centroid x (3), centroid y (3), 1/(N LRMSD)
    const float* grad_out;  // [B] dL/dLRMSD
    float* grad_x;          // [B][stride][3]
    unsigned* err;
};
cudaError_t lrmsd_forward_launch(const LRArgs& a, cudaStream_t st);
cudaError_t lrmsd_backward_launch(const LRArgs& a, cudaStream_t st);

int fa_rpt_for(int Lmax);
int fa_tile_for(int Lmax);
cudaError_t fa_forward_launch(const FAArgs& a, cudaStream_t st);
cudaError_t fa_backward_launch(const FAArgs& a, cudaStream_t st);
cudaError_t fa_backward_xyz_launch(const FAArgs& a, cudaStream_t st);  // a.coords is the input
constexpr int kFAXMaxL = 65536;  // longest chain of the coordinate backward (restype staged on chip)

}  // namespace tpl
