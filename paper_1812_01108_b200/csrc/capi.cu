// capi.cu -- the C ABI of libtpl.so (include/tpl.h): argument validation,
// workspace sizing, residue-table upload and kernel launch configuration.
// All arithmetic of the method lives in backbone.cu / fullatom.cu.
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "../../include/tpl.h"
#include "kernels.h"

using namespace tpl;

// Programmatic dependent launch of the kernels: opt-in (TPL_PDL=1).  Measured
// in CUDA graphs on B200 (tools/step_timing.py): at 256 x 700 an alternating
// forward/backward step is 17.2 us without PDL and 19.5 us with it (the early
// launched dependents hold SM slots); at 1024 x 700 PDL gains ~2%.
bool tpl::pdl_enabled() {
    static int v = -1;
    if (v < 0) {
        const char* e = std::getenv("TPL_PDL");
        v = (e && e[0] == '1') ? 1 : 0;
    }
    return v == 1;
}

namespace {

thread_local std::string g_last_error;

tpl_status fail(tpl_status s, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
tpl_status fail(tpl_status s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return s;
}

tpl_status cuda_fail(cudaError_t e, const char* where) {
    return fail(TPL_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

bool aligned4(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 3u) == 0; }

// Newton-Schulz re-orthonormalisation policy of the affine scan (TPL_ORTHO):
// 0 = off, 1 = chunk aggregates, scan results and carries (backbone default),
// 2 = additionally after every combine inside the scan, 3 = as 1 plus the warp
// totals and every cross-warp combine (full-atom default).  Backbone forward at
// L = 700 (tools/gpu_ortho.sh): helix / strand / extended 4.1e-3 / 6.5e-3 /
// 1.9e-3 A under 1, 2.5e-4 / 4.9e-4 / 5.1e-4 A under 2, for +0.5 us (256 x 700).
int ns_policy() {
    static int v = -1;
    if (v < 0) {
        const char* e = std::getenv("TPL_ORTHO");
        v = (e && e[0] >= '0' && e[0] <= '3') ? e[0] - '0' : 1;
    }
    return v;
}

// the backbone transform table.  theta and d are the
// paper's decimal constants; cos/sin are evaluated in fp64 and rounded once
// (reading Q20).  k = 0: C-N (omega), 1: N-CA (phi), 2: CA-C (psi).
BBConst backbone_constants() {
    const double theta[3] = {M_PI - 2.1186, M_PI - 1.9391, M_PI - 2.0610};
    const double d[3] = {1.330, 1.460, 1.525};
    BBConst K;
    for (int k = 0; k < 3; ++k) {
        K.b[k].ct = static_cast<float>(std::cos(theta[k]));
        K.b[k].st = static_cast<float>(std::sin(theta[k]));
        K.b[k].d = static_cast<float>(d[k]);
    }
    return K;
}

// The kernels use kBBct/kBBst/kBBd as compile-time literals; check once per
// process that they are the fp64-evaluated constants rounded to fp32.
bool constants_consistent() {
    static int ok = -1;
    if (ok < 0) {
        const BBConst K = backbone_constants();
        ok = 1;
        for (int k = 0; k < 3; ++k)
            if (K.b[k].ct != kBBct[k] || K.b[k].st != kBBst[k] || K.b[k].d != kBBd[k]) ok = 0;
    }
    return ok == 1;
}

constexpr size_t kWsHeader = 256;  // error word + reserved

int tile_for(int model, int Lmax) { return model == TPL_MODEL_FULLATOM ? fa_tile_for(Lmax) : bb_tile_for(Lmax); }
int max_tiles_for(int model, int Lmax) {
    if (model == TPL_MODEL_BACKBONE) {  // the decoupled kernels' tiles (>= 128 residues) need the most slots
        const int t = tile_for(model, Lmax), old = (Lmax + t - 1) / t, dl = bb_dl_max_tiles(Lmax);
        return old > dl ? old : dl;
    }
    const int t = tile_for(model, Lmax);
    return (Lmax + t - 1) / t;
}

tpl_status check_ws(int model, int B, int Lmax, void* ws, size_t ws_bytes) {
    if (!constants_consistent()) return fail(TPL_ERR_CUDA, "internal: backbone constant literals do not match fp64");
    if (!ws) return fail(TPL_ERR_WORKSPACE, "workspace is NULL");
    if (!aligned4(ws) || (reinterpret_cast<uintptr_t>(ws) & 15u))
        return fail(TPL_ERR_ALIGN, "workspace must be 16-byte aligned");
    const size_t need = tpl_workspace_bytes(model, B, Lmax);
    if (ws_bytes < need) return fail(TPL_ERR_WORKSPACE, "workspace %zu bytes < required %zu", ws_bytes, need);
    return TPL_OK;
}

}  // namespace

struct tpl_tables {
    FAType* dev = nullptr;
    int n_types = 0;
    int atoms[TPL_MAX_TYPES] = {0};
    int max_atoms = 0;
    int device = 0;
    // every frame an angle rotates has an atom at its origin and at its parent's
    // origin: the from-coordinates backward can read the rotation axes
    bool xyz_ok = false;
    std::string xyz_why;
};

extern "C" {

const char* tpl_last_error(void) { return g_last_error.c_str(); }
int tpl_abi_version(void) { return TPL_ABI_VERSION; }
int64_t tpl_backbone_atoms(int32_t L) { return L < 0 ? 0 : 3 * static_cast<int64_t>(L); }

size_t tpl_workspace_bytes(int32_t model, int32_t B, int32_t Lmax) {
    if (B < 1 || Lmax < 1) return kWsHeader;
    const size_t tiles = static_cast<size_t>(max_tiles_for(model, Lmax));
    const size_t slots = kWsHeader + static_cast<size_t>(B) * tiles * 16 * sizeof(float);
    return slots;
}

tpl_status tpl_sync_status(void* stream, void* workspace) {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "cudaStreamSynchronize");
    if (!workspace) return fail(TPL_ERR_WORKSPACE, "workspace is NULL");
    unsigned flags = 0;
    e = cudaMemcpy(&flags, workspace, sizeof(flags), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpy(error word)");
    if (flags) {
        e = cudaMemset(workspace, 0, sizeof(unsigned));
        if (e != cudaSuccess) return cuda_fail(e, "cudaMemset(error word)");
        return fail(TPL_ERR_DEVICE_INPUT, "device input error flags 0x%x (%s%s%s)", flags,
                    (flags & 1u) ? "length outside [1, Lmax] " : "", (flags & 2u) ? "restype >= n_types " : "",
                    (flags & 4u) ? "a chain's atoms exceed atom_stride" : "");
    }
    return TPL_OK;
}

// ---------------------------------------------------------------- backbone
static tpl_status bb_common(const float* angles, const int32_t* lengths, int32_t B, int32_t Lmax, void* ws,
                            size_t ws_bytes) {
    if (!angles || !lengths) return fail(TPL_ERR_NULL, "angles/lengths is NULL");
    if (B < 1 || Lmax < 1) return fail(TPL_ERR_SHAPE, "B=%d Lmax=%d must be >= 1", B, Lmax);
    if (!aligned4(angles) || !aligned4(lengths)) return fail(TPL_ERR_ALIGN, "angles/lengths not 4-byte aligned");
    return check_ws(TPL_MODEL_BACKBONE, B, Lmax, ws, ws_bytes);
}

tpl_status tpl_backbone_forward(const float* angles, const int32_t* lengths, int32_t B, int32_t Lmax,
                                float* coords, void* workspace, size_t ws_bytes, void* stream) {
    tpl_status s = bb_common(angles, lengths, B, Lmax, workspace, ws_bytes);
    if (s != TPL_OK) return s;
    if (!coords) return fail(TPL_ERR_NULL, "coords is NULL");
    if (!aligned4(coords)) return fail(TPL_ERR_ALIGN, "coords not 4-byte aligned");
    BBArgs a{};
    a.angles = angles;
    a.lengths = lengths;
    a.B = B;
    a.Lmax = Lmax;
    a.coords = coords;
    a.err = static_cast<unsigned*>(workspace);
    a.ws_prefix = reinterpret_cast<float*>(static_cast<char*>(workspace) + kWsHeader);
    a.max_tiles = max_tiles_for(TPL_MODEL_BACKBONE, Lmax);
    a.ns = ns_policy();
    a.K = backbone_constants();
    cudaError_t e = bb_forward_launch(a, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "backbone forward launch");
    return TPL_OK;
}

tpl_status tpl_backbone_backward(const float* angles, const int32_t* lengths, int32_t B, int32_t Lmax,
                                 const float* grad_coords, float* grad_angles, void* workspace, size_t ws_bytes,
                                 void* stream) {
    tpl_status s = bb_common(angles, lengths, B, Lmax, workspace, ws_bytes);
    if (s != TPL_OK) return s;
    if (!grad_coords || !grad_angles) return fail(TPL_ERR_NULL, "grad_coords/grad_angles is NULL");
    if (!aligned4(grad_coords) || !aligned4(grad_angles)) return fail(TPL_ERR_ALIGN, "grads not 4-byte aligned");
    BBArgs a{};
    a.angles = angles;
    a.lengths = lengths;
    a.B = B;
    a.Lmax = Lmax;
    a.grad_coords = grad_coords;
    a.grad_angles = grad_angles;
    a.err = static_cast<unsigned*>(workspace);
    a.ws_prefix = reinterpret_cast<float*>(static_cast<char*>(workspace) + kWsHeader);
    a.max_tiles = max_tiles_for(TPL_MODEL_BACKBONE, Lmax);
    a.ns = ns_policy();
    a.K = backbone_constants();
    cudaError_t e = bb_backward_launch(a, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "backbone backward launch");
    return TPL_OK;
}

tpl_status tpl_backbone_backward_from_coords(const float* coords, const int32_t* lengths, int32_t B, int32_t Lmax,
                                             const float* grad_coords, float* grad_angles, void* workspace,
                                             size_t ws_bytes, void* stream) {
    if (!coords) return fail(TPL_ERR_NULL, "coords is NULL");
    // bb_common checks lengths/B/Lmax/workspace; coords stands in for the (unused) angles
    tpl_status s = bb_common(coords, lengths, B, Lmax, workspace, ws_bytes);
    if (s != TPL_OK) return s;
    if (!grad_coords || !grad_angles) return fail(TPL_ERR_NULL, "grad_coords/grad_angles is NULL");
    if (!aligned4(grad_coords) || !aligned4(grad_angles)) return fail(TPL_ERR_ALIGN, "grads not 4-byte aligned");
    BBArgs a{};
    a.lengths = lengths;
    a.B = B;
    a.Lmax = Lmax;
    a.coords = const_cast<float*>(coords);
    a.grad_coords = grad_coords;
    a.grad_angles = grad_angles;
    a.err = static_cast<unsigned*>(workspace);
    a.ws_prefix = reinterpret_cast<float*>(static_cast<char*>(workspace) + kWsHeader);  // tile carry slots
    a.max_tiles = max_tiles_for(TPL_MODEL_BACKBONE, Lmax);
    cudaError_t e = bb_backward_xyz_launch(a, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "backbone backward (from coords) launch");
    return TPL_OK;
}

// ---------------------------------------------------------------- f2: fp64-internal forward
tpl_status tpl_backbone_forward_precise(const float* angles, const int32_t* lengths, int32_t B, int32_t Lmax,
                                        float* coords, void* workspace, size_t ws_bytes, void* stream) {
    tpl_status s = bb_common(angles, lengths, B, Lmax, workspace, ws_bytes);
    if (s != TPL_OK) return s;
    if (!coords) return fail(TPL_ERR_NULL, "coords is NULL");
    if (!aligned4(coords)) return fail(TPL_ERR_ALIGN, "coords not 4-byte aligned");
    BBArgs a{};
    a.angles = angles;
    a.lengths = lengths;
    a.B = B;
    a.Lmax = Lmax;
    a.coords = coords;
    a.err = static_cast<unsigned*>(workspace);
    cudaError_t e = bb_forward_precise_launch(a, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "precise backbone forward launch");
    return TPL_OK;
}

// ---------------------------------------------------------------- f1: backbone + LRMSD, fused
tpl_status tpl_backbone_lrmsd_forward(const float* angles, const int32_t* lengths, int32_t B, int32_t Lmax,
                                      const float* target, float* coords, float* lrmsd, float* state,
                                      void* workspace, size_t ws_bytes, void* stream) {
    tpl_status s = bb_common(angles, lengths, B, Lmax, workspace, ws_bytes);
    if (s != TPL_OK) return s;
    if (!target || !coords || !lrmsd || !state) return fail(TPL_ERR_NULL, "target/coords/lrmsd/state is NULL");
    if (!aligned4(target) || !aligned4(coords) || !aligned4(lrmsd) || !aligned4(state))
        return fail(TPL_ERR_ALIGN, "pointers not 4-byte aligned");
    BBArgs a{};
    a.angles = angles;
    a.lengths = lengths;
    a.B = B;
    a.Lmax = Lmax;
    a.coords = coords;
    a.err = static_cast<unsigned*>(workspace);
    a.ws_prefix = reinterpret_cast<float*>(static_cast<char*>(workspace) + kWsHeader);
    a.max_tiles = max_tiles_for(TPL_MODEL_BACKBONE, Lmax);
    a.ns = ns_policy();
    a.K = backbone_constants();
    a.loss_target = target;
    a.loss_out = lrmsd;
    a.loss_state_out = state;
    cudaError_t e = bb_forward_launch(a, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "fused backbone+LRMSD forward launch");
    return TPL_OK;
}

int32_t tpl_backbone_lrmsd_fused_max_L(void) { return bbp_lrmsd_max_L(); }

tpl_status tpl_backbone_lrmsd_fused(const float* angles, const int32_t* lengths, int32_t B, int32_t Lmax,
                                    const float* target, float* coords, float* lrmsd, float* state,
                                    float* grad_angles, void* workspace, size_t ws_bytes, void* stream) {
    tpl_status s = bb_common(angles, lengths, B, Lmax, workspace, ws_bytes);
    if (s != TPL_OK) return s;
    if (!target || !lrmsd || !state || !grad_angles)
        return fail(TPL_ERR_NULL, "target/lrmsd/state/grad_angles is NULL");
    if (!aligned4(target) || (coords && !aligned4(coords)) || !aligned4(lrmsd) || !aligned4(state) ||
        !aligned4(grad_angles))
        return fail(TPL_ERR_ALIGN, "pointers not 4-byte aligned");
    if (Lmax > bbp_lrmsd_max_L())
        return fail(TPL_ERR_SHAPE, "Lmax %d > %d: use tpl_backbone_lrmsd_forward/_backward", Lmax, bbp_lrmsd_max_L());
    BBArgs a{};
    a.angles = angles;
    a.lengths = lengths;
    a.B = B;
    a.Lmax = Lmax;
    a.coords = coords;
    a.err = static_cast<unsigned*>(workspace);
    a.ns = ns_policy() >= 1 ? 1 : 0;
    a.K = backbone_constants();
    a.loss_target = target;
    a.loss_out = lrmsd;
    a.loss_state_out = state;
    cudaError_t e = bbp_lrmsd_fused_launch(a, grad_angles, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "one-pass backbone+LRMSD launch");
    return TPL_OK;
}

tpl_status tpl_chain_scale(const float* x, const float* scale, int32_t B, int32_t per_chain, float* y, void* stream) {
    if (!x || !scale || !y) return fail(TPL_ERR_NULL, "x/scale/y is NULL");
    if (B < 0 || per_chain < 0) return fail(TPL_ERR_SHAPE, "B=%d per_chain=%d", B, per_chain);
    if (!aligned4(x) || !aligned4(scale) || !aligned4(y)) return fail(TPL_ERR_ALIGN, "pointers not 4-byte aligned");
    cudaError_t e = chain_scale_launch(x, scale, B, per_chain, y, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "chain scale launch");
    return TPL_OK;
}

tpl_status tpl_backbone_lrmsd_backward(const float* coords, const int32_t* lengths, int32_t B, int32_t Lmax,
                                       const float* target, const float* state, const float* grad_lrmsd,
                                       float* grad_angles, void* workspace, size_t ws_bytes, void* stream) {
    tpl_status s = bb_common(coords, lengths, B, Lmax, workspace, ws_bytes);
    if (s != TPL_OK) return s;
    if (!target || !state || !grad_lrmsd || !grad_angles)
        return fail(TPL_ERR_NULL, "target/state/grad_lrmsd/grad_angles is NULL");
    if (!aligned4(target) || !aligned4(state) || !aligned4(grad_lrmsd) || !aligned4(grad_angles))
        return fail(TPL_ERR_ALIGN, "pointers not 4-byte aligned");
    BBArgs a{};
    a.lengths = lengths;
    a.B = B;
    a.Lmax = Lmax;
    a.coords = const_cast<float*>(coords);
    a.grad_angles = grad_angles;
    a.err = static_cast<unsigned*>(workspace);
    a.ws_prefix = reinterpret_cast<float*>(static_cast<char*>(workspace) + kWsHeader);
    a.max_tiles = max_tiles_for(TPL_MODEL_BACKBONE, Lmax);
    a.loss_target = target;
    a.loss_state = state;
    a.loss_grad = grad_lrmsd;
    cudaError_t e = bb_backward_xyz_launch(a, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "fused LRMSD+backbone backward launch");
    return TPL_OK;
}

// ---------------------------------------------------------------- f4: one chain over several ranks
static tpl_status seg_args(BBArgs& a, const float* coords_or_angles, const int32_t* lengths, int32_t B, int32_t Lmax,
                           void* workspace, size_t ws_bytes) {
    tpl_status s = bb_common(coords_or_angles, lengths, B, Lmax, workspace, ws_bytes);
    if (s != TPL_OK) return s;
    a = BBArgs{};
    a.lengths = lengths;
    a.B = B;
    a.Lmax = Lmax;
    a.err = static_cast<unsigned*>(workspace);
    a.ws_prefix = reinterpret_cast<float*>(static_cast<char*>(workspace) + kWsHeader);
    a.max_tiles = max_tiles_for(TPL_MODEL_BACKBONE, Lmax);
    a.ns = ns_policy();
    a.K = backbone_constants();
    return TPL_OK;
}

tpl_status tpl_backbone_segment_forward(const float* angles, const int32_t* lengths, int32_t B, int32_t Lmax,
                                        const float* omega_prev, float* coords, float* aggregate, void* workspace,
                                        size_t ws_bytes, void* stream) {
    BBArgs a;
    tpl_status s = seg_args(a, angles, lengths, B, Lmax, workspace, ws_bytes);
    if (s != TPL_OK) return s;
    if (!coords || !aggregate) return fail(TPL_ERR_NULL, "coords/aggregate is NULL");
    if (!aligned4(coords) || !aligned4(aggregate) || (omega_prev && !aligned4(omega_prev)))
        return fail(TPL_ERR_ALIGN, "pointers not 4-byte aligned");
    a.angles = angles;
    a.coords = coords;
    a.seg_omega_prev = omega_prev;
    a.seg_agg_out = aggregate;
    cudaError_t e = bb_forward_launch(a, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "segment forward launch");
    return TPL_OK;
}

tpl_status tpl_backbone_segment_place(float* coords, const int32_t* lengths, int32_t B, int32_t Lmax,
                                      const float* aggregates, int32_t n_seg, int32_t seg, void* workspace,
                                      size_t ws_bytes, void* stream) {
    BBArgs a;
    tpl_status s = seg_args(a, coords, lengths, B, Lmax, workspace, ws_bytes);
    if (s != TPL_OK) return s;
    if (!aggregates) return fail(TPL_ERR_NULL, "aggregates is NULL");
    if (n_seg < 1 || seg < 0 || seg >= n_seg) return fail(TPL_ERR_SHAPE, "seg=%d n_seg=%d", seg, n_seg);
    a.coords = coords;
    cudaError_t e = segment_place_launch(a, aggregates, seg, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "segment place launch");
    return TPL_OK;
}

tpl_status tpl_backbone_segment_totals(const float* coords, const int32_t* lengths, int32_t B, int32_t Lmax,
                                       const float* grad_coords, float* totals, void* workspace, size_t ws_bytes,
                                       void* stream) {
    BBArgs a;
    tpl_status s = seg_args(a, coords, lengths, B, Lmax, workspace, ws_bytes);
    if (s != TPL_OK) return s;
    if (!grad_coords || !totals) return fail(TPL_ERR_NULL, "grad_coords/totals is NULL");
    a.coords = const_cast<float*>(coords);
    a.grad_coords = grad_coords;
    cudaError_t e = segment_totals_launch(a, totals, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "segment totals launch");
    return TPL_OK;
}

tpl_status tpl_backbone_segment_backward(const float* coords, const int32_t* lengths, int32_t B, int32_t Lmax,
                                         const float* grad_coords, const float* totals, int32_t n_seg, int32_t seg,
                                         float* grad_angles, void* workspace, size_t ws_bytes, void* stream) {
    BBArgs a;
    tpl_status s = seg_args(a, coords, lengths, B, Lmax, workspace, ws_bytes);
    if (s != TPL_OK) return s;
    if (!grad_coords || !totals || !grad_angles) return fail(TPL_ERR_NULL, "grad_coords/totals/grad_angles is NULL");
    if (n_seg < 1 || seg < 0 || seg >= n_seg) return fail(TPL_ERR_SHAPE, "seg=%d n_seg=%d", seg, n_seg);
    a.coords = const_cast<float*>(coords);
    a.grad_coords = grad_coords;
    a.grad_angles = grad_angles;
    a.seg_totals = totals;
    a.n_seg = n_seg;
    a.seg = seg;
    cudaError_t e = bb_backward_xyz_launch(a, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "segment backward launch");
    return TPL_OK;
}

// ---------------------------------------------------------------- f3: the paper's GPU design
int64_t tpl_paper_backbone_saved_floats(int32_t B, int32_t Lmax) {
    return (B < 1 || Lmax < 1) ? 0 : static_cast<int64_t>(B) * 3 * Lmax * 16;
}

tpl_status tpl_paper_backbone_forward(const float* angles, const int32_t* lengths, int32_t B, int32_t Lmax,
                                      float* coords, float* saved_M, void* workspace, size_t ws_bytes, void* stream) {
    tpl_status s = bb_common(angles, lengths, B, Lmax, workspace, ws_bytes);
    if (s != TPL_OK) return s;
    if (!coords || !saved_M) return fail(TPL_ERR_NULL, "coords/saved_M is NULL");
    if (!aligned4(coords) || (reinterpret_cast<uintptr_t>(saved_M) & 15u))
        return fail(TPL_ERR_ALIGN, "coords not 4-byte or saved_M not 16-byte aligned");
    BBArgs a{};
    a.angles = angles;
    a.lengths = lengths;
    a.B = B;
    a.Lmax = Lmax;
    a.coords = coords;
    a.err = static_cast<unsigned*>(workspace);
    cudaError_t e = paper_bb_forward_launch(a, saved_M, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "paper-design backbone forward launch");
    return TPL_OK;
}

tpl_status tpl_paper_backbone_backward(const float* angles, const int32_t* lengths, int32_t B, int32_t Lmax,
                                       const float* saved_M, const float* grad_coords, float* grad_angles,
                                       void* workspace, size_t ws_bytes, void* stream) {
    tpl_status s = bb_common(angles, lengths, B, Lmax, workspace, ws_bytes);
    if (s != TPL_OK) return s;
    if (!saved_M || !grad_coords || !grad_angles) return fail(TPL_ERR_NULL, "saved_M/grad_coords/grad_angles is NULL");
    if (!aligned4(grad_coords) || !aligned4(grad_angles) || !aligned4(saved_M))
        return fail(TPL_ERR_ALIGN, "pointers not 4-byte aligned");
    BBArgs a{};
    a.angles = angles;
    a.lengths = lengths;
    a.B = B;
    a.Lmax = Lmax;
    a.grad_coords = grad_coords;
    a.grad_angles = grad_angles;
    a.err = static_cast<unsigned*>(workspace);
    cudaError_t e = paper_bb_backward_launch(a, saved_M, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "paper-design backbone backward launch");
    return TPL_OK;
}

// ---------------------------------------------------------------- tables
static int owner_rank(int owner, int n_groups) {
    if (owner == TPL_OWNER_N) return 0;
    if (owner == TPL_OWNER_CA) return 1;
    if (owner == TPL_OWNER_C) return 2 + n_groups;
    return 2 + owner;
}

tpl_status tpl_tables_create(const tpl_residue_desc* types, int32_t n_types, tpl_tables** out) {
    if (!out) return fail(TPL_ERR_NULL, "out is NULL");
    *out = nullptr;
    if (!types) return fail(TPL_ERR_NULL, "types is NULL");
    if (n_types < 1 || n_types > TPL_MAX_TYPES)
        return fail(TPL_ERR_TABLE, "n_types=%d outside [1, %d]", n_types, TPL_MAX_TYPES);
    FAType host[TPL_MAX_TYPES];
    std::memset(host, 0, sizeof(host));
    tpl_tables* T = new (std::nothrow) tpl_tables();
    if (!T) return fail(TPL_ERR_CUDA, "out of host memory");
    for (int t = 0; t < n_types; ++t) {
        const tpl_residue_desc& d = types[t];
        FAType& h = host[t];
        if (d.n_groups < 0 || d.n_groups > TPL_MAX_GROUPS || d.n_atoms < 0 || d.n_atoms > TPL_MAX_ATOMS) {
            delete T;
            return fail(TPL_ERR_TABLE, "type %d: n_groups=%d n_atoms=%d out of range", t, d.n_groups, d.n_atoms);
        }
        h.n_groups = d.n_groups;
        h.n_atoms = d.n_atoms;
        for (int g = 0; g < d.n_groups; ++g) {
            const int p = d.group_parent[g];
            const int sl = d.group_slot[g];
            if (!(p == -1 || p == g - 1)) {
                delete T;
                return fail(TPL_ERR_TABLE, "type %d group %d: parent %d must be -1 (CA) or g-1 (v1)", t, g, p);
            }
            if (!(sl < 0 || (sl >= TPL_SLOT_CHI1 && sl < TPL_FA_SLOTS))) {
                delete T;
                return fail(TPL_ERR_TABLE, "type %d group %d: slot %d not in {-1, 3..7}", t, g, sl);
            }
            if (!std::isfinite(d.group_theta[g]) || !std::isfinite(d.group_d[g]) || !std::isfinite(d.group_alpha[g]) ||
                !std::isfinite(d.group_pre_rx[g])) {
                delete T;
                return fail(TPL_ERR_TABLE, "type %d group %d: non-finite constant", t, g);
            }
            FAGroup& G = h.g[g];
            G.ca = static_cast<float>(std::cos(d.group_alpha[g]));
            G.sa = static_cast<float>(std::sin(d.group_alpha[g]));
            G.ct = static_cast<float>(std::cos(d.group_theta[g]));
            G.st = static_cast<float>(std::sin(d.group_theta[g]));
            G.d = static_cast<float>(d.group_d[g]);
            G.has_pre = d.group_pre_rx[g] != 0.0;
            G.cb = static_cast<float>(std::cos(d.group_pre_rx[g]));
            G.sb = static_cast<float>(std::sin(d.group_pre_rx[g]));
            G.parent = p;
            G.slot = sl;
            G.first_atom = -1;
            G.end_atom = -1;
            G.origin = -1;
            G.porigin = -1;
        }
        h.iN = h.iCA = h.iC = -1;
        int prev_rank = -1;
        h.n_N = h.n_CA = 0;
        h.first_C = d.n_atoms;
        for (int k = 0; k < d.n_atoms; ++k) {
            const int o = d.atom_owner[k];
            if (!(o == TPL_OWNER_N || o == TPL_OWNER_CA || o == TPL_OWNER_C || (o >= 0 && o < d.n_groups))) {
                delete T;
                return fail(TPL_ERR_TABLE, "type %d atom %d: owner %d invalid", t, k, o);
            }
            const int r = owner_rank(o, d.n_groups);
            if (r < prev_rank) {
                delete T;
                return fail(TPL_ERR_TABLE, "type %d atom %d: atoms must be owner-sorted (N, CA, groups, C)", t, k);
            }
            prev_rank = r;
            for (int c = 0; c < 3; ++c) {
                if (!std::isfinite(d.atom_r[k][c])) {
                    delete T;
                    return fail(TPL_ERR_TABLE, "type %d atom %d: non-finite r", t, k);
                }
                h.r[k][c] = static_cast<float>(d.atom_r[k][c]);
            }
            if (o == TPL_OWNER_N) h.n_N++;
            if (o == TPL_OWNER_CA) h.n_CA++;
            if (o == TPL_OWNER_C && h.first_C == d.n_atoms) h.first_C = k;
            if (o >= 0) {
                if (h.g[o].first_atom < 0) h.g[o].first_atom = k;
                h.g[o].end_atom = k + 1;
            }
            if (d.atom_r[k][0] == 0.0 && d.atom_r[k][1] == 0.0 && d.atom_r[k][2] == 0.0) {
                int* slot = o == TPL_OWNER_N ? &h.iN : o == TPL_OWNER_CA ? &h.iCA : o == TPL_OWNER_C ? &h.iC
                                                                                     : &h.g[o].origin;
                if (*slot < 0) *slot = k;
            }
        }
        for (int g = 0; g < d.n_groups; ++g) h.g[g].porigin = h.g[g].parent < 0 ? h.iCA : h.g[g - 1].origin;
        if (T->xyz_why.empty()) {
            char why[160] = {0};
            if (h.iN < 0 || h.iCA < 0 || h.iC < 0)
                std::snprintf(why, sizeof(why), "type %d: no atom at the N, CA or C frame origin", t);
            for (int g = 0; g < d.n_groups && !why[0]; ++g)
                if (h.g[g].slot >= 0 && (h.g[g].origin < 0 || h.g[g].porigin < 0))
                    std::snprintf(why, sizeof(why), "type %d group %d: no atom at its frame's or parent's origin", t,
                                  g);
            if (why[0]) T->xyz_why = why;
        }
        // empty groups: give them an empty range at the right position
        int next = h.n_N + h.n_CA;
        for (int g = 0; g < d.n_groups; ++g) {
            if (h.g[g].first_atom < 0) {
                h.g[g].first_atom = next;
                h.g[g].end_atom = next;
            }
            next = h.g[g].end_atom;
        }
        T->atoms[t] = d.n_atoms;
        if (d.n_atoms > T->max_atoms) T->max_atoms = d.n_atoms;
    }
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) {
        delete T;
        return cuda_fail(e, "cudaGetDevice");
    }
    e = cudaMalloc(&T->dev, sizeof(FAType) * n_types);
    if (e != cudaSuccess) {
        delete T;
        return cuda_fail(e, "cudaMalloc(tables)");
    }
    e = cudaMemcpy(T->dev, host, sizeof(FAType) * n_types, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        cudaFree(T->dev);
        delete T;
        return cuda_fail(e, "cudaMemcpy(tables)");
    }
    T->n_types = n_types;
    T->device = dev;
    T->xyz_ok = T->xyz_why.empty();
    *out = T;
    return TPL_OK;
}

void tpl_tables_destroy(tpl_tables* T) {
    if (!T) return;
    if (T->dev) cudaFree(T->dev);
    delete T;
}

int32_t tpl_tables_n_types(const tpl_tables* T) { return T ? T->n_types : 0; }

tpl_status tpl_fullatom_atoms(const tpl_tables* T, const uint8_t* restype_host, const int32_t* lengths_host,
                              int32_t B, int32_t Lmax, int32_t* atoms_per_chain, int32_t* atom_stride) {
    if (!T || !restype_host || !lengths_host || !atom_stride) return fail(TPL_ERR_NULL, "NULL argument");
    if (B < 1 || Lmax < 1) return fail(TPL_ERR_SHAPE, "B=%d Lmax=%d must be >= 1", B, Lmax);
    int64_t mx = 0;
    for (int b = 0; b < B; ++b) {
        const int L = lengths_host[b];
        if (L < 1 || L > Lmax) return fail(TPL_ERR_SHAPE, "lengths[%d]=%d outside [1, %d]", b, L, Lmax);
        int64_t n = 0;
        for (int j = 0; j < L; ++j) {
            const int t = restype_host[static_cast<size_t>(b) * Lmax + j];
            if (t >= T->n_types) return fail(TPL_ERR_SHAPE, "restype[%d][%d]=%d >= n_types %d", b, j, t, T->n_types);
            n += T->atoms[t];
        }
        if (atoms_per_chain) atoms_per_chain[b] = static_cast<int32_t>(n);
        if (n > mx) mx = n;
    }
    mx = (mx + 3) & ~int64_t(3);
    if (mx > INT32_MAX) return fail(TPL_ERR_SHAPE, "atom stride overflows int32");
    *atom_stride = static_cast<int32_t>(mx < 4 ? 4 : mx);
    return TPL_OK;
}

static tpl_status fa_common(const tpl_tables* T, const float* angles, const uint8_t* restype, const int32_t* lengths,
                            int32_t B, int32_t Lmax, int32_t atom_stride, void* ws, size_t ws_bytes) {
    if (!T || !angles || !restype || !lengths) return fail(TPL_ERR_NULL, "tables/angles/restype/lengths is NULL");
    if (B < 1 || Lmax < 1) return fail(TPL_ERR_SHAPE, "B=%d Lmax=%d must be >= 1", B, Lmax);
    if (atom_stride < 1) return fail(TPL_ERR_SHAPE, "atom_stride=%d must be >= 1", atom_stride);
    if (!aligned4(angles) || !aligned4(lengths)) return fail(TPL_ERR_ALIGN, "angles/lengths not 4-byte aligned");
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess && dev != T->device)
        return fail(TPL_ERR_TABLE, "tables were created on device %d, current device is %d", T->device, dev);
    return check_ws(TPL_MODEL_FULLATOM, B, Lmax, ws, ws_bytes);
}

static FAArgs fa_args(const tpl_tables* T, const float* angles, const uint8_t* restype, const int32_t* lengths,
                      int32_t B, int32_t Lmax, int32_t atom_stride, void* ws) {
    FAArgs a{};
    a.types = T->dev;
    a.n_types = T->n_types;
    a.angles = angles;
    a.restype = restype;
    a.lengths = lengths;
    a.B = B;
    a.Lmax = Lmax;
    a.atom_stride = atom_stride;
    a.err = static_cast<unsigned*>(ws);
    a.ws_prefix = reinterpret_cast<float*>(static_cast<char*>(ws) + kWsHeader);
    a.max_tiles = max_tiles_for(TPL_MODEL_FULLATOM, Lmax);
    a.ns = ns_policy();
    a.max_atoms = T->max_atoms > 0 ? T->max_atoms : 1;
    a.K = backbone_constants();
    return a;
}

tpl_status tpl_fullatom_forward(const tpl_tables* T, const float* angles, const uint8_t* restype,
                                const int32_t* lengths, int32_t B, int32_t Lmax, int32_t atom_stride, float* coords,
                                void* workspace, size_t ws_bytes, void* stream) {
    tpl_status s = fa_common(T, angles, restype, lengths, B, Lmax, atom_stride, workspace, ws_bytes);
    if (s != TPL_OK) return s;
    if (!coords) return fail(TPL_ERR_NULL, "coords is NULL");
    if (!aligned4(coords)) return fail(TPL_ERR_ALIGN, "coords not 4-byte aligned");
    FAArgs a = fa_args(T, angles, restype, lengths, B, Lmax, atom_stride, workspace);
    a.coords = coords;
    cudaError_t e = fa_forward_launch(a, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "full-atom forward launch");
    return TPL_OK;
}

tpl_status tpl_fullatom_backward(const tpl_tables* T, const float* angles, const uint8_t* restype,
                                 const int32_t* lengths, int32_t B, int32_t Lmax, int32_t atom_stride,
                                 const float* grad_coords, float* grad_angles, void* workspace, size_t ws_bytes,
                                 void* stream) {
    tpl_status s = fa_common(T, angles, restype, lengths, B, Lmax, atom_stride, workspace, ws_bytes);
    if (s != TPL_OK) return s;
    if (!grad_coords || !grad_angles) return fail(TPL_ERR_NULL, "grad_coords/grad_angles is NULL");
    if (!aligned4(grad_coords) || !aligned4(grad_angles)) return fail(TPL_ERR_ALIGN, "grads not 4-byte aligned");
    FAArgs a = fa_args(T, angles, restype, lengths, B, Lmax, atom_stride, workspace);
    a.grad_coords = grad_coords;
    a.grad_angles = grad_angles;
    cudaError_t e = fa_backward_launch(a, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "full-atom backward launch");
    return TPL_OK;
}

tpl_status tpl_fullatom_backward_from_coords(const tpl_tables* T, const float* coords, const uint8_t* restype,
                                             const int32_t* lengths, int32_t B, int32_t Lmax, int32_t atom_stride,
                                             const float* grad_coords, float* grad_angles, void* workspace,
                                             size_t ws_bytes, void* stream) {
    if (!coords) return fail(TPL_ERR_NULL, "coords is NULL");
    // fa_common's angle checks apply to coords (same pointer rules)
    tpl_status s = fa_common(T, coords, restype, lengths, B, Lmax, atom_stride, workspace, ws_bytes);
    if (s != TPL_OK) return s;
    if (!T->xyz_ok) return fail(TPL_ERR_TABLE, "table cannot back-propagate from coordinates: %s", T->xyz_why.c_str());
    if (Lmax > kFAXMaxL) return fail(TPL_ERR_SHAPE, "Lmax=%d > %d (the chain's types are staged on chip)", Lmax, kFAXMaxL);
    if (!grad_coords || !grad_angles) return fail(TPL_ERR_NULL, "grad_coords/grad_angles is NULL");
    if (!aligned4(grad_coords) || !aligned4(grad_angles)) return fail(TPL_ERR_ALIGN, "grads not 4-byte aligned");
    FAArgs a = fa_args(T, nullptr, restype, lengths, B, Lmax, atom_stride, workspace);
    a.coords = const_cast<float*>(coords);
    a.grad_coords = grad_coords;
    a.grad_angles = grad_angles;
    cudaError_t e = fa_backward_xyz_launch(a, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "full-atom backward (from coords) launch");
    return TPL_OK;
}

int32_t tpl_tables_backward_from_coords_ok(const tpl_tables* T) { return T && T->xyz_ok ? 1 : 0; }

// ---------------------------------------------------------------- LRMSD
static tpl_status lr_common(const float* x, const float* y, const int32_t* n_atoms, int32_t B, int32_t stride,
                            void* ws, size_t ws_bytes) {
    if (!x || !y || !n_atoms) return fail(TPL_ERR_NULL, "x/y/n_atoms is NULL");
    if (B < 1 || stride < 1) return fail(TPL_ERR_SHAPE, "B=%d stride=%d must be >= 1", B, stride);
    if (!aligned4(x) || !aligned4(y) || !aligned4(n_atoms)) return fail(TPL_ERR_ALIGN, "inputs not 4-byte aligned");
    if (!ws) return fail(TPL_ERR_WORKSPACE, "workspace is NULL");
    if (ws_bytes < kWsHeader) return fail(TPL_ERR_WORKSPACE, "workspace %zu bytes < %zu", ws_bytes, kWsHeader);
    return TPL_OK;
}

tpl_status tpl_lrmsd_forward(const float* x, const float* y, const int32_t* n_atoms, int32_t B, int32_t stride,
                             float* lrmsd, float* state, void* workspace, size_t ws_bytes, void* stream) {
    tpl_status s = lr_common(x, y, n_atoms, B, stride, workspace, ws_bytes);
    if (s != TPL_OK) return s;
    if (!lrmsd || !state) return fail(TPL_ERR_NULL, "lrmsd/state is NULL");
    LRArgs a{};
    a.x = x;
    a.y = y;
    a.n_atoms = n_atoms;
    a.B = B;
    a.stride = stride;
    a.out = lrmsd;
    a.state = state;
    a.err = static_cast<unsigned*>(workspace);
    cudaError_t e = lrmsd_forward_launch(a, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "lrmsd forward launch");
    return TPL_OK;
}

tpl_status tpl_lrmsd_backward(const float* x, const float* y, const int32_t* n_atoms, int32_t B, int32_t stride,
                              const float* state, const float* grad_lrmsd, float* grad_x, void* workspace,
                              size_t ws_bytes, void* stream) {
    tpl_status s = lr_common(x, y, n_atoms, B, stride, workspace, ws_bytes);
    if (s != TPL_OK) return s;
    if (!state || !grad_lrmsd || !grad_x) return fail(TPL_ERR_NULL, "state/grad_lrmsd/grad_x is NULL");
    LRArgs a{};
    a.x = x;
    a.y = y;
    a.n_atoms = n_atoms;
    a.B = B;
    a.stride = stride;
    a.state = const_cast<float*>(state);
    a.grad_out = grad_lrmsd;
    a.grad_x = grad_x;
    a.err = static_cast<unsigned*>(workspace);
    cudaError_t e = lrmsd_backward_launch(a, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "lrmsd backward launch");
    return TPL_OK;
}

}  // extern "C"
