// Operator dispatch shared by the C-ABI and the solvers: projector model (Joseph /
// Siddon) x precision (f32 performance kernels / f64 exact-parity kernels) x
// backprojector variant (projector.hpp:283-297).
#include <cstdio>

#include "ctk_internal.h"

namespace ctkb {

// z-slab sharding is implemented for the f32 Joseph operators (the C5 path of SURVEY.md 8(d))
template <class T>
void require_slab_support(const Geometry& g) {
    if (g.slab && (sizeof(T) != 4 || g.projector != CTK_PROJ_JOSEPH))
        fail(CTK_E_UNSUPPORTED, "z-slab sharding is implemented for the f32 Joseph operators only");
}

// Checked builds (make checked -> lib/checked/libctk_b200.so, -DCTK_CHECKED): the kernels
// record every out-of-range index they would have used (and use a safe one instead) as bits
// in g.d_chk; each operator application synchronises and fails on any recorded bit.  This is
// the memory-safety check that stands in for compute-sanitizer, which this GPU pool disallows.
static void check_bounds(Geometry& g, cudaStream_t s, const char* what) {
#ifdef CTK_CHECKED
    unsigned bits = 0;
    CTK_CUDA(cudaStreamSynchronize(s));
    CTK_CUDA(cudaMemcpy(&bits, g.d_chk.p, sizeof bits, cudaMemcpyDeviceToHost));
    if (bits) {
        CTK_CUDA(cudaMemset(g.d_chk.p, 0, sizeof bits));
        fail(CTK_E_CUDA, std::string("checked build: out-of-range index in ") + what + " (bits 0x" +
                             [&] { char b[16]; std::snprintf(b, sizeof b, "%x", bits); return std::string(b); }() + ")");
    }
#else
    (void)g;
    (void)s;
    (void)what;
#endif
}

template <class T>
void op_ax(Geometry& g, const T* x, T* y, cudaStream_t s) {
    require_slab_support<T>(g);
    if constexpr (sizeof(T) == 4) {
        ax_f32(g, x, y, s);  // Joseph or the f32 Siddon slab model; records its own events
    } else if (g.projector == CTK_PROJ_SIDDON) {
        CTK_CUDA(cudaEventRecord(g.ev0, s));
        siddon_ax<T>(g, x, y, s);
        CTK_CUDA(cudaEventRecord(g.ev1, s));
    } else {
        CTK_CUDA(cudaEventRecord(g.ev0, s));
        launch_ax_exact_f64(g, x, y, s);
        CTK_CUDA(cudaEventRecord(g.ev1, s));
    }
    check_bounds(g, s, "Ax");
}

template <class T>
void op_atb(Geometry& g, int variant, const T* y, T* x, cudaStream_t s) {
    if (variant != CTK_BP_MATCHED && variant != CTK_BP_VOXEL_DRIVEN) fail(CTK_E_PARAMETER, "unknown backprojector variant");
    require_slab_support<T>(g);
    if (variant == CTK_BP_MATCHED && g.projector == CTK_PROJ_SIDDON && sizeof(T) == 8) {
        CTK_CUDA(cudaEventRecord(g.ev0, s));
        siddon_atb<T>(g, y, x, s);
        CTK_CUDA(cudaEventRecord(g.ev1, s));
    } else if constexpr (sizeof(T) == 4) {
        if (variant == CTK_BP_MATCHED) atb_matched_f32(g, y, x, s);
        else atb_voxel_f32(g, y, x, s);
    } else {
        CTK_CUDA(cudaEventRecord(g.ev0, s));
        if (variant == CTK_BP_MATCHED) launch_atb_matched_exact_f64(g, y, x, s);
        else launch_atb_voxel_f64(g, y, x, s);
        CTK_CUDA(cudaEventRecord(g.ev1, s));
    }
    check_bounds(g, s, "A^T b");
}

template void op_ax<float>(Geometry&, const float*, float*, cudaStream_t);
template void op_ax<double>(Geometry&, const double*, double*, cudaStream_t);
template void op_atb<float>(Geometry&, int, const float*, float*, cudaStream_t);
template void op_atb<double>(Geometry&, int, const double*, double*, cudaStream_t);

}  // namespace ctkb
