// Operator dispatch shared by the C-ABI and the solvers: projector model (Joseph /
// Siddon) x precision (f32 performance kernels / f64 exact-parity kernels) x
// backprojector variant (projector.hpp:283-297).
#include "ctk_internal.h"

namespace ctkb {

// z-slab sharding is implemented for the f32 Joseph operators (the C5 path of SURVEY.md 8(d))
template <class T>
void require_slab_support(const Geometry& g) {
    if (g.slab && (sizeof(T) != 4 || g.projector != CTK_PROJ_JOSEPH))
        fail(CTK_E_UNSUPPORTED, "z-slab sharding is implemented for the f32 Joseph operators only");
}

template <class T>
void op_ax(Geometry& g, const T* x, T* y, cudaStream_t s) {
    require_slab_support<T>(g);
    if (g.projector == CTK_PROJ_SIDDON) {
        CTK_CUDA(cudaEventRecord(g.ev0, s));
        siddon_ax<T>(g, x, y, s);
        CTK_CUDA(cudaEventRecord(g.ev1, s));
    } else if constexpr (sizeof(T) == 4) {
        ax_f32(g, x, y, s);  // records its own events around the main kernel
    } else {
        CTK_CUDA(cudaEventRecord(g.ev0, s));
        launch_ax_exact_f64(g, x, y, s);
        CTK_CUDA(cudaEventRecord(g.ev1, s));
    }
}

template <class T>
void op_atb(Geometry& g, int variant, const T* y, T* x, cudaStream_t s) {
    if (variant != CTK_BP_MATCHED && variant != CTK_BP_VOXEL_DRIVEN) fail(CTK_E_PARAMETER, "unknown backprojector variant");
    require_slab_support<T>(g);
    if (variant == CTK_BP_MATCHED && g.projector == CTK_PROJ_SIDDON) {
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
}

template void op_ax<float>(Geometry&, const float*, float*, cudaStream_t);
template void op_ax<double>(Geometry&, const double*, double*, cudaStream_t);
template void op_atb<float>(Geometry&, int, const float*, float*, cudaStream_t);
template void op_atb<double>(Geometry&, int, const double*, double*, cudaStream_t);

}  // namespace ctkb
