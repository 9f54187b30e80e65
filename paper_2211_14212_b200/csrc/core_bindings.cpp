// _core -- the reference's pybind11 module (bindings/bindings.cpp:1-2, CMakeLists.txt:33-45:
// `pybind11_add_module(_core ...)`, installed into the `ctkrylov` package), which the reference
// ships empty.  Same module name, filled in over the C-ABI (include/ctk_b200.h): the
// reference's types and entry points with the names of geometry.hpp, types.hpp,
// operators.hpp, solve_log.hpp, solvers.hpp, hybrid.hpp and tv.hpp, on host (numpy) buffers.
// Every call goes through the same native entry points as the ctypes mirror (api.py), so
// both faces return bit-identical results (tests/test_gpu_core.py).
//
// Built in-tree by __graft_entry__.build() / `make -C paper_2211_14212_b200/csrc core`:
// paper_2211_14212_b200/_core<EXT_SUFFIX>, rpath $ORIGIN/lib -> lib/libctk_b200.so.
#include <pybind11/numpy.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include <cmath>
#include <memory>
#include <numbers>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/ctk_b200.h"

namespace py = pybind11;

namespace {

// ---- errors: the reference taxonomy (types.hpp:14-31) -----------------------------------
struct CtkError : std::runtime_error {
    int code, iteration;
    CtkError(int c, const std::string& m, int it) : std::runtime_error(m), code(c), iteration(it) {}
};
[[noreturn]] void raise_status(int rc) {
    char msg[512];
    ctk_last_error(msg, sizeof msg);
    throw CtkError(rc, msg, ctk_last_error_iteration());
}
void check(int rc) {
    if (rc != CTK_OK) raise_status(rc);
}
[[noreturn]] void fail(int code, const char* msg) { throw CtkError(code, msg, -1); }

enum class BeamMode { parallel2d = CTK_PARALLEL2D, parallel3d = CTK_PARALLEL3D, cone3d = CTK_CONE3D };
enum class BackprojectVariant { matched = CTK_BP_MATCHED, voxel_driven = CTK_BP_VOXEL_DRIVEN };
enum class ProjectorKind { joseph = CTK_PROJ_JOSEPH, siddon = CTK_PROJ_SIDDON };
enum class StopReason {
    max_iters = CTK_STOP_MAX_ITERS,
    residual_increase = CTK_STOP_RESIDUAL_INCREASE,
    tolerance = CTK_STOP_TOLERANCE,
    breakdown = CTK_STOP_BREAKDOWN
};
enum class LambdaStrategy { fixed = CTK_LAMBDA_FIXED, dp = CTK_LAMBDA_DP, gcv = CTK_LAMBDA_GCV };

constexpr double kTwoPi = 2.0 * std::numbers::pi;
double canonical_angle(double a) {  // types.hpp:172-177
    double r = std::fmod(a, kTwoPi);
    if (r < 0.0) r += kTwoPi;
    return r;
}

// ---- geometry (types.hpp:35-41, geometry.hpp:24-87) -------------------------------------
struct VolumeShape {
    int nx = 0, ny = 0, nz = 0;
    double spacing = 1.0;
    size_t size() const { return size_t(nx) * ny * nz; }
};

struct ConeGeometry {
    BeamMode mode = BeamMode::parallel2d;
    double source_to_origin = 0.0, origin_to_detector = 0.0, detector_pixel_size = 1.0;
    int nu = 0, nv = 0;
    VolumeShape vol;
    std::vector<double> angles;

    ctk_geom_desc desc() const {
        ctk_geom_desc d{};
        d.mode = int(mode);
        d.source_to_origin = source_to_origin;
        d.origin_to_detector = origin_to_detector;
        d.detector_pixel_size = detector_pixel_size;
        d.nu = nu;
        d.nv = nv;
        d.nx = vol.nx;
        d.ny = vol.ny;
        d.nz = vol.nz;
        d.spacing = vol.spacing;
        d.n_angles = int(angles.size());
        d.angles = angles.data();
        return d;
    }
    void validate() const {  // geometry.hpp:35-54, the native checks (no device work)
        const ctk_geom_desc d = desc();
        check(ctk_geom_validate(&d));
    }
};

std::vector<double> equidistant_angles(int n, double start_rad, double range_rad) {  // geometry.hpp:57-64
    if (n <= 0) fail(CTK_E_GEOMETRY, "angle count must be positive");
    std::vector<double> a(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) a[size_t(i)] = canonical_angle(start_rad + range_rad * i / n);
    return a;
}

ConeGeometry default_geometry(BeamMode mode, const VolumeShape& vol, int n_angles, double range_rad) {  // :66-87
    ConeGeometry g;
    g.mode = mode;
    g.vol = vol;
    g.angles = equidistant_angles(n_angles, 0.0, range_rad);
    const int n = std::max(vol.nx, std::max(vol.ny, vol.nz));
    if (mode == BeamMode::cone3d) {
        g.source_to_origin = 2.0 * n * vol.spacing;
        g.origin_to_detector = 1.0 * n * vol.spacing;
        g.detector_pixel_size = 1.5 * vol.spacing;
        g.nu = g.nv = (3 * n) / 2;
    } else {
        g.origin_to_detector = 1.0 * n * vol.spacing;
        g.detector_pixel_size = vol.spacing;
        g.nu = (3 * n) / 2;
        g.nv = mode == BeamMode::parallel2d ? 1 : (3 * vol.nz) / 2;
    }
    g.validate();
    return g;
}

// ---- operator pair (operators.hpp:18-45, 91-115) ----------------------------------------
using Handle = std::shared_ptr<ctk_geom>;

struct OperatorPair {
    Handle h;
    size_t domain_size = 0, range_size = 0;
    bool matched = true;
    VolumeShape domain_shape;
    BackprojectVariant variant = BackprojectVariant::matched;
    bool f64 = false;

    void check_domain(size_t n) const {
        if (n != domain_size) fail(CTK_E_DIMENSION, "operator domain size mismatch");
    }
    void check_range(size_t n) const {
        if (n != range_size) fail(CTK_E_DIMENSION, "operator range size mismatch");
    }
    template <class T>
    py::array_t<T> fwd(py::array_t<T, py::array::c_style | py::array::forcecast> x) const {
        check_domain(size_t(x.size()));
        py::array_t<T> y(range_size);
        const T* xp = x.data();
        T* yp = y.mutable_data();
        int rc;
        {
            py::gil_scoped_release nogil;
            if constexpr (sizeof(T) == 4) rc = ctk_ax_host_f32(h.get(), xp, yp);
            else rc = ctk_ax_host_f64(h.get(), xp, yp);
        }
        check(rc);
        return y;
    }
    template <class T>
    py::array_t<T> back(py::array_t<T, py::array::c_style | py::array::forcecast> y) const {
        check_range(size_t(y.size()));
        py::array_t<T> x(domain_size);
        const T* yp = y.data();
        T* xp = x.mutable_data();
        int rc;
        {
            py::gil_scoped_release nogil;
            if constexpr (sizeof(T) == 4) rc = ctk_atb_host_f32(h.get(), int(variant), yp, xp);
            else rc = ctk_atb_host_f64(h.get(), int(variant), yp, xp);
        }
        check(rc);
        return x;
    }
    py::array apply_forward(const py::array& x) const { return f64 ? py::array(fwd<double>(x)) : py::array(fwd<float>(x)); }
    py::array apply_back(const py::array& y) const { return f64 ? py::array(back<double>(y)) : py::array(back<float>(y)); }
};

bool is_f64(const py::object& dtype) {
    const py::dtype dt = py::dtype::from_args(dtype);
    if (dt.kind() != 'f' || (dt.itemsize() != 4 && dt.itemsize() != 8))
        fail(CTK_E_PARAMETER, "projector_pair: dtype must be float32 or float64");
    return dt.itemsize() == 8;
}

OperatorPair projector_pair(const ConeGeometry& geom, BackprojectVariant variant, const py::object& dtype,
                            ProjectorKind projector) {
    geom.validate();
    const ctk_geom_desc d = geom.desc();  // angles are canonicalised natively (operators.hpp:96)
    ctk_geom* raw = nullptr;
    check(ctk_geom_create(&d, &raw));
    OperatorPair p;
    p.h = Handle(raw, ctk_geom_destroy);
    check(ctk_geom_set_projector(raw, int(projector)));
    check(ctk_geom_sizes(raw, &p.domain_size, &p.range_size));
    p.variant = variant;
    p.matched = variant == BackprojectVariant::matched;
    p.domain_shape = geom.vol;
    p.f64 = is_f64(dtype);
    return p;
}

// ---- solvers (solve_log.hpp:28-76, solvers.hpp, hybrid.hpp, tv.hpp) ---------------------
struct SolverOptions {
    int max_iters = 100;
    bool stop_on_explicit_residual_increase = true;
    double residual_tolerance = 1e-6;
    bool reorth = true;
    py::object ground_truth = py::none();
    void validate() const {
        if (max_iters < 1) fail(CTK_E_PARAMETER, "max_iters must be >= 1");
        if (residual_tolerance < 0.0) fail(CTK_E_PARAMETER, "residual tolerance must be >= 0");
    }
};

struct HybridStrategy {
    LambdaStrategy kind = LambdaStrategy::fixed;
    double lambda_ = 0.0, noise_level = 0.0;
    static HybridStrategy fixed(double lam) {
        if (lam < 0.0) fail(CTK_E_PARAMETER, "fixed lambda must be nonnegative");
        return {LambdaStrategy::fixed, lam, 0.0};
    }
    static HybridStrategy dp(double nl) {
        if (!(nl > 0.0 && nl < 1.0)) fail(CTK_E_PARAMETER, "dp strategy needs a noise level in (0,1)");
        return {LambdaStrategy::dp, 0.0, nl};
    }
    static HybridStrategy gcv() { return {LambdaStrategy::gcv, 0.0, 0.0}; }
};

struct ConvergenceLog {
    std::vector<double> implicit_residual, explicit_residual, relative_error, lambda_;
    std::string solver, precision;
    bool matched = true;
    size_t iterations() const { return explicit_residual.size(); }
};

struct SolveResult {
    py::array x;
    VolumeShape shape;
    int iterations_run = 0;
    StopReason stop_reason = StopReason::max_iters;
    ConvergenceLog log;
    std::vector<int> outer_starts;
    int stored_domain_basis = 0, stored_range_basis = 0;
    std::vector<std::string> warnings;
};

enum class Solver { cgls, lsqr, lsmr, hybrid_lsqr, cgls_tv, sirt, ab_gmres, ba_gmres, flsqr_tv };
const char* solver_name(Solver s) {
    static const char* n[] = {"cgls", "lsqr", "lsmr", "hybrid_lsqr", "cgls_tv", "sirt", "ab_gmres", "ba_gmres", "flsqr_tv"};
    return n[int(s)];
}

struct SolveArgs {
    double lambda = 0.0;
    const HybridStrategy* strategy = nullptr;
    int outer = 1, inner = 1;
    bool warm = false;
};

template <class T>
SolveResult solve_t(Solver s, const OperatorPair& pair, const py::array& b_in, const SolverOptions& opts,
                    const SolveArgs& a) {
    py::array_t<T, py::array::c_style | py::array::forcecast> b(b_in);
    pair.check_range(size_t(b.size()));
    py::array_t<T, py::array::c_style | py::array::forcecast> gt;
    if (!opts.ground_truth.is_none()) {
        gt = py::array_t<T, py::array::c_style | py::array::forcecast>(opts.ground_truth);
        pair.check_domain(size_t(gt.size()));
    }
    const int cap = s == Solver::cgls_tv ? a.outer * a.inner : opts.max_iters;
    std::vector<double> imp(size_t(cap) + 1), expl(size_t(cap) + 1), rel(size_t(cap) + 1), lam(size_t(cap) + 1);
    std::vector<int> starts(size_t(a.outer) + 1), wits(size_t(cap) + 1);
    ctk_solve_log log{};
    log.capacity = cap;
    log.implicit_residual = imp.data();
    log.explicit_residual = expl.data();
    log.relative_error = rel.data();
    log.lambda = lam.data();
    log.outer_starts = starts.data();
    log.warning_iterations = wits.data();
    ctk_solver_opts o{};
    o.max_iters = opts.max_iters;
    o.stop_on_explicit_residual_increase = opts.stop_on_explicit_residual_increase;
    o.residual_tolerance = opts.residual_tolerance;
    o.reorth = opts.reorth;
    o.ground_truth = gt ? static_cast<const void*>(gt.data()) : nullptr;
    ctk_hybrid_strategy st{};
    if (a.strategy) {
        st.kind = int(a.strategy->kind);
        st.lambda = a.strategy->lambda_;
        st.noise_level = a.strategy->noise_level;
    }
    py::array_t<T> x(pair.domain_size);
    const T* bp = b.data();
    T* xp = x.mutable_data();
    ctk_geom* g = pair.h.get();
    const int v = int(pair.variant);
    constexpr bool F = sizeof(T) == 4;
    int rc;
    {
        py::gil_scoped_release nogil;
        switch (s) {
            case Solver::cgls: rc = F ? ctk_cgls_f32(g, v, (const float*)bp, &o, (float*)xp, &log)
                                      : ctk_cgls_f64(g, v, (const double*)bp, &o, (double*)xp, &log); break;
            case Solver::lsqr: rc = F ? ctk_lsqr_f32(g, v, (const float*)bp, &o, (float*)xp, &log)
                                      : ctk_lsqr_f64(g, v, (const double*)bp, &o, (double*)xp, &log); break;
            case Solver::sirt: rc = F ? ctk_sirt_f32(g, v, (const float*)bp, &o, (float*)xp, &log)
                                      : ctk_sirt_f64(g, v, (const double*)bp, &o, (double*)xp, &log); break;
            case Solver::ab_gmres: rc = F ? ctk_ab_gmres_f32(g, v, (const float*)bp, &o, (float*)xp, &log)
                                          : ctk_ab_gmres_f64(g, v, (const double*)bp, &o, (double*)xp, &log); break;
            case Solver::ba_gmres: rc = F ? ctk_ba_gmres_f32(g, v, (const float*)bp, &o, (float*)xp, &log)
                                          : ctk_ba_gmres_f64(g, v, (const double*)bp, &o, (double*)xp, &log); break;
            case Solver::lsmr: rc = F ? ctk_lsmr_f32(g, v, (const float*)bp, a.lambda, &o, (float*)xp, &log)
                                      : ctk_lsmr_f64(g, v, (const double*)bp, a.lambda, &o, (double*)xp, &log); break;
            case Solver::hybrid_lsqr:
                rc = F ? ctk_hybrid_lsqr_f32(g, v, (const float*)bp, &st, &o, (float*)xp, &log)
                       : ctk_hybrid_lsqr_f64(g, v, (const double*)bp, &st, &o, (double*)xp, &log); break;
            case Solver::flsqr_tv:
                rc = F ? ctk_flsqr_tv_f32(g, v, (const float*)bp, &st, &o, (float*)xp, &log)
                       : ctk_flsqr_tv_f64(g, v, (const double*)bp, &st, &o, (double*)xp, &log); break;
            default:
                rc = F ? ctk_cgls_tv_f32(g, v, (const float*)bp, a.lambda, a.outer, a.inner, &o, a.warm, (float*)xp, &log)
                       : ctk_cgls_tv_f64(g, v, (const double*)bp, a.lambda, a.outer, a.inner, &o, a.warm, (double*)xp, &log);
        }
    }
    check(rc);
    SolveResult r;
    r.x = x;
    r.shape = pair.domain_shape;
    r.iterations_run = log.iterations_run;
    r.stop_reason = StopReason(log.stop_reason);
    r.log.implicit_residual.assign(imp.begin(), imp.begin() + log.iterations);
    r.log.explicit_residual.assign(expl.begin(), expl.begin() + log.iterations);
    r.log.relative_error.assign(rel.begin(), rel.begin() + log.n_relative_error);
    r.log.lambda_.assign(lam.begin(), lam.begin() + log.n_lambda);
    r.log.solver = solver_name(s);
    r.log.precision = F ? "single" : "double";
    r.log.matched = pair.matched;
    r.outer_starts.assign(starts.begin(), starts.begin() + log.n_outer_starts);
    r.stored_domain_basis = log.stored_domain_basis;
    r.stored_range_basis = log.stored_range_basis;
    for (int i = 0; i < log.n_warnings; ++i)
        r.warnings.push_back("tv preconditioner: inner CG not converged at iteration " + std::to_string(wits[size_t(i)]));
    return r;
}

SolveResult solve(Solver s, const OperatorPair& pair, const py::array& b, const SolverOptions& opts,
                  const SolveArgs& a = {}) {
    opts.validate();
    return pair.f64 ? solve_t<double>(s, pair, b, opts, a) : solve_t<float>(s, pair, b, opts, a);
}

}  // namespace

PYBIND11_MODULE(_core, m) {
    m.doc() = "ctkrylov _core on sm_100a: the reference's types, projector pair and solvers over libctk_b200";

    // exception classes, the reference's names (types.hpp:14-31); NumericalError carries .iteration
    static py::exception<CtkError> base(m, "CtkError", PyExc_RuntimeError);
    static const char* names[] = {nullptr, "DimensionError", "GeometryError", "ParameterError",
                                  "DegenerateInputError", "NumericalError", "CudaError", "UnsupportedError"};
    static py::object cls[8];
    for (int c = 1; c < 8; ++c) {
        cls[c] = py::reinterpret_steal<py::object>(
            PyErr_NewException((std::string("paper_2211_14212_b200._core.") + names[c]).c_str(), base.ptr(), nullptr));
        m.attr(names[c]) = cls[c];
    }
    py::register_exception_translator([](std::exception_ptr p) {
        try {
            if (p) std::rethrow_exception(p);
        } catch (const CtkError& e) {
            const int c = (e.code >= 1 && e.code < 8) ? e.code : CTK_E_CUDA;
            py::object inst = cls[c](e.what());
            inst.attr("iteration") = e.iteration;
            PyErr_SetObject(cls[c].ptr(), inst.ptr());
        }
    });

    py::enum_<BeamMode>(m, "BeamMode")
        .value("parallel2d", BeamMode::parallel2d)
        .value("parallel3d", BeamMode::parallel3d)
        .value("cone3d", BeamMode::cone3d);
    py::enum_<BackprojectVariant>(m, "BackprojectVariant")
        .value("matched", BackprojectVariant::matched)
        .value("voxel_driven", BackprojectVariant::voxel_driven);
    py::enum_<ProjectorKind>(m, "ProjectorKind").value("joseph", ProjectorKind::joseph).value("siddon", ProjectorKind::siddon);
    py::enum_<StopReason>(m, "StopReason")
        .value("max_iters", StopReason::max_iters)
        .value("residual_increase", StopReason::residual_increase)
        .value("tolerance", StopReason::tolerance)
        .value("breakdown", StopReason::breakdown);
    py::enum_<LambdaStrategy>(m, "LambdaStrategy")
        .value("fixed", LambdaStrategy::fixed)
        .value("dp", LambdaStrategy::dp)
        .value("gcv", LambdaStrategy::gcv);

    py::class_<VolumeShape>(m, "VolumeShape")
        .def(py::init<>())
        .def(py::init([](int nx, int ny, int nz, double sp) { return VolumeShape{nx, ny, nz, sp}; }), py::arg("nx"),
             py::arg("ny"), py::arg("nz"), py::arg("spacing") = 1.0)
        .def_readwrite("nx", &VolumeShape::nx)
        .def_readwrite("ny", &VolumeShape::ny)
        .def_readwrite("nz", &VolumeShape::nz)
        .def_readwrite("spacing", &VolumeShape::spacing)
        .def("size", &VolumeShape::size);
    py::class_<ConeGeometry>(m, "ConeGeometry")
        .def(py::init<>())
        .def_readwrite("mode", &ConeGeometry::mode)
        .def_readwrite("source_to_origin", &ConeGeometry::source_to_origin)
        .def_readwrite("origin_to_detector", &ConeGeometry::origin_to_detector)
        .def_readwrite("detector_pixel_size", &ConeGeometry::detector_pixel_size)
        .def_readwrite("nu", &ConeGeometry::nu)
        .def_readwrite("nv", &ConeGeometry::nv)
        .def_readwrite("vol", &ConeGeometry::vol)
        .def_readwrite("angles", &ConeGeometry::angles)
        .def("validate", &ConeGeometry::validate);
    m.def("canonical_angle", &canonical_angle);
    m.def("equidistant_angles", &equidistant_angles, py::arg("n"), py::arg("start_rad") = 0.0,
          py::arg("range_rad") = kTwoPi);
    m.def("default_geometry", &default_geometry, py::arg("mode"), py::arg("vol"), py::arg("n_angles"),
          py::arg("range_rad") = kTwoPi);

    py::class_<OperatorPair>(m, "OperatorPair")
        .def_readonly("domain_size", &OperatorPair::domain_size)
        .def_readonly("range_size", &OperatorPair::range_size)
        .def_readonly("matched", &OperatorPair::matched)
        .def_readonly("domain_shape", &OperatorPair::domain_shape)
        .def_readonly("variant", &OperatorPair::variant)
        .def_property_readonly("dtype", [](const OperatorPair& p) { return py::dtype(p.f64 ? "float64" : "float32"); })
        .def("check_domain", &OperatorPair::check_domain)
        .def("check_range", &OperatorPair::check_range)
        .def("apply_forward", &OperatorPair::apply_forward)
        .def("apply_back", &OperatorPair::apply_back);
    m.def("projector_pair", &projector_pair, py::arg("geom"), py::arg("variant") = BackprojectVariant::matched,
          py::arg("dtype") = py::str("float32"), py::arg("projector") = ProjectorKind::joseph);

    py::class_<SolverOptions>(m, "SolverOptions")
        .def(py::init<>())
        .def(py::init([](int mi, bool stop, double tol, bool reorth, py::object gt) {
                 SolverOptions o;
                 o.max_iters = mi;
                 o.stop_on_explicit_residual_increase = stop;
                 o.residual_tolerance = tol;
                 o.reorth = reorth;
                 o.ground_truth = gt;
                 return o;
             }),
             py::arg("max_iters") = 100, py::arg("stop_on_explicit_residual_increase") = true,
             py::arg("residual_tolerance") = 1e-6, py::arg("reorth") = true, py::arg("ground_truth") = py::none())
        .def_readwrite("max_iters", &SolverOptions::max_iters)
        .def_readwrite("stop_on_explicit_residual_increase", &SolverOptions::stop_on_explicit_residual_increase)
        .def_readwrite("residual_tolerance", &SolverOptions::residual_tolerance)
        .def_readwrite("reorth", &SolverOptions::reorth)
        .def_readwrite("ground_truth", &SolverOptions::ground_truth)
        .def("validate", &SolverOptions::validate);
    py::class_<HybridStrategy>(m, "HybridStrategy")
        .def_readonly("kind", &HybridStrategy::kind)
        .def_readonly("lambda_", &HybridStrategy::lambda_)
        .def_readonly("noise_level", &HybridStrategy::noise_level)
        .def_static("fixed", &HybridStrategy::fixed)
        .def_static("dp", &HybridStrategy::dp)
        .def_static("gcv", &HybridStrategy::gcv);
    py::class_<ConvergenceLog>(m, "ConvergenceLog")
        .def_readonly("implicit_residual", &ConvergenceLog::implicit_residual)
        .def_readonly("explicit_residual", &ConvergenceLog::explicit_residual)
        .def_readonly("relative_error", &ConvergenceLog::relative_error)
        .def_readonly("lambda_", &ConvergenceLog::lambda_)
        .def_readonly("solver", &ConvergenceLog::solver)
        .def_readonly("precision", &ConvergenceLog::precision)
        .def_readonly("matched", &ConvergenceLog::matched)
        .def("iterations", &ConvergenceLog::iterations);
    py::class_<SolveResult>(m, "SolveResult")
        .def_readonly("x", &SolveResult::x)
        .def_readonly("shape", &SolveResult::shape)
        .def_readonly("iterations_run", &SolveResult::iterations_run)
        .def_readonly("stop_reason", &SolveResult::stop_reason)
        .def_readonly("log", &SolveResult::log)
        .def_readonly("outer_starts", &SolveResult::outer_starts)
        .def_readonly("stored_domain_basis", &SolveResult::stored_domain_basis)
        .def_readonly("stored_range_basis", &SolveResult::stored_range_basis)
        .def_readonly("warnings", &SolveResult::warnings);

    const auto O = py::arg("opts");
    m.def("cgls", [](const OperatorPair& p, const py::array& b, const SolverOptions& o) { return solve(Solver::cgls, p, b, o); },
          py::arg("pair"), py::arg("b"), O);
    m.def("lsqr", [](const OperatorPair& p, const py::array& b, const SolverOptions& o) { return solve(Solver::lsqr, p, b, o); },
          py::arg("pair"), py::arg("b"), O);
    m.def("sirt", [](const OperatorPair& p, const py::array& b, const SolverOptions& o) { return solve(Solver::sirt, p, b, o); },
          py::arg("pair"), py::arg("b"), O);
    m.def("ab_gmres", [](const OperatorPair& p, const py::array& b, const SolverOptions& o) {
        return solve(Solver::ab_gmres, p, b, o); }, py::arg("pair"), py::arg("b"), O);
    m.def("ba_gmres", [](const OperatorPair& p, const py::array& b, const SolverOptions& o) {
        return solve(Solver::ba_gmres, p, b, o); }, py::arg("pair"), py::arg("b"), O);
    m.def("lsmr", [](const OperatorPair& p, const py::array& b, double lam, const SolverOptions& o) {
        o.validate();
        if (lam < 0.0) fail(CTK_E_PARAMETER, "lsmr: lambda must be nonnegative");
        SolveArgs a;
        a.lambda = lam;
        return solve(Solver::lsmr, p, b, o, a); }, py::arg("pair"), py::arg("b"), py::arg("lambda_"), O);
    m.def("hybrid_lsqr", [](const OperatorPair& p, const py::array& b, const HybridStrategy& s, const SolverOptions& o) {
        SolveArgs a;
        a.strategy = &s;
        return solve(Solver::hybrid_lsqr, p, b, o, a); }, py::arg("pair"), py::arg("b"), py::arg("strategy"), O);
    m.def("flsqr_tv", [](const OperatorPair& p, const py::array& b, const HybridStrategy& s, const SolverOptions& o) {
        if (s.kind == LambdaStrategy::dp) fail(CTK_E_PARAMETER, "flsqr_tv: dp strategy is not supported, use fixed or gcv");
        SolveArgs a;
        a.strategy = &s;
        return solve(Solver::flsqr_tv, p, b, o, a); }, py::arg("pair"), py::arg("b"), py::arg("strategy"), O);
    m.def("cgls_tv", [](const OperatorPair& p, const py::array& b, double lam, int outer, int inner,
                        const SolverOptions& o, bool warm) {
        SolveArgs a;
        a.lambda = lam;
        a.outer = outer;
        a.inner = inner;
        a.warm = warm;
        return solve(Solver::cgls_tv, p, b, o, a); }, py::arg("pair"), py::arg("b"), py::arg("lambda_"),
        py::arg("outer_iters"), py::arg("inner_iters"), O, py::arg("warm_start") = false);
    m.attr("abi_version") = ctk_abi_version();
}
