// TEST INFRASTRUCTURE: exercises include/ctkrylov_b200/ctkrylov_b200.hpp against the
// UNMODIFIED reference headers.  Built by oracle/Makefile into oracle/_ref/dropin_test
// (needs /root/reference at compile time only); run by tests/test_gpu_dropin.py.
//  1. ctkb::projector_pair<double> is bit-identical to ctk::projector_pair<double>.
//  2. The reference's own CPU lsqr accepts the B200 pair (OperatorPair compatibility).
//  3. The device-resident ctkb::lsqr / lsmr / cgls / sirt / ab_gmres / ba_gmres match the
//     reference solvers (gmres.hpp compiled against the test-only Eigen shim).
//  4. Errors come back as the reference's exception types.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>

#include "ctkrylov/gmres.hpp"
#include "ctkrylov/tv.hpp"
#include "ctkrylov/operators.hpp"
#include "ctkrylov/phantom.hpp"
#include "ctkrylov/solvers.hpp"
#include "ctkrylov_b200/ctkrylov_b200.hpp"

static int failures = 0;
#define EXPECT(c)                                                        \
    do {                                                                 \
        if (!(c)) {                                                      \
            std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #c); \
            ++failures;                                                  \
        }                                                                \
    } while (0)

static double rel(const std::vector<double>& a, const std::vector<double>& b) {
    double n = 0, d = 0;
    for (size_t i = 0; i < a.size(); ++i) {
        n += (a[i] - b[i]) * (a[i] - b[i]);
        d += b[i] * b[i];
    }
    return std::sqrt(n / d);
}

int main() {
    ctk::ConeGeometry g = ctk::default_geometry(ctk::BeamMode::cone3d, {16, 16, 16, 1.0}, 12);
    auto ref = ctk::projector_pair<double>(g);
    auto b200 = ctkb::projector_pair<double>(g);
    std::mt19937_64 rng(7);
    std::normal_distribution<double> nd;
    std::vector<double> x(ref.domain_size), y(ref.range_size);
    for (auto& v : x) v = nd(rng);
    for (auto& v : y) v = nd(rng);
    EXPECT(ref.apply_forward(ctk::cspan(x)) == b200.apply_forward(ctk::cspan(x)));
    EXPECT(ref.apply_back(ctk::cspan(y)) == b200.apply_back(ctk::cspan(y)));

    const auto gt = ctk::make_phantom<double>(ctk::PhantomKind::shepp_logan_3d, 16);
    const auto b = ref.apply_forward(ctk::cspan(gt.data));
    ctk::SolverOptions<double> opts;
    opts.max_iters = 8;
    opts.residual_tolerance = 0.0;
    opts.stop_on_explicit_residual_increase = false;
    const auto r_ref = ctk::lsqr(ref, ctk::cspan(b), opts);
    const auto r_cpu_on_b200 = ctk::lsqr<double>(b200, ctk::cspan(b), opts);  // reference solver, B200 operators
    EXPECT(r_ref.x == r_cpu_on_b200.x);
    const auto r_dev = ctkb::lsqr(b200, ctk::cspan(b), opts);
    EXPECT(rel(r_dev.x, r_ref.x) < 1e-10);
    EXPECT(r_dev.log.explicit_residual.size() == r_ref.log.explicit_residual.size());
    for (size_t i = 0; i < r_ref.log.explicit_residual.size(); ++i)
        EXPECT(std::abs(r_dev.log.explicit_residual[i] - r_ref.log.explicit_residual[i]) <=
               1e-10 * r_ref.log.explicit_residual[i]);
    const auto m_ref = ctk::lsmr(ref, ctk::cspan(b), 3.0, opts);
    const auto m_dev = ctkb::lsmr(b200, ctk::cspan(b), 3.0, opts);
    EXPECT(rel(m_dev.x, m_ref.x) < 1e-10);
    EXPECT(m_dev.log.lambda == m_ref.log.lambda);
    const auto c_ref = ctk::cgls(ref, ctk::cspan(b), opts);
    const auto c_dev = ctkb::cgls(b200, ctk::cspan(b), opts);
    EXPECT(rel(c_dev.x, c_ref.x) < 1e-10);
    const auto s_ref = ctk::sirt(ref, ctk::cspan(b), opts);
    const auto s_dev = ctkb::sirt(b200, ctk::cspan(b), opts);
    EXPECT(rel(s_dev.x, s_ref.x) < 1e-10);
    EXPECT(s_dev.log.lambda.empty());
    const auto ab_ref = ctk::ab_gmres(ref, ctk::cspan(b), opts);
    const auto ab_dev = ctkb::ab_gmres(b200, ctk::cspan(b), opts);
    EXPECT(rel(ab_dev.x, ab_ref.x) < 1e-9);
    EXPECT(ab_dev.stored_range_basis == ab_ref.stored_range_basis);
    const auto ba_ref = ctk::ba_gmres(ref, ctk::cspan(b), opts);
    const auto ba_dev = ctkb::ba_gmres(b200, ctk::cspan(b), opts);
    EXPECT(rel(ba_dev.x, ba_ref.x) < 1e-9);
    EXPECT(ba_dev.stored_domain_basis == ba_ref.stored_domain_basis);
    const auto f_ref = ctk::flsqr_tv(ref, ctk::cspan(b), ctk::HybridStrategy::gcv(), opts);
    const auto f_dev = ctkb::flsqr_tv(b200, ctk::cspan(b), ctk::HybridStrategy::gcv(), opts);
    EXPECT(rel(f_dev.x, f_ref.x) < 1e-6);
    EXPECT(f_dev.warnings == f_ref.warnings);

    // f32 pair through the same API
    auto b32 = ctkb::projector_pair<float>(g);
    std::vector<float> xf(gt.data.begin(), gt.data.end());
    const auto yf = b32.apply_forward(ctk::cspan(xf));
    std::vector<double> yd(yf.begin(), yf.end());
    EXPECT(rel(yd, b) < 1e-5);

    // error taxonomy
    bool got = false;
    try {
        std::vector<double> wrong(5);
        b200.apply_forward(ctk::cspan(wrong));
    } catch (const ctk::DimensionError&) {
        got = true;
    }
    EXPECT(got);
    got = false;
    try {
        ctk::ConeGeometry bad = g;
        bad.source_to_origin = 2.0;
        ctkb::projector_pair<double>(bad);
    } catch (const ctk::GeometryError&) {
        got = true;
    }
    EXPECT(got);
    got = false;
    try {
        std::vector<double> zero(b.size(), 0.0);
        ctkb::lsqr(b200, ctk::cspan(zero), opts);
    } catch (const ctk::DegenerateInputError&) {
        got = true;
    }
    EXPECT(got);
    std::printf("dropin_test: %s (%d failures)\n", failures ? "FAILED" : "ok", failures);
    return failures ? 1 : 0;
}
