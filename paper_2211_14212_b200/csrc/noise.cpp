// Count-domain CT noise, the reference's add_noise (noise.hpp:26-47), host side.
//
// The sampling scheme is a single mt19937_64 stream consumed in detector-index order, one
// Poisson draw then (sigma > 0) one Gaussian draw per sample -- a sequential dependency
// chain with data-dependent draw counts (the Poisson sampler rejects), so there is nothing
// to parallelise without changing the stream; it is data preparation, not solver work,
// and runs once per simulated acquisition.  Using the same standard-library engine and
// distributions makes the output bit-identical to the reference built against the same
// libstdc++ (tests/test_pipeline.py).  The Gaussian distribution object lives across
// samples, as in the reference, because it caches the second value of each polar pair.
#include <algorithm>
#include <cmath>
#include <random>

#include "ctk_internal.h"

namespace ctkb {

template <class T>
void add_noise(size_t n, const T* in, double i0, double sigma, uint64_t seed, T* out) {
    if (!(i0 > 0.0)) fail(CTK_E_PARAMETER, "noise model: I0 must be positive");        // NoiseModel::validate
    if (sigma < 0.0) fail(CTK_E_PARAMETER, "noise model: sigma must be nonnegative");
    if (n > 0 && (in == nullptr || out == nullptr)) fail(CTK_E_PARAMETER, "add_noise: null buffer");
    for (size_t i = 0; i < n; ++i)
        if (!(in[i] >= T(0))) fail(CTK_E_DEGENERATE, "add_noise: negative line integral");
    std::mt19937_64 rng(seed);
    std::normal_distribution<double> gauss(0.0, sigma);
    const double log_i0 = std::log(i0);
    for (size_t i = 0; i < n; ++i) {
        const double counts = i0 * std::exp(-double(in[i]));
        double noisy = double(std::poisson_distribution<long long>(counts)(rng));
        if (sigma > 0.0) noisy += gauss(rng);
        noisy = std::max(noisy, 1.0);
        out[i] = T(log_i0 - std::log(noisy));
    }
}

template void add_noise<float>(size_t, const float*, double, double, uint64_t, float*);
template void add_noise<double>(size_t, const double*, double, double, uint64_t, double*);

}  // namespace ctkb
