// construct.cpp -- code construction (non-hot, host; product code).
//
// The paper's codes are "constructed according to [Tal2011a]" at a design SNR it does not
// state.  Reading C1 of DESIGN.md: Gaussian approximation (GA) of the bit-channel
// LLR means for BPSK over AWGN, designed at the configuration's Eb/N0, freezing the N-K
// channels with the smallest mean (ties: the lower index is frozen).
//
// GA step for one polarisation level: a channel of mean m splits into a check-node
// ("minus") channel of mean phi^-1(1 - (1 - phi(m))^2) and a variable-node ("plus") channel
// of mean 2m.  With natural indexing the minus child of entry j is entry 2j and the
// plus child is 2j+1.  phi is Chung's two-piece approximation, handled in the log domain so
// that large means do not underflow.
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <numeric>
#include <vector>
#include <algorithm>

namespace polar {

// ln phi(x): -0.4527 x^0.86 + 0.0218 below 10, ln(sqrt(pi/x) e^{-x/4} (1 - 10/(7x))) above.
static double ga_ln_phi(double x) {
    if (x < 10.0) return -0.4527 * std::pow(x, 0.86) + 0.0218;
    return 0.5 * std::log(M_PI / x) - x / 4.0 + std::log(1.0 - 10.0 / (7.0 * x));
}

// The mean x >= 0 whose ln phi equals target (ln phi is decreasing): bracket, then bisect.
static double ga_ln_phi_inverse(double target) {
    double lo = 0.0, hi = 1.0;
    while (ga_ln_phi(hi) > target) hi *= 2.0;
    for (int step = 0; step < 200; ++step) {
        double mid = 0.5 * (lo + hi);
        if (ga_ln_phi(mid) > target) lo = mid;
        else hi = mid;
    }
    return 0.5 * (lo + hi);
}

void ga_means(int N, int K, double design_ebn0_db, std::vector<double>& mean) {
    const double rate = double(K) / double(N);
    const double sigma2 = 1.0 / (2.0 * rate * std::pow(10.0, design_ebn0_db / 10.0));
    std::vector<double> level(1, 2.0 / sigma2), next;
    while ((int)level.size() < N) {
        next.assign(level.size() * 2, 0.0);
        for (size_t j = 0; j < level.size(); ++j) {
            const double m = level[j];
            const double lp = ga_ln_phi(m);
            // 1 - (1 - p)^2 = p (2 - p)
            next[2 * j] = ga_ln_phi_inverse(lp + std::log(2.0 - std::exp(lp)));
            next[2 * j + 1] = 2.0 * m;
        }
        level.swap(next);
    }
    mean.swap(level);
}

void construct_ga(int N, int K, double design_ebn0_db, uint8_t* frozen) {
    std::vector<double> mean;
    ga_means(N, K, design_ebn0_db, mean);
    std::vector<int> order(N);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return mean[a] < mean[b]; });
    for (int i = 0; i < N; ++i) frozen[i] = 0;
    for (int t = 0; t < N - K; ++t) frozen[order[t]] = 1;
}

}  // namespace polar
