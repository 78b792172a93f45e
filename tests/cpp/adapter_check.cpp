// Drives the C++ adapter (include/fastmtgp_b200.hpp) exactly as the reference's GpModel drives
// fast_gram.hpp: build_spectrum(R_internal, spatial, xi) -> invert_and_logdet -> solve.
// Input (stdin, whitespace separated):
//   kind d L  m[L]  n_max g[d] | m_cols columns[d*m_cols]   shift_bits[L*d]
//   gamma si_alpha b[4] eta[d]  R[L*L]  xi[L]  N  y[N]
// Output: "logdet <v>" then "x <N values>".  Exit 0 ok, 2 SchurBreakdown, 3 FastMtgpError.
#include <cstdio>
#include <iostream>

#include "fastmtgp_b200.hpp"

int main() {
    using namespace fastmtgp_b200;
    Design dz;
    int L;
    std::cin >> dz.kind >> dz.d >> L;
    dz.m.resize(L);
    for (auto& v : dz.m) std::cin >> v;
    if (dz.kind == 0) {
        std::cin >> dz.n_max;
        dz.g.resize(dz.d);
        for (auto& v : dz.g) std::cin >> v;
    } else {
        std::cin >> dz.m_cols;
        dz.columns.resize(std::size_t(dz.d) * dz.m_cols);
        for (auto& v : dz.columns) std::cin >> v;
    }
    dz.shift_bits.resize(std::size_t(L) * dz.d);
    for (auto& v : dz.shift_bits) std::cin >> v;
    Spatial q;
    std::cin >> q.gamma >> q.si_alpha >> q.b[0] >> q.b[1] >> q.b[2] >> q.b[3];
    q.eta.resize(dz.d);
    for (auto& v : q.eta) std::cin >> v;
    std::vector<double> R(std::size_t(L) * L), xi(L);
    for (auto& v : R) std::cin >> v;
    for (auto& v : xi) std::cin >> v;
    std::size_t N;
    std::cin >> N;
    std::vector<double> y(N);
    for (auto& v : y) std::cin >> v;
    try {
        Session s(dz);
        s.build_spectrum(R, q, xi);
        const double ld = s.invert_and_logdet();
        const std::vector<double> x = s.solve(y);
        std::printf("logdet %.17g\nx", ld);
        for (double v : x) std::printf(" %.17g", v);
        std::printf("\n");
    } catch (const SchurBreakdown& e) {
        std::fprintf(stderr, "SchurBreakdown: %s\n", e.what());
        return 2;
    } catch (const FastMtgpError& e) {
        std::fprintf(stderr, "FastMtgpError: %s\n", e.what());
        return 3;
    }
    return 0;
}
