// test_ref_backend.cpp -- TEST INFRASTRUCTURE: the reference's own driver through the
// reference-side binding (integration/voxreg/ffdp_backend.hpp).
//
// Built only where /root/reference exists (oracle/Makefile target `ref-backend`, output
// oracle/_ref/test_ref_backend, which travels to the GPU box like libvoxreg_ref.so): the
// UNMODIFIED reference headers are compiled with the shim, so deformable_stage<float>
// (registration.hpp:230-331) runs its ring_sample / dist_lncc / dist_mi /
// ring_sample_backward / gp_convolve on the B200 through libffdp.so, while
// deformable_stage<double> runs the reference's CPU templates. Prints one JSON object per
// loss with both loss traces and the warp difference; tests/test_gpu_ref_backend.py judges.
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "voxreg/registration.hpp"
#include "voxreg/synth.hpp"
#include "voxreg/ffdp_backend.hpp"

using namespace voxreg;

template <typename T>
Volume3<T> cast(const Volume3<double>& v) {
    Volume3<T> r = Volume3<T>::zeros(v.dims);
    r.spacing = v.spacing;
    r.origin = v.origin;
    for (std::size_t i = 0; i < v.data.size(); ++i) r.data[i] = static_cast<T>(v.data[i]);
    return r;
}

int main(int argc, char** argv) {
    const int n = argc > 1 ? std::atoi(argv[1]) : 48;
    const SynthPair sp = synth_pair(20261017, Dims3{n, n, n}, 4, 0.08);
    std::printf("[\n");
    const char* names[2] = {"lncc", "mi"};
    for (int which = 0; which < 2; ++which) {
        ScaleSchedule sch;
        sch.steps = {ScaleStep{2, 8}, ScaleStep{1, 6}};
        sch.loss.kind = which == 0 ? LossKind::lncc : LossKind::mi;
        sch.loss.mi_bspline_kernel = true;
        AffineMap id;
        std::vector<TraceEntry> t32, t64;
        const WarpField<float> w32 =
            deformable_stage<float>(cast<float>(sp.fixed), cast<float>(sp.moving), id, sch, {}, &t32);
        const WarpField<double> w64 = deformable_stage<double>(sp.fixed, sp.moving, id, sch, {}, &t64);
        double dmax = 0, wmax = 0, d2 = 0, w2 = 0;
        for (std::size_t i = 0; i < w64.data.size(); ++i) {
            const double d = static_cast<double>(w32.data[i]) - w64.data[i];
            dmax = std::max(dmax, std::abs(d));
            wmax = std::max(wmax, std::abs(w64.data[i]));
            d2 += d * d;
            w2 += w64.data[i] * w64.data[i];
        }
        std::printf("  {\"loss\": \"%s\", \"n\": %d, \"trace_ffdp_f32\": [", names[which], n);
        for (std::size_t i = 0; i < t32.size(); ++i) std::printf("%s%.17g", i ? ", " : "", t32[i].loss);
        std::printf("], \"trace_ref_f64\": [");
        for (std::size_t i = 0; i < t64.size(); ++i) std::printf("%s%.17g", i ? ", " : "", t64[i].loss);
        std::printf("], \"warp_maxabs_diff\": %.6g, \"warp_maxabs\": %.6g, \"warp_l2rel\": %.6g}%s\n", dmax, wmax,
                    std::sqrt(d2 / (w2 > 0 ? w2 : 1.0)), which == 0 ? "," : "");
    }
    std::printf("]\n");
    return 0;
}
