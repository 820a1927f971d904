// oracle/ref_io_shim.cpp -- TEST INFRASTRUCTURE ONLY: an extern "C" shim over the
// UNMODIFIED reference's NIfTI-1 / raw+JSON IO (proj/include/voxreg/nifti.hpp), used by
// tests/golden/make_golden.py to write and parse the IO golden fixtures. nifti.hpp needs
// nlohmann/json.hpp, which the reference vendors outside the repository (CMakeLists.txt:5);
// `make -C oracle ref-io` points -I at a copy of that header when one is found.
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "voxreg/nifti.hpp"

using namespace voxreg;

namespace {
thread_local char g_err[512];
template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const FormatError& e) {
        std::snprintf(g_err, sizeof(g_err), "%s", e.what());
        return 4;
    } catch (const IoError& e) {
        std::snprintf(g_err, sizeof(g_err), "%s", e.what());
        return 5;
    } catch (const std::invalid_argument& e) {
        std::snprintf(g_err, sizeof(g_err), "%s", e.what());
        return 1;
    } catch (const std::exception& e) {
        std::snprintf(g_err, sizeof(g_err), "%s", e.what());
        return 2;
    }
}
Dims3 D(const int64_t* d) { return Dims3{d[0], d[1], d[2]}; }
}  // namespace

extern "C" {
const char* refio_last_error() { return g_err; }

// write_nifti (nifti.hpp:230-239) of a T = float (f64 = 0) or T = double volume.
int refio_write_nifti(const double* v, const int64_t* dims, const double* spacing, const double* origin, int f64,
                      const char* path) {
    return guarded([&] {
        const Dims3 d = D(dims);
        if (f64) {
            auto vol = Volume3<double>::zeros(d);
            for (std::size_t i = 0; i < vol.data.size(); ++i) vol.data[i] = v[i];
            for (int c = 0; c < 3; ++c) vol.spacing[c] = spacing[c], vol.origin[c] = origin[c];
            write_nifti(vol, path);
        } else {
            auto vol = Volume3<float>::zeros(d);
            for (std::size_t i = 0; i < vol.data.size(); ++i) vol.data[i] = static_cast<float>(v[i]);
            for (int c = 0; c < 3; ++c) vol.spacing[c] = spacing[c], vol.origin[c] = origin[c];
            write_nifti(vol, path);
        }
    });
}

// write_nifti of a LabelVolume (nifti.hpp:241-251).
int refio_write_labels(const uint16_t* v, const int64_t* dims, const double* spacing, const char* path) {
    return guarded([&] {
        auto lv = LabelVolume::zeros(D(dims));
        for (std::size_t i = 0; i < lv.data.size(); ++i) lv.data[i] = v[i];
        for (int c = 0; c < 3; ++c) lv.spacing[c] = spacing[c];
        write_nifti(lv, path);
    });
}

// read_nifti (nifti.hpp:99-186): dims first (out = NULL to query), then the values.
int refio_read_nifti(const char* path, int64_t* dims, double* spacing, double* origin, double* out) {
    return guarded([&] {
        const NiftiVolume nv = read_nifti(path);
        dims[0] = nv.volume.dims.nx, dims[1] = nv.volume.dims.ny, dims[2] = nv.volume.dims.nz;
        for (int c = 0; c < 3; ++c) spacing[c] = nv.volume.spacing[c], origin[c] = nv.volume.origin[c];
        if (out) std::memcpy(out, nv.volume.data.data(), nv.volume.data.size() * sizeof(double));
    });
}

// write_warp / read_warp (nifti.hpp:268-303).
int refio_write_warp(const double* w, const int64_t* dims, const double* spacing, const double* origin,
                     const char* prefix) {
    return guarded([&] {
        auto wf = WarpField<double>::zeros(D(dims));
        for (std::size_t i = 0; i < wf.data.size(); ++i) wf.data[i] = w[i];
        write_warp(wf, prefix, Vec3{spacing[0], spacing[1], spacing[2]}, Vec3{origin[0], origin[1], origin[2]});
    });
}

int refio_read_warp(const char* prefix, int64_t* dims, double* out) {
    return guarded([&] {
        const auto wf = read_warp(prefix);
        dims[0] = wf.dims.nx, dims[1] = wf.dims.ny, dims[2] = wf.dims.nz;
        if (out) std::memcpy(out, wf.data.data(), wf.data.size() * sizeof(double));
    });
}
}  // extern "C"
