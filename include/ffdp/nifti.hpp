// ffdp/nifti.hpp -- NIfTI-1 single-file volumes and raw + JSON warp fields for the C++
// mirror (the reference's nifti.hpp:24-303), byte-compatible with the reference: files it
// writes are read here value for value, and volumes written here are byte-identical to its
// write_nifti. Host-side IO; the device containers of ffdp/voxreg.hpp are read back /
// uploaded around it. No JSON library: the warp sidecar has a fixed schema.
#pragma once

#include <array>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <iterator>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "ffdp/voxreg.hpp"

namespace ffdp {
namespace voxreg {

struct FormatError : std::runtime_error {
    std::size_t offset;
    FormatError(const std::string& what, std::size_t off)
        : std::runtime_error(what + " (at byte " + std::to_string(off) + ")"), offset(off) {}
};

struct IoError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

struct NiftiHeader {
    std::array<std::int16_t, 8> dim{};
    std::int16_t datatype = 0, bitpix = 0;
    std::array<float, 8> pixdim{};
    float vox_offset = 352, scl_slope = 0, scl_inter = 0;
    std::array<float, 3> qoffset{};
    std::array<char, 4> magic{};
    bool big_endian = false;
};

// The reference's NiftiVolume (Volume3<double> on the host).
struct NiftiVolume {
    NiftiHeader header;
    Dims3 dims;
    Vec3 spacing{{1, 1, 1}}, origin{{0, 0, 0}};
    std::vector<double> data;  // x fastest

    Volume3 to_device(cudaStream_t s = nullptr) const {
        std::vector<float> f(data.begin(), data.end());
        Volume3 v = Volume3::from_host(dims, f.data(), s);
        v.spacing = spacing;
        v.origin = origin;
        return v;
    }
};

namespace nifti_detail {
constexpr std::size_t kHeaderBytes = 348, kVoxOffset = 352;

template <typename T>
T rd(const std::vector<unsigned char>& b, std::size_t off, bool swap) {
    if (off + sizeof(T) > b.size()) throw FormatError("truncated header", off);
    unsigned char tmp[sizeof(T)];
    std::memcpy(tmp, b.data() + off, sizeof(T));
    if (swap)
        for (std::size_t i = 0; i < sizeof(T) / 2; ++i) std::swap(tmp[i], tmp[sizeof(T) - 1 - i]);
    T v;
    std::memcpy(&v, tmp, sizeof(T));
    return v;
}

template <typename T>
void wr(std::vector<unsigned char>& b, std::size_t off, T v) {
    std::memcpy(b.data() + off, &v, sizeof(T));
}

inline std::vector<unsigned char> header(Dims3 d, const Vec3& spacing, const Vec3& origin, std::int16_t datatype,
                                         std::int16_t bitpix) {
    if (d.nx > 32767 || d.ny > 32767 || d.nz > 32767)
        throw std::invalid_argument("write_nifti: dims exceed int16 header fields");
    std::vector<unsigned char> b(kVoxOffset, 0);
    wr<std::int32_t>(b, 0, 348);
    const std::int16_t dim[8] = {3, (std::int16_t)d.nx, (std::int16_t)d.ny, (std::int16_t)d.nz, 1, 1, 1, 1};
    for (int i = 0; i < 8; ++i) wr<std::int16_t>(b, 40 + 2 * i, dim[i]);
    wr<std::int16_t>(b, 70, datatype);
    wr<std::int16_t>(b, 72, bitpix);
    wr<float>(b, 76, 1.0f);
    for (int c = 0; c < 3; ++c) wr<float>(b, 80 + 4 * c, static_cast<float>(spacing[c]));
    wr<float>(b, 108, static_cast<float>(kVoxOffset));
    for (int c = 0; c < 3; ++c) wr<float>(b, 268 + 4 * c, static_cast<float>(origin[c]));
    b[344] = 'n', b[345] = '+', b[346] = '1', b[347] = 0;
    return b;
}

inline void dump(const std::string& path, const std::vector<unsigned char>& bytes) {
    if (path.empty()) throw IoError("empty output path");
    std::ofstream f(path, std::ios::binary);
    if (!f) throw IoError("cannot open " + path + " for writing");
    f.write(reinterpret_cast<const char*>(bytes.data()), static_cast<std::streamsize>(bytes.size()));
    if (!f) throw IoError("short write to " + path);
}

// the numbers of the JSON array stored under "key" (the sidecar's fixed schema)
inline std::vector<double> json_numbers(const std::string& text, const std::string& key, bool array) {
    const std::size_t k = text.find("\"" + key + "\"");
    if (k == std::string::npos) throw IoError("warp sidecar: missing " + key);
    std::size_t p = text.find(':', k);
    if (p == std::string::npos) throw IoError("warp sidecar: malformed " + key);
    ++p;
    std::size_t end = array ? text.find(']', p) : text.find_first_of(",}", p);
    std::string body = text.substr(p, end - p);
    for (char& ch : body)
        if (ch == '[' || ch == ',') ch = ' ';
    std::istringstream is(body);
    std::vector<double> out;
    double v;
    while (is >> v) out.push_back(v);
    return out;
}
}  // namespace nifti_detail

// read_nifti_bytes / read_nifti (nifti.hpp:99-186).
inline NiftiVolume read_nifti_bytes(const std::vector<unsigned char>& b) {
    using namespace nifti_detail;
    if (b.size() < kHeaderBytes) throw FormatError("file shorter than header", b.size());
    bool swap = false;
    if (rd<std::int32_t>(b, 0, false) != 348) {
        if (rd<std::int32_t>(b, 0, true) == 348)
            swap = true;
        else
            throw FormatError("sizeof_hdr is not 348 in either byte order", 0);
    }
    NiftiVolume out;
    NiftiHeader& h = out.header;
    h.big_endian = swap;
    for (int i = 0; i < 8; ++i) h.dim[i] = rd<std::int16_t>(b, 40 + 2 * i, swap);
    h.datatype = rd<std::int16_t>(b, 70, swap);
    h.bitpix = rd<std::int16_t>(b, 72, swap);
    for (int i = 0; i < 8; ++i) h.pixdim[i] = rd<float>(b, 76 + 4 * i, swap);
    h.vox_offset = rd<float>(b, 108, swap);
    h.scl_slope = rd<float>(b, 112, swap);
    h.scl_inter = rd<float>(b, 116, swap);
    for (int i = 0; i < 3; ++i) h.qoffset[i] = rd<float>(b, 268 + 4 * i, swap);
    std::memcpy(h.magic.data(), b.data() + 344, 4);
    if (std::memcmp(h.magic.data(), "ni1", 4) == 0) throw FormatError("two-file NIfTI (magic \"ni1\") is unsupported", 344);
    if (std::memcmp(h.magic.data(), "n+1", 4) != 0) throw FormatError("bad magic", 344);
    if (h.dim[0] < 1 || h.dim[0] > 3) throw FormatError("only 3-D volumes supported", 40);
    const Dims3 d{h.dim[1], h.dim[0] >= 2 ? h.dim[2] : 1, h.dim[0] >= 3 ? h.dim[3] : 1};
    if (!d.positive()) throw FormatError("non-positive dims", 40);
    int bpv = 0;
    switch (h.datatype) {
        case 2: bpv = 1; break;
        case 4: bpv = 2; break;
        case 16: bpv = 4; break;
        case 64: bpv = 8; break;
        default: throw FormatError("unsupported datatype " + std::to_string(h.datatype), 70);
    }
    const auto off = static_cast<std::size_t>(h.vox_offset);
    if (b.size() < off + static_cast<std::size_t>(d.voxels()) * bpv) throw FormatError("truncated payload", b.size());
    out.dims = d;
    for (int c = 0; c < 3; ++c) {
        const float s = h.pixdim[c + 1];
        out.spacing[c] = s > 0 ? s : 1.0;
        out.origin[c] = h.qoffset[c];
    }
    out.data.resize(static_cast<std::size_t>(d.voxels()));
    const bool scl = h.scl_slope != 0.0f;
    for (std::int64_t k = 0; k < d.voxels(); ++k) {
        const std::size_t p = off + static_cast<std::size_t>(k) * bpv;
        double v = 0;
        switch (h.datatype) {
            case 2: v = b[p]; break;
            case 4: v = rd<std::int16_t>(b, p, swap); break;
            case 16: v = rd<float>(b, p, swap); break;
            case 64: v = rd<double>(b, p, swap); break;
        }
        if (scl) v = static_cast<double>(h.scl_slope) * v + static_cast<double>(h.scl_inter);
        out.data[static_cast<std::size_t>(k)] = v;
    }
    return out;
}

inline NiftiVolume read_nifti(const std::string& path) {
    std::ifstream f(path, std::ios::binary);
    if (!f) throw IoError("cannot open " + path);
    std::vector<unsigned char> bytes((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
    return read_nifti_bytes(bytes);
}

// write_nifti (nifti.hpp:230-239) of a device volume (T = float: datatype 16).
inline void write_nifti(const Volume3& v, const std::string& path, cudaStream_t s = nullptr) {
    auto bytes = nifti_detail::header(v.dims, v.spacing, v.origin, 16, 32);
    const std::vector<float> h = v.to_host(s);
    const std::size_t payload = h.size() * sizeof(float);
    bytes.resize(nifti_detail::kVoxOffset + payload);
    std::memcpy(bytes.data() + nifti_detail::kVoxOffset, h.data(), payload);
    nifti_detail::dump(path, bytes);
}

// write_warp / read_warp (nifti.hpp:268-303): fp64 raw payload + JSON sidecar.
inline void write_warp(const WarpField& w, const std::string& prefix, const Vec3& spacing = Vec3{{1, 1, 1}},
                       const Vec3& origin = Vec3{{0, 0, 0}}, cudaStream_t s = nullptr) {
    const std::vector<float> h = w.to_host(s);
    std::vector<unsigned char> raw(h.size() * sizeof(double));
    for (std::size_t i = 0; i < h.size(); ++i) {
        const double v = h[i];
        std::memcpy(raw.data() + i * sizeof(double), &v, sizeof(double));
    }
    nifti_detail::dump(prefix + ".raw", raw);
    std::ostringstream js;
    js.precision(17);
    js << "{\n  \"dims\": [" << w.dims.nx << ", " << w.dims.ny << ", " << w.dims.nz << "],\n  \"spacing\": ["
       << spacing[0] << ", " << spacing[1] << ", " << spacing[2] << "],\n  \"origin\": [" << origin[0] << ", "
       << origin[1] << ", " << origin[2] << "],\n  \"channels\": 3\n}\n";
    const std::string t = js.str();
    nifti_detail::dump(prefix + ".json", std::vector<unsigned char>(t.begin(), t.end()));
}

inline WarpField read_warp(const std::string& prefix, cudaStream_t s = nullptr) {
    std::ifstream jf(prefix + ".json");
    if (!jf) throw IoError("cannot open " + prefix + ".json");
    const std::string text((std::istreambuf_iterator<char>(jf)), std::istreambuf_iterator<char>());
    const auto dims = nifti_detail::json_numbers(text, "dims", true);
    const auto ch = nifti_detail::json_numbers(text, "channels", false);
    if (dims.size() != 3 || ch.size() != 1) throw IoError("warp sidecar: malformed");
    if (ch[0] != 3) throw IoError("warp sidecar: channels must be 3");
    const Dims3 d{static_cast<std::int64_t>(dims[0]), static_cast<std::int64_t>(dims[1]),
                  static_cast<std::int64_t>(dims[2])};
    std::ifstream rf(prefix + ".raw", std::ios::binary);
    if (!rf) throw IoError("cannot open " + prefix + ".raw");
    std::vector<double> raw(static_cast<std::size_t>(3 * d.voxels()));
    rf.read(reinterpret_cast<char*>(raw.data()), static_cast<std::streamsize>(raw.size() * sizeof(double)));
    if (rf.gcount() != static_cast<std::streamsize>(raw.size() * sizeof(double)))
        throw IoError("warp raw payload truncated");
    std::vector<float> f(raw.begin(), raw.end());
    return WarpField::from_host(d, f.data(), s);
}

}  // namespace voxreg
}  // namespace ffdp
