// raster_io.cpp -- FBMP float32 container (semantics of proj/src/raster_io.cpp:41-122): bit-exact
// round trips of float32 data, little-endian header, strict length / magic / version / dtype checks.
#include "fbmp/raster_io.hpp"

#include <cstring>
#include <fstream>
#include <vector>

#include "fbmp/errors.hpp"

namespace fbmp {
namespace {

constexpr std::size_t kHeader = 18;  // 4 + 2 + 4 + 4 + 2 + 2

void le(unsigned char* p, std::uint32_t v, int bytes) {
    for (int i = 0; i < bytes; ++i) p[i] = static_cast<unsigned char>((v >> (8 * i)) & 0xffu);
}
std::uint32_t rd(const unsigned char* p, int bytes) {
    std::uint32_t v = 0;
    for (int i = 0; i < bytes; ++i) v |= static_cast<std::uint32_t>(p[i]) << (8 * i);
    return v;
}

}  // namespace

void save_raster(const MultiBandImage& img, const std::string& path) {
    std::ofstream os(path, std::ios::binary);
    if (!os) throw IoError("cannot open for writing: " + path);
    unsigned char h[kHeader];
    std::memcpy(h, RasterHeader::kMagic, 4);
    le(h + 4, RasterHeader::kVersion, 2);
    le(h + 6, static_cast<std::uint32_t>(img.height()), 4);
    le(h + 10, static_cast<std::uint32_t>(img.width()), 4);
    le(h + 14, static_cast<std::uint32_t>(img.band_count()), 2);
    le(h + 16, RasterHeader::kDtypeF32, 2);
    os.write(reinterpret_cast<const char*>(h), kHeader);
    std::vector<unsigned char> buf;
    for (const Plane& b : img.bands()) {
        buf.resize(b.size() * 4);
        for (std::size_t i = 0; i < b.size(); ++i) {
            const float f = static_cast<float>(b.data()[i]);
            std::uint32_t bits;
            std::memcpy(&bits, &f, 4);
            le(buf.data() + 4 * i, bits, 4);
        }
        os.write(reinterpret_cast<const char*>(buf.data()), static_cast<std::streamsize>(buf.size()));
    }
    if (!os) throw IoError("write failed: " + path);
}

MultiBandImage load_raster(const std::string& path) {
    std::ifstream is(path, std::ios::binary | std::ios::ate);
    if (!is) throw IoError("cannot open: " + path);
    const std::streamoff total = is.tellg();
    is.seekg(0);
    if (total < static_cast<std::streamoff>(kHeader)) throw FormatError("raster too short for header: " + path);
    unsigned char h[kHeader];
    is.read(reinterpret_cast<char*>(h), kHeader);
    if (std::memcmp(h, RasterHeader::kMagic, 4) != 0) throw FormatError("bad magic (expected FBMP): " + path);
    const std::uint32_t version = rd(h + 4, 2), height = rd(h + 6, 4), width = rd(h + 10, 4), bands = rd(h + 14, 2),
                        dtype = rd(h + 16, 2);
    if (version != RasterHeader::kVersion)
        throw FormatError("unsupported raster version " + std::to_string(version) + ": " + path);
    if (dtype != RasterHeader::kDtypeF32)
        throw FormatError("unsupported dtype code " + std::to_string(dtype) + ": " + path);
    if (height == 0 || width == 0 || bands == 0) throw FormatError("empty raster dimensions: " + path);
    const std::size_t plane = static_cast<std::size_t>(height) * width, payload = plane * bands * 4;
    if (static_cast<std::size_t>(total) != kHeader + payload)
        throw FormatError("payload length mismatch (expected " + std::to_string(payload) + " bytes): " + path);
    std::vector<Plane> out;
    out.reserve(bands);
    std::vector<unsigned char> buf(plane * 4);
    for (std::uint32_t b = 0; b < bands; ++b) {
        is.read(reinterpret_cast<char*>(buf.data()), static_cast<std::streamsize>(buf.size()));
        if (!is) throw FormatError("truncated payload: " + path);
        Plane p(static_cast<int>(height), static_cast<int>(width));
        for (std::size_t i = 0; i < plane; ++i) {
            const std::uint32_t bits = rd(buf.data() + 4 * i, 4);
            float f;
            std::memcpy(&f, &bits, 4);
            p.data()[i] = f;
        }
        out.push_back(std::move(p));
    }
    return MultiBandImage(std::move(out));
}

void save_kernel(const Kernel2D& k, const std::string& path) { save_raster(MultiBandImage({k.taps()}), path); }

Kernel2D load_kernel(const std::string& path) {
    const MultiBandImage img = load_raster(path);
    if (img.band_count() != 1 || img.height() != img.width() || img.height() % 2 == 0)
        throw FormatError("kernel raster must be one odd square band: " + path);
    Kernel2D k(img.height());
    for (std::size_t i = 0; i < img.band(0).size(); ++i) k.taps().data()[i] = img.band(0).data()[i];
    return k;
}

}  // namespace fbmp
