// On-disk formats next to the path, host side of the C-ABI:
//  * .stnt raw tensors (video_io.cpp:52-117): "STNT", u32 t, h, w, f (little endian), one
//    width byte (4 = f32, 8 = f64), then t*h*w*f little-endian elements, F fastest.
//  * Middlebury .flo (flow.cpp:53-112): f32 magic 202021.25, i32 width, i32 height, then
//    (u, v) = (dx, dy) f32 pairs row-major; fields here are (dy, dx) like FlowField.
// Errors carry the reference's IoError / DomainError messages (status SNLS_EIO / EDOMAIN).
#include <cmath>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <iterator>
#include <string>
#include <vector>

#include "snls_cuda.h"

namespace snls_capi {
int fail(int code, const std::string& msg);
}

namespace {

using snls_capi::fail;

bool read_all(const char* path, std::vector<unsigned char>& buf) {
    std::ifstream in(path, std::ios::binary);
    if (!in) return false;
    buf.assign(std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>());
    return true;
}

uint32_t u32le(const unsigned char* p) {
    return uint32_t(p[0]) | (uint32_t(p[1]) << 8) | (uint32_t(p[2]) << 16) | (uint32_t(p[3]) << 24);
}

void put_u32le(std::string& o, uint32_t v) {
    for (int i = 0; i < 4; ++i) o.push_back(char((v >> (8 * i)) & 0xff));
}

float f32le(const unsigned char* p) {
    const uint32_t b = u32le(p);
    float x;
    std::memcpy(&x, &b, 4);
    return x;
}

void put_f32le(std::string& o, float x) {
    uint32_t b;
    std::memcpy(&b, &x, 4);
    put_u32le(o, b);
}

int write_all(const char* path, const std::string& bytes) {
    std::ofstream out(path, std::ios::binary | std::ios::trunc);
    if (!out) return fail(SNLS_EIO, std::string("cannot open ") + path + " for writing");
    out.write(bytes.data(), std::streamoff(bytes.size()));
    if (!out) return fail(SNLS_EIO, std::string("short write on ") + path);
    return SNLS_OK;
}

constexpr float kFloMagic = 202021.25f;

// load_raw's header checks (video_io.cpp:52-69)
int raw_header(const char* path, const std::vector<unsigned char>& buf, snls_dims* d, int* width) {
    const std::string p(path);
    if (buf.size() < 21) return fail(SNLS_EIO, p + ": truncated header");
    if (std::memcmp(buf.data(), "STNT", 4) != 0) return fail(SNLS_EIO, p + ": bad magic");
    const uint32_t t = u32le(&buf[4]), h = u32le(&buf[8]), w = u32le(&buf[12]), f = u32le(&buf[16]);
    const int wd = buf[20];
    if (t == 0 || h == 0 || w == 0 || f == 0) return fail(SNLS_EIO, p + ": zero extent in header");
    if (wd != 4 && wd != 8) return fail(SNLS_EIO, p + ": element width must be 4 or 8");
    const size_t count = size_t(t) * h * w * f;
    if (buf.size() != 21 + count * size_t(wd)) return fail(SNLS_EIO, p + ": payload size does not match header");
    *d = snls_dims{int(t), int(h), int(w), int(f)};
    *width = wd;
    return SNLS_OK;
}

}  // namespace

extern "C" {

int snls_raw_info(const char* path, snls_dims* dims, int* width) {
    if (!path || !dims || !width) return fail(SNLS_EARG, "snls_raw_info: null argument");
    std::vector<unsigned char> buf;
    if (!read_all(path, buf)) return fail(SNLS_EIO, std::string("cannot open ") + path);
    return raw_header(path, buf, dims, width);
}

int snls_raw_read(const char* path, float* out, int64_t capacity) {
    if (!path || !out) return fail(SNLS_EARG, "snls_raw_read: null argument");
    std::vector<unsigned char> buf;
    if (!read_all(path, buf)) return fail(SNLS_EIO, std::string("cannot open ") + path);
    snls_dims d;
    int wd = 0;
    if (int rc = raw_header(path, buf, &d, &wd)) return rc;
    const int64_t count = int64_t(d.t) * d.h * d.w * d.f;
    if (capacity < count) return fail(SNLS_EARG, "snls_raw_read: output too small");
    const unsigned char* p = buf.data() + 21;
    for (int64_t i = 0; i < count; ++i) {
        double x;
        if (wd == 4) {
            x = double(f32le(p));
            p += 4;
        } else {
            const uint64_t b = uint64_t(u32le(p)) | (uint64_t(u32le(p + 4)) << 32);
            std::memcpy(&x, &b, 8);
            p += 8;
        }
        if (!std::isfinite(x))  // VideoTensor::require_finite (tensor.cpp:18-21)
            return fail(SNLS_EDOMAIN, std::string(path) + ": tensor holds a non-finite value");
        out[i] = float(x);
    }
    return SNLS_OK;
}

int snls_raw_write(const char* path, snls_dims d, const float* data, int width) {
    if (!path || !data) return fail(SNLS_EARG, "snls_raw_write: null argument");
    if (width != 4 && width != 8) return fail(SNLS_EARG, "snls_raw_write: element width must be 4 or 8");
    const int64_t count = int64_t(d.t) * d.h * d.w * d.f;
    std::string out;
    out.reserve(size_t(21 + count * width));
    out.append("STNT", 4);
    put_u32le(out, uint32_t(d.t));
    put_u32le(out, uint32_t(d.h));
    put_u32le(out, uint32_t(d.w));
    put_u32le(out, uint32_t(d.f));
    out.push_back(char(width));
    for (int64_t i = 0; i < count; ++i) {
        if (width == 4) {
            put_f32le(out, data[i]);
        } else {
            const double x = double(data[i]);
            uint64_t b;
            std::memcpy(&b, &x, 8);
            put_u32le(out, uint32_t(b & 0xffffffffu));
            put_u32le(out, uint32_t(b >> 32));
        }
    }
    return write_all(path, out);
}

// read_flo (flow.cpp:53-80): out (may be NULL to query the size) h x w x 2 as (dy, dx).
int snls_flo_read(const char* path, int* h, int* w, float* out) {
    if (!path || !h || !w) return fail(SNLS_EARG, "snls_flo_read: null argument");
    std::vector<unsigned char> buf;
    if (!read_all(path, buf)) return fail(SNLS_EIO, std::string("cannot open ") + path);
    const std::string p(path);
    if (buf.size() < 12) return fail(SNLS_EIO, p + ": truncated header");
    if (f32le(buf.data()) != kFloMagic) return fail(SNLS_EIO, p + ": bad magic");
    const int32_t ww = int32_t(u32le(&buf[4])), hh = int32_t(u32le(&buf[8]));
    if (ww < 1 || hh < 1 || ww > 99999 || hh > 99999)
        return fail(SNLS_EIO, p + ": nonsensical dimensions " + std::to_string(ww) + "x" + std::to_string(hh));
    const size_t count = size_t(ww) * hh * 2;
    if (buf.size() != 12 + count * 4) return fail(SNLS_EIO, p + ": truncated payload");
    *h = hh;
    *w = ww;
    if (!out) return SNLS_OK;
    const unsigned char* q = buf.data() + 12;
    for (size_t i = 0; i < size_t(ww) * hh; ++i, q += 8) {
        const float u = f32le(q), v = f32le(q + 4);  // file stores (u, v) = (dx, dy)
        if (!std::isfinite(u) || !std::isfinite(v))
            return fail(SNLS_EDOMAIN, p + ": flow holds a non-finite value");
        out[2 * i] = v;
        out[2 * i + 1] = u;
    }
    return SNLS_OK;
}

// write_flo (flow.cpp:82-112): one frame h x w x 2 (dy, dx).
int snls_flo_write(const char* path, int h, int w, const float* flow) {
    if (!path || !flow) return fail(SNLS_EARG, "snls_flo_write: null argument");
    std::string out;
    out.reserve(12 + size_t(h) * w * 8);
    put_f32le(out, kFloMagic);
    put_u32le(out, uint32_t(w));
    put_u32le(out, uint32_t(h));
    for (size_t i = 0; i < size_t(h) * w; ++i) {
        put_f32le(out, flow[2 * i + 1]);  // u = dx first
        put_f32le(out, flow[2 * i]);      // v = dy second
    }
    return write_all(path, out);
}

}  // extern "C"
