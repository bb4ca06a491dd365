// Stiffness containers: the hand-off of integrated
// element matrices to a consumer.
//
//  * PRISTIF1 -- the reference's single-element container (io.cpp:112-168):
//    8-byte magic "PRISTIF1", u32 LE JSON header length, the JSON header
//    {"dim","element_id","n_eq","n_shape","p"} (nlohmann's sorted compact
//    dump), then the canonical payload as LE float32.  Written byte-for-byte
//    like save_stiffness and read like load_stiffness.  float32 only, so it
//    cannot carry the 1e-12 FP64 results.
//  * PRISTIF2 -- the FP64 batch container of this library: magic
//    "PRISTIF2", u32 LE header length, JSON header {"count","dim",
//    "dtype":"f64","element_id_base","layout":"canonical","n_eq","n_shape",
//    "p"}, then count x dim x dim LE float64 in mesh order.
// Host code only (the matrices come back from pi_integrate_host / a D2H
// copy); no JSON library: the headers are fixed-schema and parsed by key.
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "pi_internal.hpp"

namespace pib {
namespace {

constexpr char kMagic1[8] = {'P', 'R', 'I', 'S', 'T', 'I', 'F', '1'};
constexpr char kMagic2[8] = {'P', 'R', 'I', 'S', 'T', 'I', 'F', '2'};

void put_u32(std::string& s, uint32_t v) {
  for (int i = 0; i < 4; ++i) s.push_back(static_cast<char>((v >> (8 * i)) & 0xff));
}
uint32_t get_u32(const unsigned char* p) {
  return uint32_t(p[0]) | (uint32_t(p[1]) << 8) | (uint32_t(p[2]) << 16) | (uint32_t(p[3]) << 24);
}
bool little_endian() {
  const uint16_t x = 1;
  return *reinterpret_cast<const unsigned char*>(&x) == 1;
}

// Integer value of "key" in a flat JSON object; false if absent.
bool json_int(const std::string& h, const char* key, int64_t& out) {
  const std::string k = std::string("\"") + key + "\"";
  size_t pos = h.find(k);
  if (pos == std::string::npos) return false;
  pos = h.find(':', pos + k.size());
  if (pos == std::string::npos) return false;
  ++pos;
  while (pos < h.size() && (h[pos] == ' ' || h[pos] == '\t' || h[pos] == '\n' || h[pos] == '\r')) ++pos;
  char* end = nullptr;
  const long long v = std::strtoll(h.c_str() + pos, &end, 10);
  if (end == h.c_str() + pos) return false;
  out = v;
  return true;
}
bool json_str(const std::string& h, const char* key, std::string& out) {
  const std::string k = std::string("\"") + key + "\"";
  size_t pos = h.find(k);
  if (pos == std::string::npos) return false;
  pos = h.find(':', pos + k.size());
  if (pos == std::string::npos) return false;
  const size_t q0 = h.find('"', pos + 1);
  if (q0 == std::string::npos) return false;
  const size_t q1 = h.find('"', q0 + 1);
  if (q1 == std::string::npos) return false;
  out = h.substr(q0 + 1, q1 - q0 - 1);
  return true;
}

bool read_all(const char* path, std::string& blob) {
  FILE* f = std::fopen(path, "rb");
  if (!f) return false;
  std::fseek(f, 0, SEEK_END);
  const long n = std::ftell(f);
  std::fseek(f, 0, SEEK_SET);
  blob.resize(n > 0 ? static_cast<size_t>(n) : 0);
  const size_t got = n > 0 ? std::fread(&blob[0], 1, blob.size(), f) : 0;
  std::fclose(f);
  return got == blob.size();
}

struct Header {
  int version = 0;  // 1 = PRISTIF1, 2 = PRISTIF2
  int64_t p = 0, n_eq = 0, n_shape = 0, dim = 0, count = 1, base = -1;
  size_t payload_off = 0;
};

pi_status parse(const std::string& blob, const char* path, Header& h, pi_error_info* err) {
  if (blob.size() < 12) return set_error(err, PI_E_IO, "'%s' is not a stiffness container", path);
  if (std::memcmp(blob.data(), kMagic1, 8) == 0)
    h.version = 1;
  else if (std::memcmp(blob.data(), kMagic2, 8) == 0)
    h.version = 2;
  else
    return set_error(err, PI_E_IO, "'%s' is not a stiffness container", path);
  const auto* u = reinterpret_cast<const unsigned char*>(blob.data());
  const uint32_t hl = get_u32(u + 8);
  if (blob.size() < 12 + static_cast<size_t>(hl)) return set_error(err, PI_E_IO, "'%s': truncated header", path);
  const std::string js = blob.substr(12, hl);
  if (!json_int(js, "p", h.p) || !json_int(js, "n_eq", h.n_eq) || !json_int(js, "n_shape", h.n_shape))
    return set_error(err, PI_E_IO, "'%s': bad header", path);
  h.dim = h.n_eq * h.n_shape;
  if (h.version == 1) {
    if (!json_int(js, "element_id", h.base)) h.base = -1;
    h.count = 1;
  } else {
    std::string dtype, layout;
    if (!json_int(js, "count", h.count) || !json_int(js, "element_id_base", h.base) || !json_str(js, "dtype", dtype) ||
        !json_str(js, "layout", layout) || dtype != "f64" || layout != "canonical" || h.count < 0)
      return set_error(err, PI_E_IO, "'%s': bad header", path);
  }
  h.payload_off = 12 + hl;
  const size_t esz = h.version == 1 ? 4 : 8;
  const size_t need = h.payload_off + static_cast<size_t>(h.count) * h.dim * h.dim * esz;
  if (blob.size() != need) return set_error(err, PI_E_IO, "'%s': payload size mismatch", path);
  return PI_OK;
}

}  // namespace
}  // namespace pib

using namespace pib;

extern "C" {

pi_status pi_save_stiffness(const char* path, int format, int p, int n_eq, int64_t count, int64_t element_id_base,
                            const double* k, pi_error_info* err) {
  if (err) std::memset(err, 0, sizeof(*err)), err->element = -1;
  if (!path || !k || count < 0) return set_error(err, PI_E_CONTRACT, "pi_save_stiffness: bad arguments");
  const int nsh = shape_count(p);
  if (nsh < 0) return set_error(err, PI_E_DOMAIN, "approximation order p=%d outside supported range [1, 7]", p);
  if (n_eq < 1) return set_error(err, PI_E_CONFIG, "n_eq=%d", n_eq);
  if (!little_endian()) return set_error(err, PI_E_IO, "big-endian host");
  const int64_t dim = static_cast<int64_t>(n_eq) * nsh, kk = dim * dim;
  std::string blob;
  char hdr[512];
  if (format == PI_STIFFNESS_PRISTIF1) {
    if (count != 1) return set_error(err, PI_E_CONFIG, "PRISTIF1 holds one element matrix (count=%lld)", (long long)count);
    std::snprintf(hdr, sizeof hdr, "{\"dim\":%lld,\"element_id\":%lld,\"n_eq\":%d,\"n_shape\":%d,\"p\":%d}",
                  (long long)dim, (long long)element_id_base, n_eq, nsh, p);
    blob.assign(kMagic1, 8);
  } else if (format == PI_STIFFNESS_PRISTIF2) {
    std::snprintf(hdr, sizeof hdr,
                  "{\"count\":%lld,\"dim\":%lld,\"dtype\":\"f64\",\"element_id_base\":%lld,\"layout\":\"canonical\","
                  "\"n_eq\":%d,\"n_shape\":%d,\"p\":%d}",
                  (long long)count, (long long)dim, (long long)element_id_base, n_eq, nsh, p);
    blob.assign(kMagic2, 8);
  } else {
    return set_error(err, PI_E_CONFIG, "unknown stiffness format %d", format);
  }
  const std::string h(hdr);
  put_u32(blob, static_cast<uint32_t>(h.size()));
  blob += h;
  FILE* f = std::fopen(path, "wb");
  if (!f) return set_error(err, PI_E_IO, "cannot open '%s' for writing", path);
  bool ok = std::fwrite(blob.data(), 1, blob.size(), f) == blob.size();
  if (format == PI_STIFFNESS_PRISTIF1) {
    std::vector<float> v(k, k + kk);  // the reference's payload (io.cpp:124-125)
    ok = ok && std::fwrite(v.data(), 4, v.size(), f) == v.size();
  } else {
    ok = ok && std::fwrite(k, 8, static_cast<size_t>(count * kk), f) == static_cast<size_t>(count * kk);
  }
  ok = (std::fclose(f) == 0) && ok;
  return ok ? PI_OK : set_error(err, PI_E_IO, "write to '%s' failed", path);
}

pi_status pi_stiffness_info(const char* path, int* format, int* p, int* n_eq, int64_t* count,
                            int64_t* element_id_base, pi_error_info* err) {
  if (err) std::memset(err, 0, sizeof(*err)), err->element = -1;
  std::string blob;
  if (!path || !read_all(path, blob)) return set_error(err, PI_E_IO, "cannot read '%s'", path ? path : "(null)");
  Header h;
  const pi_status st = parse(blob, path, h, err);
  if (st != PI_OK) return st;
  if (format) *format = h.version == 1 ? PI_STIFFNESS_PRISTIF1 : PI_STIFFNESS_PRISTIF2;
  if (p) *p = static_cast<int>(h.p);
  if (n_eq) *n_eq = static_cast<int>(h.n_eq);
  if (count) *count = h.count;
  if (element_id_base) *element_id_base = h.base;
  return PI_OK;
}

pi_status pi_load_stiffness(const char* path, double* out, int64_t capacity, pi_error_info* err) {
  if (err) std::memset(err, 0, sizeof(*err)), err->element = -1;
  std::string blob;
  if (!path || !read_all(path, blob)) return set_error(err, PI_E_IO, "cannot read '%s'", path ? path : "(null)");
  Header h;
  const pi_status st = parse(blob, path, h, err);
  if (st != PI_OK) return st;
  const int64_t n = h.count * h.dim * h.dim;
  if (!out || capacity < n)
    return set_error(err, PI_E_CONTRACT, "output holds %lld doubles, the container %lld", (long long)capacity,
                     (long long)n);
  const char* src = blob.data() + h.payload_off;
  if (h.version == 1) {
    for (int64_t i = 0; i < n; ++i) {
      float f;
      std::memcpy(&f, src + 4 * i, 4);
      out[i] = static_cast<double>(f);
    }
  } else {
    std::memcpy(out, src, sizeof(double) * n);
  }
  return PI_OK;
}

}  // extern "C"
