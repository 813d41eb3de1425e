// DPLN checkpoints (dp/checkpoint.hpp:121-198): the
// reference's on-disk format.  "DPLN", version u32 (1), element size u32,
// epoch u32, entry count u32; per entry a u32-length-prefixed name, four i64
// dims and the raw little-endian elements; a trailing CRC-32 (IEEE, reflected)
// of every preceding byte.  Host code: parameters move between the GPU and
// the file through host buffers.
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "dpb_internal.h"

namespace {

uint32_t crc32(const unsigned char* p, size_t n) {
  static uint32_t table[256];
  static bool init = false;
  if (!init) {
    for (uint32_t i = 0; i < 256; ++i) {
      uint32_t c = i;
      for (int k = 0; k < 8; ++k) c = (c & 1) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
      table[i] = c;
    }
    init = true;
  }
  uint32_t crc = 0xFFFFFFFFu;
  for (size_t i = 0; i < n; ++i) crc = table[(crc ^ p[i]) & 0xFFu] ^ (crc >> 8);
  return crc ^ 0xFFFFFFFFu;
}

constexpr uint32_t kVersion = 1;

template <typename V>
void put(std::vector<unsigned char>& b, V v) {
  const auto* p = reinterpret_cast<const unsigned char*>(&v);
  b.insert(b.end(), p, p + sizeof(V));
}

struct Reader {
  const std::vector<unsigned char>& b;
  size_t pos, end;
  bool get(void* dst, size_t n) {
    if (pos + n > end) return false;
    std::memcpy(dst, b.data() + pos, n);
    pos += n;
    return true;
  }
};

}  // namespace

using dpb::fail;

extern "C" {

DPB_API int dpb_checkpoint_save(const char* path, int count, const char* const* names, const int64_t* dims,
                                const float* data, int epoch) {
  if (!path || count < 0 || (count > 0 && (!names || !dims || !data)))
    return fail(DPB_CONFIG_ERROR, "invalid checkpoint arguments");
  std::vector<unsigned char> b;
  b.insert(b.end(), {'D', 'P', 'L', 'N'});
  put<uint32_t>(b, kVersion);
  put<uint32_t>(b, sizeof(float));
  put<uint32_t>(b, static_cast<uint32_t>(epoch));
  put<uint32_t>(b, static_cast<uint32_t>(count));
  const float* src = data;
  for (int i = 0; i < count; ++i) {
    const size_t len = std::strlen(names[i]);
    put<uint32_t>(b, static_cast<uint32_t>(len));
    b.insert(b.end(), names[i], names[i] + len);
    int64_t elems = 1;
    for (int d = 0; d < 4; ++d) {
      put<int64_t>(b, dims[4 * i + d]);
      elems *= dims[4 * i + d];
    }
    const auto* p = reinterpret_cast<const unsigned char*>(src);
    b.insert(b.end(), p, p + elems * sizeof(float));
    src += elems;
  }
  put<uint32_t>(b, crc32(b.data(), b.size()));
  FILE* f = std::fopen(path, "wb");
  if (!f) return fail(DPB_FORMAT_ERROR, std::string("cannot open ") + path + " for writing");
  const bool ok = std::fwrite(b.data(), 1, b.size(), f) == b.size();
  if (std::fclose(f) != 0 || !ok) return fail(DPB_FORMAT_ERROR, "checkpoint write failed");
  return DPB_OK;
}

DPB_API int dpb_checkpoint_load(const char* path, int count, const char* const* names, const int64_t* dims,
                                float* data, int* epoch) {
  if (!path || count < 0 || (count > 0 && (!names || !dims || !data)))
    return fail(DPB_CONFIG_ERROR, "invalid checkpoint arguments");
  FILE* f = std::fopen(path, "rb");
  if (!f) return fail(DPB_FORMAT_ERROR, std::string("cannot open ") + path);
  std::vector<unsigned char> b;
  unsigned char buf[1 << 16];
  size_t n;
  while ((n = std::fread(buf, 1, sizeof(buf), f)) > 0) b.insert(b.end(), buf, buf + n);
  std::fclose(f);
  if (b.size() < sizeof(uint32_t)) return fail(DPB_FORMAT_ERROR, std::string("checkpoint too short: ") + path);
  const size_t payload = b.size() - sizeof(uint32_t);
  uint32_t stored;
  std::memcpy(&stored, b.data() + payload, sizeof(stored));
  if (stored != crc32(b.data(), payload))
    return fail(DPB_FORMAT_ERROR, std::string("checkpoint checksum mismatch in ") + path);
  Reader r{b, 0, payload};
  char magic[4];
  uint32_t version, esize, ep, cnt;
  if (!r.get(magic, 4) || std::memcmp(magic, "DPLN", 4) != 0)
    return fail(DPB_FORMAT_ERROR, std::string("bad checkpoint magic in ") + path);
  if (!r.get(&version, 4) || version != kVersion)
    return fail(DPB_FORMAT_ERROR, "unsupported checkpoint version " + std::to_string(version));
  if (!r.get(&esize, 4) || esize != sizeof(float))
    return fail(DPB_FORMAT_ERROR, "checkpoint element size " + std::to_string(esize) +
                                      " does not match requested element type");
  if (!r.get(&ep, 4) || !r.get(&cnt, 4)) return fail(DPB_FORMAT_ERROR, "checkpoint truncated");
  if (cnt != static_cast<uint32_t>(count))
    return fail(DPB_FORMAT_ERROR, "checkpoint holds " + std::to_string(cnt) + " tensors, expected " +
                                      std::to_string(count));
  float* dst = data;
  for (int i = 0; i < count; ++i) {
    uint32_t len;
    if (!r.get(&len, 4) || r.pos + len > r.end) return fail(DPB_FORMAT_ERROR, "checkpoint truncated");
    const std::string name(reinterpret_cast<const char*>(b.data() + r.pos), len);
    r.pos += len;
    if (name != names[i])
      return fail(DPB_FORMAT_ERROR,
                  "checkpoint tensor '" + name + "' where '" + names[i] + "' was expected");
    int64_t s[4], elems = 1;
    if (!r.get(s, sizeof(s))) return fail(DPB_FORMAT_ERROR, "checkpoint truncated");
    for (int d = 0; d < 4; ++d) {
      if (s[d] != dims[4 * i + d])
        return fail(DPB_FORMAT_ERROR, "checkpoint tensor '" + name + "' has a different shape");
      elems *= s[d];
    }
    if (!r.get(dst, static_cast<size_t>(elems) * sizeof(float)))
      return fail(DPB_FORMAT_ERROR, "checkpoint truncated");
    dst += elems;
  }
  if (epoch) *epoch = static_cast<int>(ep);
  return DPB_OK;
}

}  // extern "C"
