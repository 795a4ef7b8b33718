// mcg_checkpoint.h — the reference's checkpoint container, MCSCKPT1
// (engine.cpp:1036-1148): named f64 / u64 arrays in two std::maps, serialized
// in map (name) order, little-endian, magic + version + endianness probe.
// Host code; the engine fills and reads it from device state (mcg_engine.cu).
#pragma once
#include <cstdint>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "mcg_build.h"

namespace mcg {

struct Ckpt {
  std::map<std::string, std::vector<double>> f64;
  std::map<std::string, std::vector<uint64_t>> u64;
};

inline void ck_put_u32(std::vector<uint8_t>& b, uint32_t v) {
  for (int i = 0; i < 4; ++i) b.push_back((v >> (8 * i)) & 0xFF);
}
inline void ck_put_u64(std::vector<uint8_t>& b, uint64_t v) {
  for (int i = 0; i < 8; ++i) b.push_back((v >> (8 * i)) & 0xFF);
}

inline constexpr char kCkMagic[8] = {'M', 'C', 'S', 'C', 'K', 'P', 'T', '1'};

// Checkpoint::serialize (engine.cpp:1070-1093)
inline std::vector<uint8_t> ck_serialize(const Ckpt& c) {
  std::vector<uint8_t> b;
  b.insert(b.end(), kCkMagic, kCkMagic + 8);
  ck_put_u32(b, 1);
  ck_put_u32(b, 0x01020304);
  auto put_name = [&](const std::string& n) {
    ck_put_u32(b, static_cast<uint32_t>(n.size()));
    b.insert(b.end(), n.begin(), n.end());
  };
  for (const auto& [name, arr] : c.f64) {
    put_name(name);
    b.push_back(0);
    ck_put_u64(b, arr.size());
    for (double v : arr) {
      uint64_t u;
      std::memcpy(&u, &v, 8);
      ck_put_u64(b, u);
    }
  }
  for (const auto& [name, arr] : c.u64) {
    put_name(name);
    b.push_back(1);
    ck_put_u64(b, arr.size());
    for (uint64_t v : arr) ck_put_u64(b, v);
  }
  return b;
}

// Checkpoint::deserialize (engine.cpp:1095-1140), same validation and messages
inline Ckpt ck_deserialize(const uint8_t* d, size_t n) {
  auto fail = [](const char* m) { throw Error(MCG_ERR_ENGINE, m); };
  Ckpt c;
  if (n < 16 || std::memcmp(d, kCkMagic, 8) != 0) fail("checkpoint: bad magic");
  size_t pos = 8;
  auto u32 = [&]() {
    if (pos + 4 > n) fail("checkpoint: truncated");
    uint32_t v = 0;
    for (int i = 0; i < 4; ++i) v |= uint32_t(d[pos + i]) << (8 * i);
    pos += 4;
    return v;
  };
  auto u64 = [&]() {
    if (pos + 8 > n) fail("checkpoint: truncated");
    uint64_t v = 0;
    for (int i = 0; i < 8; ++i) v |= uint64_t(d[pos + i]) << (8 * i);
    pos += 8;
    return v;
  };
  if (u32() != 1) fail("checkpoint: version mismatch");
  if (u32() != 0x01020304) fail("checkpoint: endianness mismatch");
  while (pos < n) {
    const uint32_t nlen = u32();
    if (pos + nlen > n) fail("checkpoint: truncated");
    std::string name(reinterpret_cast<const char*>(d + pos), nlen);
    pos += nlen;
    if (pos >= n) fail("checkpoint: truncated");
    const uint8_t type = d[pos++];
    const uint64_t count = u64();
    if (count > (n - pos) / 8) fail("checkpoint: corrupted length header");
    if (type == 0) {
      std::vector<double> arr(count);
      for (auto& v : arr) {
        const uint64_t u = u64();
        std::memcpy(&v, &u, 8);
      }
      c.f64.emplace(std::move(name), std::move(arr));
    } else if (type == 1) {
      std::vector<uint64_t> arr(count);
      for (auto& v : arr) v = u64();
      c.u64.emplace(std::move(name), std::move(arr));
    } else {
      fail("checkpoint: unknown record type");
    }
  }
  return c;
}

// EventRec (engine.hpp:55-63) as make_checkpoint packs it (engine.cpp:1211-1225)
struct CkEvent {
  int64_t step;
  uint32_t src, seq;
  uint16_t group;
  uint8_t etype;
  uint32_t instance;
  double weight;
};

inline void ck_pack(Ckpt& c, const std::string& name, const std::vector<CkEvent>& evs) {
  std::vector<uint64_t> meta;
  std::vector<double> w;
  meta.reserve(4 * evs.size());
  w.reserve(evs.size());
  for (const auto& e : evs) {
    meta.push_back(static_cast<uint64_t>(e.step));
    meta.push_back(e.src);
    meta.push_back((uint64_t(e.group) << 48) | (uint64_t(e.etype) << 40) | e.instance);
    meta.push_back(e.seq);
    w.push_back(e.weight);
  }
  c.u64[name + "_meta"] = meta;
  c.f64[name + "_w"] = w;
}

inline std::vector<CkEvent> ck_unpack(const std::vector<uint64_t>& meta, const std::vector<double>& w) {
  if (meta.size() != w.size() * 4) throw Error(MCG_ERR_ENGINE, "checkpoint: corrupted event block");
  std::vector<CkEvent> out(w.size());
  for (size_t i = 0; i < w.size(); ++i) {
    CkEvent& e = out[i];
    e.step = static_cast<int64_t>(meta[4 * i]);
    e.src = static_cast<uint32_t>(meta[4 * i + 1]);
    const uint64_t packed = meta[4 * i + 2];
    e.group = static_cast<uint16_t>(packed >> 48);
    e.etype = static_cast<uint8_t>((packed >> 40) & 0xFF);
    e.instance = static_cast<uint32_t>(packed & 0xFFFFFFFFull);
    e.seq = static_cast<uint32_t>(meta[4 * i + 3]);
    e.weight = w[i];
  }
  return out;
}

}  // namespace mcg
