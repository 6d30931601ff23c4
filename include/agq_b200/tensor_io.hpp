// Drop-in for agq/tensor_io.hpp: LSB-first code packing and the AGQT dump
// format (/root/reference/proj/include/agq/tensor_io.hpp:16-161). The packed
// bitstream is byte-for-byte the layout the GPU codec writes to HBM, so a
// device-resident tensor dumps with one D2H copy (see dump_packed()).
#pragma once

#include <cstdint>
#include <cstring>
#include <fstream>
#include <istream>
#include <ostream>
#include <stdexcept>
#include <string>
#include <vector>

#include "quantize.hpp"

namespace agq {

inline constexpr char kDumpMagic[4] = {'A', 'G', 'Q', 'T'};
inline constexpr std::uint16_t kDumpVersion = 1;

inline std::vector<std::uint8_t> pack_codes(const std::vector<std::uint8_t>& codes,
                                            int bit_width) {
  const std::uint32_t mask = (1u << bit_width) - 1u;
  std::vector<std::uint8_t> out((codes.size() * bit_width + 7) / 8, 0);
  std::size_t bit = 0;
  for (std::uint8_t c : codes) {
    const std::uint32_t v = (c & mask) << (bit & 7);  // spans at most 2 bytes
    out[bit >> 3] |= static_cast<std::uint8_t>(v);
    if ((bit & 7) + bit_width > 8) out[(bit >> 3) + 1] |= static_cast<std::uint8_t>(v >> 8);
    bit += bit_width;
  }
  return out;
}

inline std::vector<std::uint8_t> unpack_codes(const std::vector<std::uint8_t>& bytes,
                                              int bit_width, std::size_t count) {
  if (bytes.size() < (count * bit_width + 7) / 8)
    throw std::runtime_error("tensor dump: packed codes truncated");
  const std::uint32_t mask = (1u << bit_width) - 1u;
  std::vector<std::uint8_t> out(count);
  std::size_t bit = 0;
  for (std::size_t i = 0; i < count; ++i, bit += bit_width) {
    std::uint32_t v = bytes[bit >> 3];
    if ((bit & 7) + bit_width > 8) v |= static_cast<std::uint32_t>(bytes[(bit >> 3) + 1]) << 8;
    out[i] = static_cast<std::uint8_t>((v >> (bit & 7)) & mask);
  }
  return out;
}

namespace detail {
template <typename T>
void put_le(std::ostream& os, T v) {
  unsigned char b[sizeof(T)];
  std::uint64_t u = 0;
  std::memcpy(&u, &v, sizeof(T));
  for (std::size_t i = 0; i < sizeof(T); ++i) b[i] = static_cast<unsigned char>(u >> (8 * i));
  os.write(reinterpret_cast<const char*>(b), sizeof(T));
}
template <typename T>
T get_le(std::istream& is) {
  unsigned char b[sizeof(T)];
  is.read(reinterpret_cast<char*>(b), sizeof(T));
  if (!is) throw std::runtime_error("tensor dump: truncated input");
  std::uint64_t u = 0;
  for (std::size_t i = 0; i < sizeof(T); ++i) u |= static_cast<std::uint64_t>(b[i]) << (8 * i);
  T v;
  std::memcpy(&v, &u, sizeof(T));
  return v;
}
}  // namespace detail

// Header + scales + an already packed code stream (e.g. copied from HBM).
inline void dump_packed(const QuantizedTensor& meta_only, const float* scales,
                        std::size_t n_scales, const std::uint8_t* packed,
                        std::size_t packed_bytes, std::ostream& os) {
  os.write(kDumpMagic, 4);
  detail::put_le<std::uint16_t>(os, kDumpVersion);
  detail::put_le<std::uint8_t>(os, static_cast<std::uint8_t>(meta_only.codec_kind));
  detail::put_le<std::uint8_t>(os, static_cast<std::uint8_t>(meta_only.bit_width));
  detail::put_le<std::uint32_t>(os, meta_only.block_size);
  detail::put_le<std::uint8_t>(os, static_cast<std::uint8_t>(meta_only.shape.size()));
  for (auto d : meta_only.shape) detail::put_le<std::uint64_t>(os, d);
  for (std::size_t b = 0; b < n_scales; ++b) {
    std::uint32_t u;
    std::memcpy(&u, &scales[b], 4);
    detail::put_le<std::uint32_t>(os, u);
  }
  os.write(reinterpret_cast<const char*>(packed), static_cast<std::streamsize>(packed_bytes));
  if (!os) throw std::runtime_error("tensor dump: write failed");
}

inline void dump_tensor(const QuantizedTensor& q, std::ostream& os) {
  validate(q);
  const auto packed = pack_codes(q.codes, q.bit_width);
  dump_packed(q, q.scales.data(), q.scales.size(), packed.data(), packed.size(), os);
}

inline QuantizedTensor load_tensor(std::istream& is) {
  char magic[4];
  is.read(magic, 4);
  if (!is || std::memcmp(magic, kDumpMagic, 4) != 0)
    throw std::runtime_error("tensor dump: bad magic");
  const auto version = detail::get_le<std::uint16_t>(is);
  if (version != kDumpVersion)
    throw std::runtime_error("tensor dump: unsupported version " + std::to_string(version));
  QuantizedTensor q;
  const auto codec = detail::get_le<std::uint8_t>(is);
  if (codec > 2) throw std::runtime_error("tensor dump: unknown codec kind");
  q.codec_kind = static_cast<CodecKind>(codec);
  q.bit_width = detail::get_le<std::uint8_t>(is);
  q.block_size = detail::get_le<std::uint32_t>(is);
  q.shape.resize(detail::get_le<std::uint8_t>(is));
  for (auto& d : q.shape) d = detail::get_le<std::uint64_t>(is);
  detail::check_codec_args(q.bit_width, q.block_size, q.codec_kind);
  const std::size_t n = shape_elements(q.shape);
  q.scales.resize(agq_num_blocks(n, q.block_size));
  for (auto& s : q.scales) {
    const auto u = detail::get_le<std::uint32_t>(is);
    std::memcpy(&s, &u, 4);
  }
  std::vector<std::uint8_t> packed(agq_packed_bytes(n, q.bit_width));
  is.read(reinterpret_cast<char*>(packed.data()), static_cast<std::streamsize>(packed.size()));
  if (!is) throw std::runtime_error("tensor dump: truncated codes");
  q.codes = unpack_codes(packed, q.bit_width, n);
  validate(q);
  return q;
}

inline void dump_tensor_file(const QuantizedTensor& q, const std::string& path) {
  std::ofstream os(path, std::ios::binary);
  if (!os) throw std::runtime_error("cannot open for write: " + path);
  dump_tensor(q, os);
}

inline QuantizedTensor load_tensor_file(const std::string& path) {
  std::ifstream is(path, std::ios::binary);
  if (!is) throw std::runtime_error("cannot open for read: " + path);
  return load_tensor(is);
}

}  // namespace agq
