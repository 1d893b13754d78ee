// intergrams/common.hpp — drop-in for /root/reference/proj/include/intergrams/common.hpp
// (error classes common.hpp:12-22, hex codec common.cpp:16-42).  Header-only.
#pragma once

#include <stdexcept>
#include <string>
#include <string_view>

namespace intergrams {

// Unusable configuration or parameters (CLI exit code 2).
class ConfigError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

// Filesystem or read failure (CLI exit code 3).
class IoError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

// Device, collective or allocation failure inside the B200 library (exit 4).
class DeviceError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

inline std::string to_hex(std::string_view bytes) {
  static constexpr char kHex[] = "0123456789abcdef";
  std::string out;
  out.reserve(bytes.size() * 2);
  for (unsigned char c : bytes) {
    out.push_back(kHex[c >> 4]);
    out.push_back(kHex[c & 0x0f]);
  }
  return out;
}

inline std::string from_hex(std::string_view hex) {
  auto val = [](char c) -> int {
    if (c >= '0' && c <= '9') return c - '0';
    if (c >= 'a' && c <= 'f') return c - 'a' + 10;
    if (c >= 'A' && c <= 'F') return c - 'A' + 10;
    return -1;
  };
  if (hex.size() % 2 != 0) throw ConfigError("hex string has odd length: " + std::string(hex));
  std::string out;
  out.reserve(hex.size() / 2);
  for (size_t i = 0; i < hex.size(); i += 2) {
    const int hi = val(hex[i]), lo = val(hex[i + 1]);
    if (hi < 0 || lo < 0) throw ConfigError("invalid hex string: " + std::string(hex));
    out.push_back(static_cast<char>((hi << 4) | lo));
  }
  return out;
}

}  // namespace intergrams
