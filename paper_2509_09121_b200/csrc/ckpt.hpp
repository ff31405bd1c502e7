// Reader / writer of the reference checkpoint format (proj/include/compasslab/checkpoint.hpp:4-9):
//   bytes 0..7   magic "CLCKPT1\0"
//   bytes 8..15  little-endian u64, length of the JSON header
//   header       JSON {"tensors": {name: {"offset": N, "shape": [...]}}}
//   payload      raw little-endian float32 data, offsets relative to the payload
// The writer emits the header the way the reference's nlohmann::json dump does (compact, keys in
// sorted order, tensors in name order), so files round-trip byte-exactly through the reference
// loader/saver (checkpoint.cpp:20-72). The reader accepts any JSON formatting.
#pragma once
#include <cstdint>
#include <cstring>
#include <fstream>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

namespace cmoe {

struct CkptTensor {
  std::vector<int64_t> shape;
  uint64_t offset = 0;
};

class CkptError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

// Minimal JSON reader for the checkpoint header (objects, arrays, strings, integers).
class HeaderParser {
 public:
  explicit HeaderParser(const std::string& s) : s_(s) {}
  std::map<std::string, CkptTensor> parse() {
    std::map<std::string, CkptTensor> out;
    expect('{');
    bool found = false;
    if (!peek('}')) {
      do {
        const std::string key = str();
        expect(':');
        if (key == "tensors") {
          found = true;
          expect('{');
          if (!peek('}')) {
            do {
              const std::string name = str();
              expect(':');
              out[name] = entry();
            } while (take(','));
          }
          expect('}');
        } else {
          skip_value();
        }
      } while (take(','));
    }
    expect('}');
    if (!found) throw CkptError("checkpoint header has no \"tensors\" object");
    return out;
  }

 private:
  const std::string& s_;
  size_t p_ = 0;
  void ws() {
    while (p_ < s_.size() && (s_[p_] == ' ' || s_[p_] == '\n' || s_[p_] == '\t' || s_[p_] == '\r')) ++p_;
  }
  bool peek(char c) {
    ws();
    return p_ < s_.size() && s_[p_] == c;
  }
  bool take(char c) {
    if (peek(c)) {
      ++p_;
      return true;
    }
    return false;
  }
  void expect(char c) {
    if (!take(c)) throw CkptError(std::string("malformed checkpoint header: expected '") + c + "'");
  }
  std::string str() {
    expect('"');
    std::string r;
    while (p_ < s_.size() && s_[p_] != '"') {
      if (s_[p_] == '\\' && p_ + 1 < s_.size()) ++p_;
      r += s_[p_++];
    }
    expect('"');
    return r;
  }
  int64_t integer() {
    ws();
    size_t q = p_;
    if (q < s_.size() && s_[q] == '-') ++q;
    while (q < s_.size() && s_[q] >= '0' && s_[q] <= '9') ++q;
    if (q == p_) throw CkptError("malformed checkpoint header: expected an integer");
    const int64_t v = std::stoll(s_.substr(p_, q - p_));
    p_ = q;
    return v;
  }
  CkptTensor entry() {
    CkptTensor t;
    expect('{');
    do {
      const std::string key = str();
      expect(':');
      if (key == "shape") {
        expect('[');
        if (!peek(']')) {
          do t.shape.push_back(integer());
          while (take(','));
        }
        expect(']');
      } else if (key == "offset") {
        t.offset = static_cast<uint64_t>(integer());
      } else {
        skip_value();
      }
    } while (take(','));
    expect('}');
    return t;
  }
  void skip_value() {
    ws();
    if (peek('"')) {
      str();
    } else if (take('{')) {
      if (!peek('}')) {
        do {
          str();
          expect(':');
          skip_value();
        } while (take(','));
      }
      expect('}');
    } else if (take('[')) {
      if (!peek(']')) {
        do skip_value();
        while (take(','));
      }
      expect(']');
    } else {
      while (p_ < s_.size() && s_[p_] != ',' && s_[p_] != '}' && s_[p_] != ']') ++p_;
    }
  }
};

struct Checkpoint {
  std::map<std::string, CkptTensor> tensors;
  std::vector<uint8_t> blob;
  size_t payload = 0;

  static Checkpoint load(const std::string& path) {
    std::ifstream f(path, std::ios::binary);
    if (!f) throw CkptError("cannot open checkpoint " + path);
    Checkpoint c;
    c.blob.assign(std::istreambuf_iterator<char>(f), std::istreambuf_iterator<char>());
    static const char kMagic[8] = {'C', 'L', 'C', 'K', 'P', 'T', '1', '\0'};
    if (c.blob.size() < 16 || std::memcmp(c.blob.data(), kMagic, 8) != 0) throw CkptError("not a checkpoint file: " + path);
    uint64_t hl = 0;
    std::memcpy(&hl, c.blob.data() + 8, 8);
    if (16 + hl > c.blob.size()) throw CkptError("truncated checkpoint header");
    const std::string header(reinterpret_cast<const char*>(c.blob.data()) + 16, static_cast<size_t>(hl));
    c.tensors = HeaderParser(header).parse();
    c.payload = 16 + static_cast<size_t>(hl);
    return c;
  }

  // fp32 values of `name`, checked against the expected shape. The payload starts right after a
  // header of arbitrary length, so tensors are not 4-byte aligned in the file: copy them out.
  std::vector<float> get(const std::string& name, const std::vector<int64_t>& shape) const {
    auto it = tensors.find(name);
    if (it == tensors.end()) throw CkptError("checkpoint has no tensor '" + name + "'");
    if (it->second.shape != shape) throw CkptError("tensor '" + name + "' has an unexpected shape");
    size_t n = 1;
    for (int64_t e : shape) n *= static_cast<size_t>(e);
    if (payload + it->second.offset + n * 4 > blob.size()) throw CkptError("checkpoint payload truncated for '" + name + "'");
    std::vector<float> v(n);
    std::memcpy(v.data(), blob.data() + payload + it->second.offset, n * 4);
    return v;
  }

  // Writer: name -> (shape, values), header as nlohmann::json::dump() prints it for this layout.
  static void save(const std::string& path,
                   const std::map<std::string, std::pair<std::vector<int64_t>, const float*>>& ts) {
    std::string header = "{\"tensors\":{";
    uint64_t off = 0;
    bool first = true;
    for (const auto& [name, t] : ts) {
      if (!first) header += ",";
      first = false;
      header += "\"" + name + "\":{\"offset\":" + std::to_string(off) + ",\"shape\":[";
      size_t n = 1;
      for (size_t i = 0; i < t.first.size(); ++i) {
        header += (i ? "," : "") + std::to_string(t.first[i]);
        n *= static_cast<size_t>(t.first[i]);
      }
      header += "]}";
      off += n * 4;
    }
    header += "}}";
    std::ofstream f(path, std::ios::binary);
    if (!f) throw CkptError("cannot write checkpoint " + path);
    f.write("CLCKPT1\0", 8);
    const uint64_t hl = header.size();
    f.write(reinterpret_cast<const char*>(&hl), 8);
    f.write(header.data(), static_cast<std::streamsize>(header.size()));
    for (const auto& [name, t] : ts) {
      size_t n = 1;
      for (int64_t e : t.first) n *= static_cast<size_t>(e);
      f.write(reinterpret_cast<const char*>(t.second), static_cast<std::streamsize>(n * 4));
    }
    if (!f) throw CkptError("short write to " + path);
  }
};

}  // namespace cmoe
