// FP8 quantization scheme file ("Scheme file: JSON manifest + binary scale arrays";
// QuantScheme fields SPEC.md:520-523: smoothing vector s[d], per-output-channel weight scales,
// per-tensor activation scales, tau, alpha_smooth).
//
//   <path>       JSON manifest: format/version, layer shape, alpha_smooth, tau, router mode, the
//                binary file name and one entry per array {name, dtype "f32", shape, offset}
//   <path>.bin   the arrays, little-endian float32, concatenated at the manifest's byte offsets
//
// Arrays (reference orientation, this rank's experts under EP):
//   smoothing [d], act_scale_in [N] (every expert: the source quantizes with the owner's scale),
//   act_scale_mid [N_local], w_in_scale [N_local][2f] (reference W_in column order: gate then up),
//   w_out_scale [N_local][d], router_act_scale [1], router_w_scale [N].
// Host-only code (no CUDA): a minimal JSON value reader and the manifest writer.
#pragma once
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iterator>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace cmoe {

class SchemeError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

// JSON value: null, bool, number, string, array, object.
struct JVal {
  enum Kind { Null, Bool, Num, Str, Arr, Obj } kind = Null;
  double num = 0.0;
  bool b = false;
  std::string str;
  std::vector<JVal> arr;
  std::map<std::string, JVal> obj;
  const JVal& at(const std::string& k) const {
    auto it = obj.find(k);
    if (kind != Obj || it == obj.end()) throw SchemeError("scheme manifest: missing key \"" + k + "\"");
    return it->second;
  }
  bool has(const std::string& k) const { return kind == Obj && obj.count(k); }
  double number() const {
    if (kind != Num) throw SchemeError("scheme manifest: number expected");
    return num;
  }
};

class JsonReader {
 public:
  explicit JsonReader(const std::string& s) : s_(s) {}
  JVal parse() {
    JVal v = value();
    ws();
    if (p_ != s_.size()) fail("trailing characters");
    return v;
  }

 private:
  const std::string& s_;
  size_t p_ = 0;
  [[noreturn]] void fail(const char* what) {
    throw SchemeError(std::string("scheme manifest: ") + what + " at byte " + std::to_string(p_));
  }
  void ws() {
    while (p_ < s_.size() && (s_[p_] == ' ' || s_[p_] == '\n' || s_[p_] == '\t' || s_[p_] == '\r')) ++p_;
  }
  bool take(char c) {
    ws();
    if (p_ < s_.size() && s_[p_] == c) {
      ++p_;
      return true;
    }
    return false;
  }
  void expect(char c) {
    if (!take(c)) fail("unexpected character");
  }
  bool word(const char* w) {
    const size_t n = std::char_traits<char>::length(w);
    if (s_.compare(p_, n, w) == 0) {
      p_ += n;
      return true;
    }
    return false;
  }
  std::string string() {
    expect('"');
    std::string out;
    while (p_ < s_.size() && s_[p_] != '"') {
      char c = s_[p_++];
      if (c == '\\') {
        if (p_ >= s_.size()) fail("bad escape");
        const char e = s_[p_++];
        c = e == 'n' ? '\n' : e == 't' ? '\t' : e == 'r' ? '\r' : e == 'b' ? '\b' : e == 'f' ? '\f' : e;
        if (e == 'u') fail("\\u escapes are not supported");
      }
      out += c;
    }
    if (p_ >= s_.size()) fail("unterminated string");
    ++p_;
    return out;
  }
  JVal value() {
    ws();
    if (p_ >= s_.size()) fail("unexpected end");
    JVal v;
    const char c = s_[p_];
    if (c == '{') {
      ++p_;
      v.kind = JVal::Obj;
      if (take('}')) return v;
      do {
        ws();
        const std::string k = string();
        expect(':');
        v.obj[k] = value();
      } while (take(','));
      expect('}');
    } else if (c == '[') {
      ++p_;
      v.kind = JVal::Arr;
      if (take(']')) return v;
      do v.arr.push_back(value());
      while (take(','));
      expect(']');
    } else if (c == '"') {
      v.kind = JVal::Str;
      v.str = string();
    } else if (word("null")) {
      v.kind = JVal::Null;
    } else if (word("true")) {
      v.kind = JVal::Bool;
      v.b = true;
    } else if (word("false")) {
      v.kind = JVal::Bool;
    } else {
      const char* b = s_.c_str() + p_;
      char* e = nullptr;
      v.num = std::strtod(b, &e);
      if (e == b) fail("value expected");
      p_ += static_cast<size_t>(e - b);
      v.kind = JVal::Num;
    }
    return v;
  }
};

struct SchemeArray {
  std::string name;
  std::vector<int64_t> shape;
  std::vector<float> data;
};

struct Scheme {
  int64_t d = 0, N = 0, f = 0, n_local = 0, expert0 = 0, ep_size = 1;
  double alpha = NAN;   // alpha_smooth of the last compute_smoothing (NaN: none -> null)
  int64_t tau = -1;     // tau of the last balance_calibration (-1: none -> null)
  int router_fp8 = 1;
  std::vector<SchemeArray> arrays;
  const SchemeArray& get(const std::string& n) const {
    for (const auto& a : arrays)
      if (a.name == n) return a;
    throw SchemeError("scheme file has no array \"" + n + "\"");
  }
};

inline std::string base_name(const std::string& p) {
  const size_t s = p.find_last_of('/');
  return s == std::string::npos ? p : p.substr(s + 1);
}
inline std::string dir_name(const std::string& p) {
  const size_t s = p.find_last_of('/');
  return s == std::string::npos ? std::string() : p.substr(0, s + 1);
}

inline void write_scheme(const std::string& path, const Scheme& sc) {
  const std::string bin = path + ".bin";
  std::ofstream fb(bin, std::ios::binary);
  if (!fb) throw SchemeError("cannot write " + bin);
  std::string arrs;
  uint64_t off = 0;
  for (const auto& a : sc.arrays) {
    fb.write(reinterpret_cast<const char*>(a.data.data()), static_cast<std::streamsize>(a.data.size() * 4));
    std::string shp;
    for (size_t i = 0; i < a.shape.size(); ++i) shp += (i ? "," : "") + std::to_string(a.shape[i]);
    if (!arrs.empty()) arrs += ",\n    ";
    arrs += "{\"name\": \"" + a.name + "\", \"dtype\": \"f32\", \"shape\": [" + shp + "], \"offset\": " +
            std::to_string(off) + "}";
    off += a.data.size() * 4;
  }
  if (!fb) throw SchemeError("write failed: " + bin);
  char alpha[64];
  if (std::isnan(sc.alpha)) std::snprintf(alpha, sizeof alpha, "null");
  else std::snprintf(alpha, sizeof alpha, "%.9g", sc.alpha);
  std::ofstream fm(path);
  if (!fm) throw SchemeError("cannot write " + path);
  fm << "{\n  \"format\": \"compass_moe.fp8_scheme\",\n  \"version\": 1,\n  \"fp8\": \"e4m3\",\n"
     << "  \"d_model\": " << sc.d << ",\n  \"n_experts\": " << sc.N << ",\n  \"d_ff\": " << sc.f
     << ",\n  \"ep_size\": " << sc.ep_size << ",\n  \"expert0\": " << sc.expert0 << ",\n  \"n_local\": " << sc.n_local
     << ",\n  \"alpha_smooth\": " << alpha << ",\n  \"tau\": " << (sc.tau < 0 ? std::string("null") : std::to_string(sc.tau))
     << ",\n  \"router_fp8\": " << sc.router_fp8 << ",\n  \"weight_scales\": \"per output channel, absmax/448\""
     << ",\n  \"activation_scales\": \"per tensor (per expert: expert-aware), calibration max/448\""
     << ",\n  \"data\": \"" << base_name(bin) << "\",\n  \"arrays\": [\n    " << arrs << "\n  ]\n}\n";
  if (!fm) throw SchemeError("write failed: " + path);
}

inline Scheme read_scheme(const std::string& path) {
  std::ifstream fm(path);
  if (!fm) throw SchemeError("cannot open " + path);
  const std::string txt((std::istreambuf_iterator<char>(fm)), std::istreambuf_iterator<char>());
  const JVal m = JsonReader(txt).parse();
  if (m.kind != JVal::Obj || !m.has("format") || m.at("format").str != "compass_moe.fp8_scheme")
    throw SchemeError(path + " is not a compass_moe FP8 scheme manifest");
  if (m.at("version").number() != 1) throw SchemeError("unsupported scheme version");
  Scheme sc;
  sc.d = static_cast<int64_t>(m.at("d_model").number());
  sc.N = static_cast<int64_t>(m.at("n_experts").number());
  sc.f = static_cast<int64_t>(m.at("d_ff").number());
  sc.ep_size = static_cast<int64_t>(m.at("ep_size").number());
  sc.expert0 = static_cast<int64_t>(m.at("expert0").number());
  sc.n_local = static_cast<int64_t>(m.at("n_local").number());
  sc.alpha = m.at("alpha_smooth").kind == JVal::Num ? m.at("alpha_smooth").num : NAN;
  sc.tau = m.at("tau").kind == JVal::Num ? static_cast<int64_t>(m.at("tau").num) : -1;
  sc.router_fp8 = static_cast<int>(m.at("router_fp8").number());
  const std::string bin = dir_name(path) + m.at("data").str;
  std::ifstream fb(bin, std::ios::binary);
  if (!fb) throw SchemeError("cannot open " + bin);
  const std::string raw((std::istreambuf_iterator<char>(fb)), std::istreambuf_iterator<char>());
  for (const JVal& e : m.at("arrays").arr) {
    SchemeArray a;
    a.name = e.at("name").str;
    if (e.at("dtype").str != "f32") throw SchemeError("array " + a.name + ": only f32 is supported");
    int64_t n = 1;
    for (const JVal& s : e.at("shape").arr) {
      a.shape.push_back(static_cast<int64_t>(s.number()));
      n *= a.shape.back();
    }
    const uint64_t off = static_cast<uint64_t>(e.at("offset").number());
    if (n < 0 || off + static_cast<uint64_t>(n) * 4 > raw.size()) throw SchemeError("array " + a.name + " exceeds " + bin);
    a.data.resize(static_cast<size_t>(n));
    std::memcpy(a.data.data(), raw.data() + off, static_cast<size_t>(n) * 4);
    sc.arrays.push_back(std::move(a));
  }
  return sc;
}

}  // namespace cmoe
