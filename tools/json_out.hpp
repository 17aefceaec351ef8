// Minimal insertion-ordered JSON value + writer for the CLI reports (the reference prints with
// an ordered JSON library at indent 2).  Doubles are written as the shortest round-trip digits in
// that library's layout: plain decimal for decimal exponents in (-4, 15], else d.ddde+XX; integral
// doubles keep a trailing ".0"; non-finite values become null.
#pragma once

#include <charconv>
#include <cstdio>
#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace sejson {

inline std::string fmt_double(double v) {
  if (!std::isfinite(v)) return "null";
  if (v == 0.0) return std::signbit(v) ? "-0.0" : "0.0";
  char buf[64];
  const auto r = std::to_chars(buf, buf + sizeof buf, v, std::chars_format::scientific);
  std::string s(buf, r.ptr);
  const bool neg = s[0] == '-';
  if (neg) s.erase(0, 1);
  const std::size_t e = s.find('e');
  const int ex = std::stoi(s.substr(e + 1));
  std::string digits;
  for (std::size_t i = 0; i < e; ++i)
    if (s[i] != '.') digits += s[i];
  const int k = (int)digits.size(), n = ex + 1;  // value = 0.digits x 10^n
  std::string out;
  if (k <= n && n <= 15) {
    out = digits + std::string((std::size_t)(n - k), '0') + ".0";
  } else if (0 < n && n <= 15) {
    out = digits.substr(0, (std::size_t)n) + "." + digits.substr((std::size_t)n);
  } else if (-4 < n && n <= 0) {
    out = "0." + std::string((std::size_t)(-n), '0') + digits;
  } else {
    out = digits.substr(0, 1);
    if (k > 1) out += "." + digits.substr(1);
    const int e10 = n - 1, ae = e10 < 0 ? -e10 : e10;
    out += e10 < 0 ? "e-" : "e+";
    if (ae < 10) out += '0';
    out += std::to_string(ae);
  }
  return neg ? "-" + out : out;
}

inline std::string quote(const std::string& s) {
  std::string o = "\"";
  for (unsigned char c : s) {
    switch (c) {
      case '"': o += "\\\""; break;
      case '\\': o += "\\\\"; break;
      case '\n': o += "\\n"; break;
      case '\r': o += "\\r"; break;
      case '\t': o += "\\t"; break;
      case '\b': o += "\\b"; break;
      case '\f': o += "\\f"; break;
      default:
        if (c < 0x20) {
          char u[8];
          std::snprintf(u, sizeof u, "\\u%04x", c);
          o += u;
        } else {
          o += (char)c;
        }
    }
  }
  return o + "\"";
}

class Json {
 public:
  enum Kind { kNull, kBool, kInt, kReal, kStr, kArr, kObj };
  Json() = default;
  Json(bool b) : k_(kBool), b_(b) {}
  Json(int i) : k_(kInt), i_(i) {}
  Json(long i) : k_(kInt), i_(i) {}
  Json(long long i) : k_(kInt), i_(i) {}
  Json(unsigned long i) : k_(kInt), i_((long long)i) {}
  Json(double d) : k_(kReal), d_(d) {}
  Json(const char* s) : k_(kStr), s_(s) {}
  Json(std::string s) : k_(kStr), s_(std::move(s)) {}
  template <class T>
  Json(const std::vector<T>& v) : k_(kArr) {
    for (const T& x : v) a_.emplace_back(x);
  }
  static Json array() {
    Json j;
    j.k_ = kArr;
    return j;
  }
  static Json object() {
    Json j;
    j.k_ = kObj;
    return j;
  }
  Json& operator[](const std::string& key) {
    if (k_ == kNull) k_ = kObj;
    if (k_ != kObj) throw std::logic_error("json: not an object");
    for (auto& kv : o_)
      if (kv.first == key) return kv.second;
    o_.emplace_back(key, Json());
    return o_.back().second;
  }
  void push_back(Json v) {
    if (k_ == kNull) k_ = kArr;
    if (k_ != kArr) throw std::logic_error("json: not an array");
    a_.push_back(std::move(v));
  }
  std::string dump(int indent = 2) const {
    std::string out;
    write(out, indent, 0);
    return out;
  }

 private:
  void write(std::string& out, int ind, int depth) const {
    const std::string pad((std::size_t)(ind * (depth + 1)), ' '), end((std::size_t)(ind * depth), ' ');
    switch (k_) {
      case kNull: out += "null"; break;
      case kBool: out += b_ ? "true" : "false"; break;
      case kInt: out += std::to_string(i_); break;
      case kReal: out += fmt_double(d_); break;
      case kStr: out += quote(s_); break;
      case kArr:
        if (a_.empty()) {
          out += "[]";
          break;
        }
        out += "[\n";
        for (std::size_t i = 0; i < a_.size(); ++i) {
          out += pad;
          a_[i].write(out, ind, depth + 1);
          out += i + 1 < a_.size() ? ",\n" : "\n";
        }
        out += end + "]";
        break;
      case kObj:
        if (o_.empty()) {
          out += "{}";
          break;
        }
        out += "{\n";
        for (std::size_t i = 0; i < o_.size(); ++i) {
          out += pad + quote(o_[i].first) + ": ";
          o_[i].second.write(out, ind, depth + 1);
          out += i + 1 < o_.size() ? ",\n" : "\n";
        }
        out += end + "}";
        break;
    }
  }
  Kind k_ = kNull;
  bool b_ = false;
  long long i_ = 0;
  double d_ = 0.0;
  std::string s_;
  std::vector<Json> a_;
  std::vector<std::pair<std::string, Json>> o_;
};

}  // namespace sejson
