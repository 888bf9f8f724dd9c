// Minimal JSON reader for the summary IR.
//
// Integers are parsed exactly into __int128 (summary constants are int64; the
// wider type lets the loader reject out-of-range literals instead of wrapping).
// Floats are rejected: the IR is integer-only.
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace picker {

struct JsonError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct Json {
  enum Kind { NUL, BOOL, INT, STR, ARR, OBJ } kind = NUL;
  bool b = false;
  __int128 i = 0;
  std::string s;
  std::vector<Json> a;
  std::vector<std::pair<std::string, Json>> o;

  bool is_null() const { return kind == NUL; }
  const Json* get(const std::string& key) const {
    if (kind != OBJ) return nullptr;
    for (auto& kv : o)
      if (kv.first == key) return &kv.second;
    return nullptr;
  }
  const Json& at(const std::string& key) const {
    const Json* j = get(key);
    if (!j) throw JsonError("missing key '" + key + "'");
    return *j;
  }
  const std::vector<Json>& arr() const {
    if (kind != ARR) throw JsonError("expected an array");
    return a;
  }
  const std::string& str() const {
    if (kind != STR) throw JsonError("expected a string");
    return s;
  }
  __int128 integer() const {
    if (kind != INT) throw JsonError("expected an integer");
    return i;
  }
  bool boolean() const {
    if (kind != BOOL) throw JsonError("expected a boolean");
    return b;
  }
};

class JsonParser {
 public:
  JsonParser(const char* p, size_t n) : p_(p), end_(p + n) {}
  Json parse() {
    Json v = value(0);
    ws();
    if (p_ != end_) fail("trailing characters");
    return v;
  }

 private:
  const char* p_;
  const char* end_;

  [[noreturn]] void fail(const char* what) {
    throw JsonError(std::string("JSON: ") + what);
  }
  void ws() {
    while (p_ < end_ && (*p_ == ' ' || *p_ == '\n' || *p_ == '\r' || *p_ == '\t')) ++p_;
  }
  bool lit(const char* w) {
    const char* q = p_;
    while (*w) {
      if (q >= end_ || *q != *w) return false;
      ++q, ++w;
    }
    p_ = q;
    return true;
  }
  Json value(int depth) {
    if (depth > 64) fail("nesting too deep");
    ws();
    if (p_ >= end_) fail("unexpected end");
    Json v;
    char c = *p_;
    if (c == '{') {
      v.kind = Json::OBJ;
      ++p_;
      ws();
      if (p_ < end_ && *p_ == '}') { ++p_; return v; }
      for (;;) {
        ws();
        if (p_ >= end_ || *p_ != '"') fail("expected a key");
        std::string k = string();
        ws();
        if (p_ >= end_ || *p_ != ':') fail("expected ':'");
        ++p_;
        v.o.emplace_back(std::move(k), value(depth + 1));
        ws();
        if (p_ < end_ && *p_ == ',') { ++p_; continue; }
        if (p_ < end_ && *p_ == '}') { ++p_; break; }
        fail("expected ',' or '}'");
      }
    } else if (c == '[') {
      v.kind = Json::ARR;
      ++p_;
      ws();
      if (p_ < end_ && *p_ == ']') { ++p_; return v; }
      for (;;) {
        v.a.push_back(value(depth + 1));
        ws();
        if (p_ < end_ && *p_ == ',') { ++p_; continue; }
        if (p_ < end_ && *p_ == ']') { ++p_; break; }
        fail("expected ',' or ']'");
      }
    } else if (c == '"') {
      v.kind = Json::STR;
      v.s = string();
    } else if (lit("true")) {
      v.kind = Json::BOOL, v.b = true;
    } else if (lit("false")) {
      v.kind = Json::BOOL, v.b = false;
    } else if (lit("null")) {
      v.kind = Json::NUL;
    } else if (c == '-' || (c >= '0' && c <= '9')) {
      v.kind = Json::INT;
      bool neg = false;
      if (*p_ == '-') { neg = true; ++p_; }
      if (p_ >= end_ || *p_ < '0' || *p_ > '9') fail("bad number");
      unsigned __int128 m = 0;
      const unsigned __int128 lim = (((unsigned __int128)1) << 126);
      while (p_ < end_ && *p_ >= '0' && *p_ <= '9') {
        m = m * 10 + (unsigned)(*p_ - '0');
        if (m > lim) fail("integer too large");
        ++p_;
      }
      if (p_ < end_ && (*p_ == '.' || *p_ == 'e' || *p_ == 'E')) fail("floats are not allowed");
      v.i = neg ? -(__int128)m : (__int128)m;
    } else {
      fail("unexpected character");
    }
    return v;
  }
  std::string string() {
    ++p_;  // opening quote
    std::string out;
    while (p_ < end_ && *p_ != '"') {
      if (*p_ == '\\') {
        ++p_;
        if (p_ >= end_) fail("bad escape");
        char e = *p_++;
        switch (e) {
          case '"': out += '"'; break;
          case '\\': out += '\\'; break;
          case '/': out += '/'; break;
          case 'n': out += '\n'; break;
          case 't': out += '\t'; break;
          case 'r': out += '\r'; break;
          case 'b': out += '\b'; break;
          case 'f': out += '\f'; break;
          case 'u': {
            if (end_ - p_ < 4) fail("bad \\u escape");
            unsigned cp = 0;
            for (int k = 0; k < 4; ++k) {
              char h = *p_++;
              cp <<= 4;
              if (h >= '0' && h <= '9') cp |= h - '0';
              else if (h >= 'a' && h <= 'f') cp |= h - 'a' + 10;
              else if (h >= 'A' && h <= 'F') cp |= h - 'A' + 10;
              else fail("bad \\u escape");
            }
            if (cp < 0x80) out += (char)cp;
            else out += '?';  // names are ASCII in practice; keep the parse total
            break;
          }
          default: fail("bad escape");
        }
      } else {
        out += *p_++;
      }
    }
    if (p_ >= end_) fail("unterminated string");
    ++p_;
    return out;
  }
};

}  // namespace picker
