// cmgb_json.hpp — a small JSON reader / writer for the C++ drop-in's scene
// ingest and manifold writers (include/cmgb_cmg.hpp: parse_scene, load_scene,
// manifold_to_json). The reference uses nlohmann::json for these
// (src/scene.cpp, src/manifold_io.cpp), which it does not vendor; this header
// covers the subset the scene schema and the JSON mirror need: objects,
// arrays, strings (with escapes), numbers, booleans, null. Output follows
// nlohmann's dump(2): two-space indentation, object keys sorted (std::map),
// doubles in the shortest round-trip form.
#pragma once

#include <charconv>
#include <cstdint>
#include <cstdlib>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <system_error>
#include <vector>

namespace cmgb {
namespace json {

struct ParseError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct TypeError : std::runtime_error {  // nlohmann: json::type_error
  using std::runtime_error::runtime_error;
};
struct KeyError : std::runtime_error {  // nlohmann: json::out_of_range
  using std::runtime_error::runtime_error;
};

struct Value {
  enum Kind { kNull, kBool, kNumber, kString, kArray, kObject } kind = kNull;
  bool b = false;
  double num = 0.0;
  bool integral = false;  // written without a fraction (an integer literal)
  std::string str;
  std::vector<Value> arr;
  std::map<std::string, Value> obj;

  bool is_array() const { return kind == kArray; }
  bool is_object() const { return kind == kObject; }
  bool is_number() const { return kind == kNumber; }
  bool is_string() const { return kind == kString; }
  bool is_bool() const { return kind == kBool; }
  size_t size() const { return kind == kArray ? arr.size() : kind == kObject ? obj.size() : 0; }
  bool contains(const std::string& k) const { return kind == kObject && obj.count(k) > 0; }
  const Value& at(const std::string& k) const {
    if (!contains(k)) throw KeyError("[json.exception.out_of_range.403] key '" + k + "' not found");
    return obj.at(k);
  }
  const Value& operator[](size_t i) const { return arr.at(i); }
  double as_number() const {
    if (kind == kNumber) return num;
    if (kind == kBool) return b ? 1.0 : 0.0;
    throw TypeError("[json.exception.type_error.302] type must be number");
  }
  bool as_bool() const {
    if (kind == kBool) return b;
    throw TypeError("[json.exception.type_error.302] type must be boolean");
  }
  const std::string& as_string() const {
    if (kind == kString) return str;
    throw TypeError("[json.exception.type_error.302] type must be string");
  }
  // nlohmann's value(key, default)
  double value(const std::string& k, double d) const { return contains(k) ? at(k).as_number() : d; }
  int value(const std::string& k, int d) const { return contains(k) ? (int)at(k).as_number() : d; }
  bool value(const std::string& k, bool d) const { return contains(k) ? at(k).as_bool() : d; }
  std::string value(const std::string& k, const std::string& d) const { return contains(k) ? at(k).as_string() : d; }

  static Value number(double v) {
    Value x;
    x.kind = kNumber;
    x.num = v;
    return x;
  }
  static Value integer(long long v) {
    Value x = number((double)v);
    x.integral = true;
    return x;
  }
  static Value string(std::string s) {
    Value x;
    x.kind = kString;
    x.str = std::move(s);
    return x;
  }
  static Value array() {
    Value x;
    x.kind = kArray;
    return x;
  }
  static Value object() {
    Value x;
    x.kind = kObject;
    return x;
  }
};

namespace detail {

struct Reader {
  const std::string& t;
  size_t i = 0;
  [[noreturn]] void fail(const std::string& what) const {
    throw ParseError("[json.exception.parse_error] at byte " + std::to_string(i + 1) + ": " + what);
  }
  void ws() {
    while (i < t.size() && (t[i] == ' ' || t[i] == '\t' || t[i] == '\n' || t[i] == '\r')) ++i;
  }
  bool eat(char c) {
    ws();
    if (i < t.size() && t[i] == c) {
      ++i;
      return true;
    }
    return false;
  }
  void expect(char c) {
    if (!eat(c)) fail(std::string("expected '") + c + "'");
  }
  std::string str() {
    expect('"');
    std::string out;
    while (true) {
      if (i >= t.size()) fail("unterminated string");
      const char c = t[i++];
      if (c == '"') break;
      if (c != '\\') {
        out += c;
        continue;
      }
      if (i >= t.size()) fail("bad escape");
      const char e = t[i++];
      switch (e) {
        case '"': out += '"'; break;
        case '\\': out += '\\'; break;
        case '/': out += '/'; break;
        case 'b': out += '\b'; break;
        case 'f': out += '\f'; break;
        case 'n': out += '\n'; break;
        case 'r': out += '\r'; break;
        case 't': out += '\t'; break;
        case 'u': {
          if (i + 4 > t.size()) fail("bad \\u escape");
          const unsigned cp = (unsigned)std::strtoul(t.substr(i, 4).c_str(), nullptr, 16);
          i += 4;
          if (cp < 0x80) {
            out += (char)cp;
          } else if (cp < 0x800) {
            out += (char)(0xC0 | (cp >> 6));
            out += (char)(0x80 | (cp & 0x3F));
          } else {
            out += (char)(0xE0 | (cp >> 12));
            out += (char)(0x80 | ((cp >> 6) & 0x3F));
            out += (char)(0x80 | (cp & 0x3F));
          }
          break;
        }
        default: fail("bad escape");
      }
    }
    return out;
  }
  Value val() {
    ws();
    if (i >= t.size()) fail("unexpected end of input");
    const char c = t[i];
    if (c == '{') {
      ++i;
      Value v = Value::object();
      if (eat('}')) return v;
      do {
        ws();
        std::string k = str();
        expect(':');
        v.obj[k] = val();
      } while (eat(','));
      expect('}');
      return v;
    }
    if (c == '[') {
      ++i;
      Value v = Value::array();
      if (eat(']')) return v;
      do v.arr.push_back(val());
      while (eat(','));
      expect(']');
      return v;
    }
    if (c == '"') return Value::string(str());
    if (t.compare(i, 4, "true") == 0) {
      i += 4;
      Value v;
      v.kind = Value::kBool;
      v.b = true;
      return v;
    }
    if (t.compare(i, 5, "false") == 0) {
      i += 5;
      Value v;
      v.kind = Value::kBool;
      return v;
    }
    if (t.compare(i, 4, "null") == 0) {
      i += 4;
      return Value();
    }
    const char* s = t.c_str() + i;
    char* end = nullptr;
    const double d = std::strtod(s, &end);
    if (end == s) fail("syntax error");
    const std::string lit(s, (size_t)(end - s));
    i += (size_t)(end - s);
    Value v = Value::number(d);
    v.integral = lit.find_first_of(".eE") == std::string::npos;
    return v;
  }
};

inline std::string num(const Value& v) {
  if (v.integral) return std::to_string((long long)v.num);
  char buf[64];
  const auto r = std::to_chars(buf, buf + sizeof(buf), v.num);  // shortest round trip
  std::string s(buf, r.ptr);
  if (s.find_first_of(".eEn") == std::string::npos) s += ".0";  // nlohmann keeps doubles visibly non-integral
  return s;
}

inline std::string quote(const std::string& s) {
  std::string o = "\"";
  for (char c : s) {
    if (c == '"' || c == '\\') {
      o += '\\';
      o += c;
    } else if (c == '\n') {
      o += "\\n";
    } else {
      o += c;
    }
  }
  return o + "\"";
}

inline void dump(const Value& v, int indent, int depth, std::string& out) {
  const std::string pad((size_t)indent * (depth + 1), ' '), pad0((size_t)indent * depth, ' ');
  switch (v.kind) {
    case Value::kNull: out += "null"; return;
    case Value::kBool: out += v.b ? "true" : "false"; return;
    case Value::kNumber: out += num(v); return;
    case Value::kString: out += quote(v.str); return;
    case Value::kArray: {
      if (v.arr.empty()) {
        out += "[]";
        return;
      }
      out += "[\n";
      for (size_t k = 0; k < v.arr.size(); ++k) {
        out += pad;
        dump(v.arr[k], indent, depth + 1, out);
        out += k + 1 < v.arr.size() ? ",\n" : "\n";
      }
      out += pad0 + "]";
      return;
    }
    case Value::kObject: {
      if (v.obj.empty()) {
        out += "{}";
        return;
      }
      out += "{\n";
      size_t k = 0;
      for (const auto& [key, x] : v.obj) {
        out += pad + quote(key) + ": ";
        dump(x, indent, depth + 1, out);
        out += ++k < v.obj.size() ? ",\n" : "\n";
      }
      out += pad0 + "}";
      return;
    }
  }
}

}  // namespace detail

inline Value parse(const std::string& text) {
  detail::Reader r{text};
  Value v = r.val();
  r.ws();
  if (r.i != text.size()) r.fail("trailing characters");
  return v;
}

inline std::string dump(const Value& v, int indent = 2) {
  std::string out;
  detail::dump(v, indent, 0, out);
  return out;
}

}  // namespace json
}  // namespace cmgb
