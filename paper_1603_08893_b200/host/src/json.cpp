#include "json.hpp"

#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>

namespace fftmech::json {

namespace {

struct Parser {
  const std::string& t;
  size_t k = 0;

  [[noreturn]] void fail(const char* what) const {
    throw std::runtime_error(std::string("json: ") + what + " at offset " + std::to_string(k));
  }
  void ws() {
    while (k < t.size() && (t[k] == ' ' || t[k] == '\t' || t[k] == '\n' || t[k] == '\r')) ++k;
  }
  bool eat(char c) {
    ws();
    if (k < t.size() && t[k] == c) {
      ++k;
      return true;
    }
    return false;
  }
  void expect(char c) {
    if (!eat(c)) fail((std::string("expected '") + c + "'").c_str());
  }
  bool word(const char* w) {
    size_t n = 0;
    while (w[n]) ++n;
    if (t.compare(k, n, w) == 0) {
      k += n;
      return true;
    }
    return false;
  }
  static void utf8(std::string& out, unsigned cp) {
    if (cp < 0x80) {
      out += char(cp);
    } else if (cp < 0x800) {
      out += char(0xC0 | (cp >> 6));
      out += char(0x80 | (cp & 0x3F));
    } else if (cp < 0x10000) {
      out += char(0xE0 | (cp >> 12));
      out += char(0x80 | ((cp >> 6) & 0x3F));
      out += char(0x80 | (cp & 0x3F));
    } else {
      out += char(0xF0 | (cp >> 18));
      out += char(0x80 | ((cp >> 12) & 0x3F));
      out += char(0x80 | ((cp >> 6) & 0x3F));
      out += char(0x80 | (cp & 0x3F));
    }
  }
  unsigned hex4() {
    if (k + 4 > t.size()) fail("truncated \\u escape");
    unsigned v = 0;
    for (int q = 0; q < 4; ++q) {
      const char c = t[k++];
      v <<= 4;
      if (c >= '0' && c <= '9') v |= unsigned(c - '0');
      else if (c >= 'a' && c <= 'f') v |= unsigned(c - 'a' + 10);
      else if (c >= 'A' && c <= 'F') v |= unsigned(c - 'A' + 10);
      else fail("bad \\u escape");
    }
    return v;
  }
  std::string str() {
    ws();
    if (k >= t.size() || t[k] != '"') fail("expected string");
    ++k;
    std::string out;
    while (true) {
      if (k >= t.size()) fail("unterminated string");
      const char c = t[k++];
      if (c == '"') break;
      if (static_cast<unsigned char>(c) < 0x20) fail("control character in string");
      if (c != '\\') {
        out += c;
        continue;
      }
      if (k >= t.size()) fail("unterminated escape");
      const char e = t[k++];
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
          unsigned cp = hex4();
          if (cp >= 0xD800 && cp < 0xDC00 && k + 1 < t.size() && t[k] == '\\' && t[k + 1] == 'u') {
            k += 2;
            const unsigned lo = hex4();
            cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
          }
          utf8(out, cp);
          break;
        }
        default: fail("bad escape");
      }
    }
    return out;
  }
  Value num() {
    const size_t s = k;
    if (k < t.size() && t[k] == '-') ++k;
    bool real = false;
    while (k < t.size()) {
      const char c = t[k];
      if (c >= '0' && c <= '9') {
        ++k;
      } else if (c == '.' || c == 'e' || c == 'E' || c == '+' || c == '-') {
        real = true;
        ++k;
      } else {
        break;
      }
    }
    const std::string tok = t.substr(s, k - s);
    if (tok.empty() || tok == "-") fail("bad number");
    if (!real) {
      int64_t v = 0;
      const auto r = std::from_chars(tok.data(), tok.data() + tok.size(), v);
      if (r.ec == std::errc() && r.ptr == tok.data() + tok.size()) return Value::integer(v);
    }
    char* end = nullptr;
    const double d = std::strtod(tok.c_str(), &end);
    if (end != tok.c_str() + tok.size()) fail("bad number");
    return Value::real(d);
  }
  Value value() {
    ws();
    if (k >= t.size()) fail("unexpected end");
    const char c = t[k];
    if (c == '{') {
      ++k;
      Value v = Value::object();
      if (eat('}')) return v;
      do {
        const std::string key = str();
        expect(':');
        v.o[key] = value();
      } while (eat(','));
      expect('}');
      return v;
    }
    if (c == '[') {
      ++k;
      Value v = Value::array();
      if (eat(']')) return v;
      do v.a.push_back(value());
      while (eat(','));
      expect(']');
      return v;
    }
    if (c == '"') return Value::string(str());
    if (word("true")) return Value::boolean(true);
    if (word("false")) return Value::boolean(false);
    if (word("null")) return Value::null();
    return num();
  }
};

std::string escape(const std::string& s) {
  std::string out = "\"";
  for (const char c : s) {
    switch (c) {
      case '"': out += "\\\""; break;
      case '\\': out += "\\\\"; break;
      case '\b': out += "\\b"; break;
      case '\f': out += "\\f"; break;
      case '\n': out += "\\n"; break;
      case '\r': out += "\\r"; break;
      case '\t': out += "\\t"; break;
      default:
        if (static_cast<unsigned char>(c) < 0x20) {
          char buf[8];
          std::snprintf(buf, sizeof buf, "\\u%04x", unsigned(c));
          out += buf;
        } else {
          out += c;
        }
    }
  }
  return out + "\"";
}

void emit(const Value& v, int indent, int depth, std::string& out) {
  const std::string pad(size_t(indent) * size_t(depth + 1), ' ');
  const std::string close(size_t(indent) * size_t(depth), ' ');
  switch (v.kind) {
    case Value::Null: out += "null"; break;
    case Value::Bool: out += v.b ? "true" : "false"; break;
    case Value::Int: out += std::to_string(v.i); break;
    case Value::Real: out += format_double(v.d); break;
    case Value::String: out += escape(v.s); break;
    case Value::Array:
      if (v.a.empty()) {
        out += "[]";
        break;
      }
      out += "[\n";
      for (size_t q = 0; q < v.a.size(); ++q) {
        out += pad;
        emit(v.a[q], indent, depth + 1, out);
        out += q + 1 < v.a.size() ? ",\n" : "\n";
      }
      out += close + "]";
      break;
    case Value::Object: {
      if (v.o.empty()) {
        out += "{}";
        break;
      }
      out += "{\n";
      size_t q = 0;
      for (const auto& [key, val] : v.o) {
        out += pad + escape(key) + ": ";
        emit(val, indent, depth + 1, out);
        out += ++q < v.o.size() ? ",\n" : "\n";
      }
      out += close + "}";
      break;
    }
  }
}

}  // namespace

Value parse(const std::string& text) {
  Parser p{text};
  Value v = p.value();
  p.ws();
  if (p.k != text.size()) p.fail("trailing characters");
  return v;
}

std::string dump(const Value& v, int indent) {
  std::string out;
  emit(v, indent, 0, out);
  return out;
}

std::string format_double(double v) {
  if (!std::isfinite(v)) return "null";
  if (v == 0.0) return std::signbit(v) ? "-0.0" : "0.0";
  // shortest round-trip digits and decimal exponent
  char buf[64];
  const auto r = std::to_chars(buf, buf + sizeof buf, v, std::chars_format::scientific);
  std::string sci(buf, r.ptr);
  std::string sign;
  if (sci[0] == '-') {
    sign = "-";
    sci.erase(0, 1);
  }
  const size_t e = sci.find('e');
  std::string digits = sci.substr(0, e);
  digits.erase(std::remove(digits.begin(), digits.end(), '.'), digits.end());
  const int exp10 = std::atoi(sci.c_str() + e + 1);
  const int kd = static_cast<int>(digits.size());
  const int n = exp10 + 1;  // decimal point position
  std::string out;
  if (kd <= n && n <= 15) {
    out = digits + std::string(size_t(n - kd), '0') + ".0";
  } else if (0 < n && n <= 15) {
    out = digits.substr(0, size_t(n)) + "." + digits.substr(size_t(n));
  } else if (-4 < n && n <= 0) {
    out = "0." + std::string(size_t(-n), '0') + digits;
  } else {
    out = digits.substr(0, 1);
    if (kd > 1) out += "." + digits.substr(1);
    char eb[16];
    std::snprintf(eb, sizeof eb, "e%c%02d", n - 1 < 0 ? '-' : '+', std::abs(n - 1));
    out += eb;
  }
  return sign + out;
}

}  // namespace fftmech::json
