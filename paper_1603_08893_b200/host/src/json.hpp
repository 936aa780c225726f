// Minimal JSON value, parser and emitter for the run/snapshot records.
//
// The emitter reproduces the byte layout the reference's records carry
// (nlohmann::json dump(2), as in proj/unit_run_out/meta_1.json): object keys
// sorted, two-space indentation, one array element per line, integers
// without a fraction, doubles as their shortest round-trip decimal with a
// ".0" suffix when integral and an exponent outside 1e-5 .. 1e15.
#pragma once

#include <cstdint>
#include <map>
#include <string>
#include <vector>

namespace fftmech::json {

struct Value {
  enum Kind { Null, Bool, Int, Real, String, Array, Object };
  Kind kind = Null;
  bool b = false;
  int64_t i = 0;
  double d = 0.0;
  std::string s;
  std::vector<Value> a;
  std::map<std::string, Value> o;  // sorted keys, like nlohmann::json

  Value() = default;
  static Value null() { return Value(); }
  static Value boolean(bool v) {
    Value x;
    x.kind = Bool;
    x.b = v;
    return x;
  }
  static Value integer(int64_t v) {
    Value x;
    x.kind = Int;
    x.i = v;
    return x;
  }
  static Value real(double v) {
    Value x;
    x.kind = Real;
    x.d = v;
    return x;
  }
  static Value string(std::string v) {
    Value x;
    x.kind = String;
    x.s = std::move(v);
    return x;
  }
  static Value array() {
    Value x;
    x.kind = Array;
    return x;
  }
  static Value object() {
    Value x;
    x.kind = Object;
    return x;
  }

  bool is_number() const { return kind == Int || kind == Real; }
  double number() const { return kind == Int ? static_cast<double>(i) : d; }
  const Value* find(const std::string& key) const {
    if (kind != Object) return nullptr;
    auto it = o.find(key);
    return it == o.end() ? nullptr : &it->second;
  }
  Value& operator[](const std::string& key) {
    kind = Object;
    return o[key];
  }
  void push(Value v) {
    kind = Array;
    a.push_back(std::move(v));
  }
};

// Throws std::runtime_error("json: <what> at offset <k>") on malformed text.
Value parse(const std::string& text);
std::string dump(const Value& v, int indent = 2);
std::string format_double(double v);

}  // namespace fftmech::json
