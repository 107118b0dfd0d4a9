// TEST INFRASTRUCTURE — a small stand-in for the subset of nlohmann::json
// (vendored by the reference under proj/vendor/, git-ignored and absent:
// proj/.gitignore:2) that the reference's sim/scene.cpp,
// sim/terrain_spec.cpp and pipeline.cpp use for their config round trips:
// initializer-list construction (nlohmann's rule: a list of [string, value]
// pairs is an object, anything else an array), operator[], at, value,
// contains, get<T>, push_back, range-for over arrays, parse and dump.
// Objects keep keys sorted (std::map), as nlohmann::json does by default.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <initializer_list>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

namespace nlohmann {

class json {
 public:
  enum class Type { Null, Bool, Int, Float, String, Array, Object };
  using array_t = std::vector<json>;
  using object_t = std::map<std::string, json>;

  json() = default;
  json(std::nullptr_t) {}
  json(bool b) : t_(Type::Bool), b_(b) {}
  template <class T>
    requires(std::is_integral_v<T> && !std::is_same_v<T, bool>)
  json(T v) : t_(Type::Int), i_(static_cast<std::int64_t>(v)) {}
  template <class T>
    requires std::is_floating_point_v<T>
  json(T v) : t_(Type::Float), f_(static_cast<double>(v)) {}
  json(const char* s) : t_(Type::String), s_(s) {}
  json(const std::string& s) : t_(Type::String), s_(s) {}
  json(std::initializer_list<json> l) {
    bool is_object = l.size() > 0;
    for (const json& e : l)
      is_object = is_object && e.t_ == Type::Array && e.a_.size() == 2 && e.a_[0].t_ == Type::String;
    if (is_object) {
      t_ = Type::Object;
      for (const json& e : l) o_[e.a_[0].s_] = e.a_[1];
    } else {
      t_ = Type::Array;
      a_.assign(l.begin(), l.end());
    }
  }

  static json array() {
    json j;
    j.t_ = Type::Array;
    return j;
  }
  static json object() {
    json j;
    j.t_ = Type::Object;
    return j;
  }

  bool is_null() const { return t_ == Type::Null; }
  bool is_array() const { return t_ == Type::Array; }
  bool is_object() const { return t_ == Type::Object; }
  bool is_number() const { return t_ == Type::Int || t_ == Type::Float; }
  bool is_string() const { return t_ == Type::String; }
  std::size_t size() const {
    return t_ == Type::Array ? a_.size() : t_ == Type::Object ? o_.size() : (t_ == Type::Null ? 0 : 1);
  }
  bool empty() const { return size() == 0; }

  // ---- element access ------------------------------------------------------
  json& operator[](const std::string& k) {
    if (t_ == Type::Null) t_ = Type::Object;
    if (t_ != Type::Object) throw std::runtime_error("json: operator[] with a key on a non-object");
    return o_[k];
  }
  json& operator[](const char* k) { return (*this)[std::string(k)]; }
  const json& operator[](const std::string& k) const {
    static const json null_value;
    if (t_ != Type::Object) throw std::runtime_error("json: operator[] with a key on a non-object");
    auto it = o_.find(k);
    return it == o_.end() ? null_value : it->second;
  }
  const json& operator[](const char* k) const { return (*this)[std::string(k)]; }
  template <class I>
    requires std::is_integral_v<I>
  json& operator[](I i) {
    if (t_ == Type::Null) t_ = Type::Array;
    if (t_ != Type::Array) throw std::runtime_error("json: index on a non-array");
    if (static_cast<std::size_t>(i) >= a_.size()) a_.resize(static_cast<std::size_t>(i) + 1);
    return a_[static_cast<std::size_t>(i)];
  }
  template <class I>
    requires std::is_integral_v<I>
  const json& operator[](I i) const {
    if (t_ != Type::Array || static_cast<std::size_t>(i) >= a_.size())
      throw std::out_of_range("json: index out of range");
    return a_[static_cast<std::size_t>(i)];
  }
  const json& at(const std::string& k) const {
    if (t_ != Type::Object) throw std::runtime_error("json: at() on a non-object");
    auto it = o_.find(k);
    if (it == o_.end()) throw std::out_of_range("json: key '" + k + "' not found");
    return it->second;
  }
  json& at(const std::string& k) { return const_cast<json&>(static_cast<const json&>(*this).at(k)); }
  const json& at(std::size_t i) const {
    if (t_ != Type::Array || i >= a_.size()) throw std::out_of_range("json: index out of range");
    return a_[i];
  }
  bool contains(const std::string& k) const { return t_ == Type::Object && o_.count(k) != 0; }

  template <class T>
  T value(const std::string& k, const T& def) const {
    if (!contains(k)) return def;
    return o_.at(k).template get<T>();
  }
  std::string value(const std::string& k, const char* def) const { return value<std::string>(k, std::string(def)); }

  template <class T>
  T get() const {
    if constexpr (std::is_same_v<T, json>) {
      return *this;
    } else if constexpr (std::is_same_v<T, bool>) {
      if (t_ != Type::Bool) throw std::runtime_error("json: not a boolean");
      return b_;
    } else if constexpr (std::is_integral_v<T>) {
      if (t_ == Type::Int) return static_cast<T>(i_);
      if (t_ == Type::Float) return static_cast<T>(f_);
      throw std::runtime_error("json: not a number");
    } else if constexpr (std::is_floating_point_v<T>) {
      if (t_ == Type::Int) return static_cast<T>(i_);
      if (t_ == Type::Float) return static_cast<T>(f_);
      throw std::runtime_error("json: not a number");
    } else if constexpr (std::is_same_v<T, std::string>) {
      if (t_ != Type::String) throw std::runtime_error("json: not a string");
      return s_;
    } else {
      static_assert(sizeof(T) == 0, "json::get: unsupported type");
    }
  }
  template <class T>
  operator T() const
    requires(std::is_arithmetic_v<T> || std::is_same_v<T, std::string>)
  {
    return get<T>();
  }

  void push_back(const json& v) {
    if (t_ == Type::Null) t_ = Type::Array;
    if (t_ != Type::Array) throw std::runtime_error("json: push_back on a non-array");
    a_.push_back(v);
  }

  // range-for over array elements (object values for objects)
  class const_iterator {
   public:
    const_iterator(const json* j, std::size_t i, object_t::const_iterator it) : j_(j), i_(i), it_(it) {}
    const json& operator*() const { return j_->t_ == Type::Object ? it_->second : j_->a_[i_]; }
    const json* operator->() const { return &**this; }
    const_iterator& operator++() {
      if (j_->t_ == Type::Object)
        ++it_;
      else
        ++i_;
      return *this;
    }
    bool operator!=(const const_iterator& o) const { return i_ != o.i_ || it_ != o.it_; }
    bool operator==(const const_iterator& o) const { return !(*this != o); }
    std::string key() const { return it_->first; }

   private:
    const json* j_;
    std::size_t i_;
    object_t::const_iterator it_;
  };
  const_iterator begin() const { return const_iterator(this, 0, o_.begin()); }
  const_iterator end() const {
    return const_iterator(this, t_ == Type::Array ? a_.size() : 0, o_.end());
  }

  // ---- text ----------------------------------------------------------------
  std::string dump(int indent = -1) const {
    std::string out;
    write(out, indent, 0);
    return out;
  }
  static json parse(const std::string& text) {
    std::size_t p = 0;
    json j = parse_value(text, p);
    skip_ws(text, p);
    if (p != text.size()) throw std::runtime_error("json: trailing characters");
    return j;
  }

 private:
  static void newline(std::string& out, int indent, int depth) {
    if (indent < 0) return;
    out += '\n';
    out.append(static_cast<std::size_t>(indent * depth), ' ');
  }
  static void write_string(std::string& out, const std::string& s) {
    out += '"';
    for (char c : s) {
      switch (c) {
        case '"': out += "\\\""; break;
        case '\\': out += "\\\\"; break;
        case '\n': out += "\\n"; break;
        case '\t': out += "\\t"; break;
        case '\r': out += "\\r"; break;
        default: out += c;
      }
    }
    out += '"';
  }
  static std::string number(double v) {
    if (!std::isfinite(v)) return "null";
    char buf[64];
    for (int prec = 1; prec <= 17; ++prec) {
      std::snprintf(buf, sizeof buf, "%.*g", prec, v);
      if (std::strtod(buf, nullptr) == v) break;
    }
    std::string s(buf);
    if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
    return s;
  }
  void write(std::string& out, int indent, int depth) const {
    switch (t_) {
      case Type::Null: out += "null"; break;
      case Type::Bool: out += b_ ? "true" : "false"; break;
      case Type::Int: out += std::to_string(i_); break;
      case Type::Float: out += number(f_); break;
      case Type::String: write_string(out, s_); break;
      case Type::Array: {
        if (a_.empty()) {
          out += "[]";
          break;
        }
        out += '[';
        for (std::size_t i = 0; i < a_.size(); ++i) {
          if (i) out += ',';
          newline(out, indent, depth + 1);
          a_[i].write(out, indent, depth + 1);
        }
        newline(out, indent, depth);
        out += ']';
        break;
      }
      case Type::Object: {
        if (o_.empty()) {
          out += "{}";
          break;
        }
        out += '{';
        bool first = true;
        for (const auto& [k, v] : o_) {
          if (!first) out += ',';
          first = false;
          newline(out, indent, depth + 1);
          write_string(out, k);
          out += indent >= 0 ? ": " : ":";
          v.write(out, indent, depth + 1);
        }
        newline(out, indent, depth);
        out += '}';
        break;
      }
    }
  }
  static void skip_ws(const std::string& s, std::size_t& p) {
    while (p < s.size() && (s[p] == ' ' || s[p] == '\n' || s[p] == '\t' || s[p] == '\r')) ++p;
  }
  static void expect(const std::string& s, std::size_t& p, char c) {
    skip_ws(s, p);
    if (p >= s.size() || s[p] != c) throw std::runtime_error(std::string("json: expected '") + c + "'");
    ++p;
  }
  static std::string parse_string(const std::string& s, std::size_t& p) {
    expect(s, p, '"');
    std::string out;
    while (p < s.size() && s[p] != '"') {
      char c = s[p++];
      if (c == '\\') {
        if (p >= s.size()) break;
        const char e = s[p++];
        switch (e) {
          case 'n': out += '\n'; break;
          case 't': out += '\t'; break;
          case 'r': out += '\r'; break;
          case 'b': out += '\b'; break;
          case 'f': out += '\f'; break;
          case 'u': {
            const unsigned cp = static_cast<unsigned>(std::stoul(s.substr(p, 4), nullptr, 16));
            p += 4;
            if (cp < 0x80) {
              out += static_cast<char>(cp);
            } else if (cp < 0x800) {
              out += static_cast<char>(0xC0 | (cp >> 6));
              out += static_cast<char>(0x80 | (cp & 0x3F));
            } else {
              out += static_cast<char>(0xE0 | (cp >> 12));
              out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
              out += static_cast<char>(0x80 | (cp & 0x3F));
            }
            break;
          }
          default: out += e;
        }
      } else {
        out += c;
      }
    }
    if (p >= s.size()) throw std::runtime_error("json: unterminated string");
    ++p;
    return out;
  }
  static json parse_value(const std::string& s, std::size_t& p) {
    skip_ws(s, p);
    if (p >= s.size()) throw std::runtime_error("json: unexpected end of input");
    const char c = s[p];
    if (c == '{') {
      ++p;
      json j = object();
      skip_ws(s, p);
      if (p < s.size() && s[p] == '}') {
        ++p;
        return j;
      }
      for (;;) {
        std::string k = parse_string(s, p);
        expect(s, p, ':');
        j.o_[k] = parse_value(s, p);
        skip_ws(s, p);
        if (p < s.size() && s[p] == ',') {
          ++p;
          continue;
        }
        expect(s, p, '}');
        return j;
      }
    }
    if (c == '[') {
      ++p;
      json j = array();
      skip_ws(s, p);
      if (p < s.size() && s[p] == ']') {
        ++p;
        return j;
      }
      for (;;) {
        j.a_.push_back(parse_value(s, p));
        skip_ws(s, p);
        if (p < s.size() && s[p] == ',') {
          ++p;
          continue;
        }
        expect(s, p, ']');
        return j;
      }
    }
    if (c == '"') return json(parse_string(s, p));
    if (s.compare(p, 4, "true") == 0) {
      p += 4;
      return json(true);
    }
    if (s.compare(p, 5, "false") == 0) {
      p += 5;
      return json(false);
    }
    if (s.compare(p, 4, "null") == 0) {
      p += 4;
      return json();
    }
    std::size_t e = p;
    bool is_float = false;
    while (e < s.size() && (std::isdigit(static_cast<unsigned char>(s[e])) || s[e] == '-' || s[e] == '+' ||
                            s[e] == '.' || s[e] == 'e' || s[e] == 'E')) {
      is_float = is_float || s[e] == '.' || s[e] == 'e' || s[e] == 'E';
      ++e;
    }
    if (e == p) throw std::runtime_error("json: unexpected character");
    const std::string tok = s.substr(p, e - p);
    p = e;
    if (is_float) return json(std::strtod(tok.c_str(), nullptr));
    return json(static_cast<std::int64_t>(std::strtoll(tok.c_str(), nullptr, 10)));
  }

  Type t_ = Type::Null;
  bool b_ = false;
  std::int64_t i_ = 0;
  double f_ = 0.0;
  std::string s_;
  array_t a_;
  object_t o_;
};

}  // namespace nlohmann
