// Test shim (NOT product code): the subset of the CLI11 command-line API that the reference's
// tools/rotavote_cli.cpp uses, written from scratch because the vendored CLI11 is absent from
// /root/reference (vendor/ is git-ignored there). Lets the reference CLI, unmodified, build against
// this repo's drop-in headers for the end-to-end CLI test (tests/test_cli_gpu.py).
// Supported: App with subcommands, add_option (scalars, strings, vectors; "--long,-s" names),
// add_flag with "!--negation", ->required(), ->check(IsMember{...}), require_subcommand, operator
// bool on a subcommand, CLI11_PARSE.
#pragma once

#include <cstdint>
#include <functional>
#include <initializer_list>
#include <iostream>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

namespace CLI {

struct ParseError : std::runtime_error {
  int code;
  ParseError(const std::string& m, int c = 106) : std::runtime_error(m), code(c) {}
};

struct IsMember {
  std::vector<std::string> allowed;
  IsMember(std::initializer_list<std::string> a) : allowed(a) {}
};

namespace detail {
template <typename T>
void convert(const std::string& s, T& out) {
  if constexpr (std::is_same_v<T, std::string>) {
    out = s;
  } else if constexpr (std::is_same_v<T, bool>) {
    out = !(s == "0" || s == "false");
  } else {
    std::istringstream in(s);
    T v{};
    if (!(in >> v) || !in.eof()) throw ParseError("invalid value '" + s + "'");
    out = v;
  }
}
}  // namespace detail

class Option {
 public:
  Option(std::vector<std::string> names, bool multi, std::function<void(const std::vector<std::string>&)> set)
      : names_(std::move(names)), multi_(multi), set_(std::move(set)) {}
  Option* required() {
    required_ = true;
    return this;
  }
  Option* check(const IsMember& m) {
    allowed_ = m.allowed;
    return this;
  }
  bool matches(const std::string& a) const {
    for (const auto& n : names_)
      if (n == a) return true;
    return false;
  }
  const std::string& name() const { return names_.front(); }
  void apply(const std::vector<std::string>& vals) {
    if (!allowed_.empty())
      for (const auto& v : vals) {
        bool ok = false;
        for (const auto& a : allowed_) ok = ok || a == v;
        if (!ok) throw ParseError(name() + ": value '" + v + "' not in the allowed set");
      }
    set_(vals);
    seen_ = true;
  }
  bool multi() const { return multi_; }
  bool flag = false;
  bool negated = false;
  bool seen_ = false;
  bool required_ = false;

 private:
  std::vector<std::string> names_;
  bool multi_;
  std::function<void(const std::vector<std::string>&)> set_;
  std::vector<std::string> allowed_;
};

class App {
 public:
  explicit App(std::string description = "", std::string name = "") : desc_(std::move(description)), name_(std::move(name)) {}

  App* add_subcommand(const std::string& name, const std::string& description = "") {
    subs_.push_back(std::make_unique<App>(description, name));
    return subs_.back().get();
  }
  void require_subcommand(int n) { require_sub_ = n; }
  explicit operator bool() const { return parsed_; }

  template <typename T>
  Option* add_option(const std::string& names, T& var, const std::string& = "") {
    std::vector<std::string> ns = split(names);
    if constexpr (is_vector<T>::value) {
      opts_.push_back(std::make_unique<Option>(ns, true, [&var](const std::vector<std::string>& v) {
        var.clear();
        for (const auto& s : v) {
          typename T::value_type x{};
          detail::convert(s, x);
          var.push_back(x);
        }
      }));
    } else {
      opts_.push_back(std::make_unique<Option>(ns, false, [&var](const std::vector<std::string>& v) {
        detail::convert(v.back(), var);
      }));
    }
    return opts_.back().get();
  }

  template <typename T>
  Option* add_flag(const std::string& names, T& var, const std::string& = "") {
    std::vector<std::string> pos, neg;
    for (const auto& n : split(names)) (n.size() > 1 && n[0] == '!' ? neg : pos).push_back(n[0] == '!' ? n.substr(1) : n);
    auto make = [&](std::vector<std::string> ns, bool value) {
      opts_.push_back(std::make_unique<Option>(ns, false, [&var, value](const std::vector<std::string>&) {
        var = static_cast<T>(value);
      }));
      opts_.back()->flag = true;
    };
    if (!neg.empty()) make(neg, false);
    make(pos, true);
    return opts_.back().get();
  }

  void parse(int argc, char** argv) {
    std::vector<std::string> args(argv + 1, argv + argc);
    parse_args(args, 0);
  }

  int exit(const ParseError& e) const {
    std::cerr << (name_.empty() ? "" : name_ + ": ") << e.what() << "\n";
    return e.code;
  }

 private:
  template <typename T>
  struct is_vector : std::false_type {};
  template <typename T>
  struct is_vector<std::vector<T>> : std::true_type {};

  static std::vector<std::string> split(const std::string& names) {
    std::vector<std::string> out;
    std::string cur;
    for (char ch : names) {
      if (ch == ',') {
        if (!cur.empty()) out.push_back(cur);
        cur.clear();
      } else {
        cur += ch;
      }
    }
    if (!cur.empty()) out.push_back(cur);
    return out;
  }

  static bool looks_like_option(const std::string& a) {
    return a.size() > 1 && a[0] == '-' && !(a[1] >= '0' && a[1] <= '9') && a[1] != '.';
  }

  void parse_args(const std::vector<std::string>& args, size_t i) {
    parsed_ = true;
    while (i < args.size()) {
      const std::string& a = args[i];
      App* sub = nullptr;
      for (auto& s : subs_)
        if (s->name_ == a) sub = s.get();
      if (sub) {
        sub->parse_args(args, i + 1);
        ++subs_parsed_;
        i = args.size();
        break;
      }
      std::string key = a, inline_val;
      const auto eq = a.find('=');
      if (looks_like_option(a) && eq != std::string::npos) {
        key = a.substr(0, eq);
        inline_val = a.substr(eq + 1);
      }
      Option* opt = nullptr;
      for (auto& o : opts_)
        if (o->matches(key)) opt = o.get();
      if (!opt) throw ParseError("unknown argument '" + a + "'", 109);
      ++i;
      if (opt->flag) {
        opt->apply({});
        continue;
      }
      std::vector<std::string> vals;
      if (eq != std::string::npos && looks_like_option(a)) vals.push_back(inline_val);
      while (i < args.size() && !looks_like_option(args[i]) && (opt->multi() || vals.empty())) {
        bool is_sub = false;
        for (auto& s : subs_) is_sub = is_sub || s->name_ == args[i];
        if (is_sub) break;
        vals.push_back(args[i++]);
      }
      if (vals.empty()) throw ParseError(key + " needs a value", 108);
      opt->apply(vals);
    }
    for (auto& o : opts_)
      if (o->required_ && !o->seen_) throw ParseError(o->name() + " is required", 106);
    if (require_sub_ > 0 && subs_parsed_ < require_sub_) throw ParseError("a subcommand is required", 106);
  }

  std::string desc_, name_;
  std::vector<std::unique_ptr<App>> subs_;
  std::vector<std::unique_ptr<Option>> opts_;
  int require_sub_ = 0, subs_parsed_ = 0;
  bool parsed_ = false;
};

}  // namespace CLI

#define CLI11_PARSE(app, argc, argv)       \
  try {                                    \
    (app).parse((argc), (argv));           \
  } catch (const CLI::ParseError& e) {     \
    return (app).exit(e);                  \
  }
