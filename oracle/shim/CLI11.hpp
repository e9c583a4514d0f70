// Test-infrastructure shim: the subset of CLI11 (https://github.com/CLIUtils/CLI11,
// version unpinned by the reference) that the reference's benchmark CLI
// (proj/tools/bench_main.cpp) uses -- App::add_option / add_flag on --long
// names, Option::required / check, CLI::IsMember and CLI11_PARSE.  Written
// for this repository (the reference's vendor/ directory is absent); it lets
// the reference's own CLI build so its acceptance criterion 10 can drive it.
#pragma once

#include <initializer_list>
#include <iostream>
#include <memory>
#include <set>
#include <sstream>
#include <stdexcept>
#include <string>
#include <functional>
#include <vector>

namespace CLI {

struct Error : std::runtime_error {
  int code;
  Error(const std::string& m, int c) : std::runtime_error(m), code(c) {}
};

struct Validator {
  std::function<std::string(const std::string&)> fn;  // empty string = valid
};
inline Validator IsMember(std::initializer_list<std::string> values) {
  std::set<std::string> s(values);
  return Validator{[s](const std::string& v) { return s.count(v) ? std::string() : "value " + v + " not in set"; }};
}

class Option {
 public:
  Option(std::string name, std::function<void(const std::string&)> set, bool flag)
      : name_(std::move(name)), set_(std::move(set)), flag_(flag) {}
  Option* required(bool r = true) {
    required_ = r;
    return this;
  }
  Option* check(Validator v) {
    checks_.push_back(std::move(v));
    return this;
  }
  const std::string& name() const { return name_; }
  bool flag() const { return flag_; }
  bool is_required() const { return required_; }
  void apply(const std::string& v) {
    for (const auto& c : checks_) {
      const std::string e = c.fn(v);
      if (!e.empty()) throw Error(name_ + ": " + e, 105);
    }
    set_(v);
    seen_ = true;
  }
  bool seen() const { return seen_; }

 private:
  std::string name_;
  std::function<void(const std::string&)> set_;
  bool flag_ = false, required_ = false, seen_ = false;
  std::vector<Validator> checks_;
};

class App {
 public:
  explicit App(std::string description = "") : desc_(std::move(description)) {}
  template <typename T>
  Option* add_option(const std::string& name, T& target, const std::string& = "") {
    opts_.push_back(std::make_unique<Option>(
        name,
        [&target, name](const std::string& v) {
          std::istringstream is(v);
          T tmp{};
          if constexpr (std::is_same_v<T, std::string>) {
            tmp = v;
          } else if (!(is >> tmp) || !is.eof()) {
            throw Error(name + ": cannot parse '" + v + "'", 106);
          }
          target = tmp;
        },
        false));
    return opts_.back().get();
  }
  Option* add_flag(const std::string& name, bool& target, const std::string& = "") {
    opts_.push_back(std::make_unique<Option>(name, [&target](const std::string&) { target = true; }, true));
    return opts_.back().get();
  }
  void parse(int argc, char** argv) {
    for (int i = 1; i < argc; ++i) {
      std::string a = argv[i], val;
      bool has_val = false;
      const auto eq = a.find('=');
      if (eq != std::string::npos) {
        val = a.substr(eq + 1);
        a = a.substr(0, eq);
        has_val = true;
      }
      if (a == "-h" || a == "--help") throw Error(desc_, 0);
      Option* o = find(a);
      if (!o) throw Error("unknown argument " + a, 109);
      if (o->flag()) {
        o->apply("1");
        continue;
      }
      if (!has_val) {
        if (i + 1 >= argc) throw Error(a + " needs a value", 107);
        val = argv[++i];
      }
      o->apply(val);
    }
    for (const auto& o : opts_)
      if (o->is_required() && !o->seen()) throw Error(o->name() + " is required", 106);
  }
  int exit(const Error& e) const {
    (e.code ? std::cerr : std::cout) << e.what() << "\n";
    return e.code;
  }

 private:
  Option* find(const std::string& a) {
    for (const auto& o : opts_)
      if (o->name() == a) return o.get();
    return nullptr;
  }
  std::string desc_;
  std::vector<std::unique_ptr<Option>> opts_;
};

}  // namespace CLI

#define CLI11_PARSE(app, argc, argv) \
  try {                              \
    (app).parse((argc), (argv));     \
  } catch (const CLI::Error& e) {    \
    return (app).exit(e);            \
  }
