// Minimal CLI11-compatible subset, enough to compile the UNMODIFIED reference
// proj/src/cli.cpp into oracle/_ref/trioalign_ref (CLI11 itself is absent
// offline).  TEST INFRASTRUCTURE ONLY.
//
// Semantics mirrored from CLI11 2.x where cli.cpp depends on them:
//  * App::parse(std::vector<std::string>&&) takes the arguments REVERSED;
//  * add_option(name, var, desc) binds var and sets run_callback_for_default,
//    so Option::default_val(v) assigns v to the bound variable immediately;
//  * errors derive from CLI::ParseError (ValidationError, RequiredError,
//    ExtrasError, ConversionError); App::exit(e) prints and returns the
//    exit code (0 for --help).
#pragma once
#include <charconv>
#include <functional>
#include <iostream>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

namespace CLI {

struct Error : std::runtime_error {
  Error(std::string name, const std::string& msg, int code) : std::runtime_error(msg), name_(std::move(name)), code_(code) {}
  int get_exit_code() const { return code_; }
  std::string name_;
  int code_;
};
struct ParseError : Error {
  ParseError(std::string name, const std::string& msg, int code = 2) : Error(std::move(name), msg, code) {}
};
struct ValidationError : ParseError {
  ValidationError(std::string name, const std::string& msg) : ParseError(std::move(name), name + ": " + msg, 105) {}
};
struct CallForHelp : ParseError {
  CallForHelp() : ParseError("CallForHelp", "This should be caught in your main function, see examples", 0) {}
};

class App;

class Option {
 public:
  Option(std::string name, std::function<void(const std::string&)> set, bool flag)
      : name_(std::move(name)), set_(std::move(set)), flag_(flag) {}
  Option* required(bool v = true) {
    required_ = v;
    return this;
  }
  template <class T>
  Option* default_val(const T& v) {
    // run_callback_for_default: the bound variable takes the default now
    set_(std::to_string(v));
    return this;
  }
  std::string name_;
  std::function<void(const std::string&)> set_;
  bool flag_ = false;
  bool required_ = false;
  bool seen_ = false;
};

class App {
 public:
  explicit App(std::string desc = "", std::string name = "") : desc_(std::move(desc)), name_(std::move(name)) {}

  App* require_subcommand(int n) {
    require_ = n;
    return this;
  }
  App* add_subcommand(const std::string& name, const std::string& desc) {
    subs_.push_back(std::make_unique<App>(desc, name));
    return subs_.back().get();
  }
  template <class T>
  Option* add_option(const std::string& name, T& var, const std::string& = "") {
    auto set = [&var, name](const std::string& v) {
      if constexpr (std::is_same_v<T, std::string>) {
        var = v;
      } else {
        T x{};
        const auto [p, ec] = std::from_chars(v.data(), v.data() + v.size(), x);
        if (ec != std::errc{} || p != v.data() + v.size())
          throw ParseError("ConversionError", "Could not convert: " + name + " = " + v, 101);
        var = x;
      }
    };
    opts_.push_back(std::make_unique<Option>(name, set, false));
    return opts_.back().get();
  }
  Option* add_flag(const std::string& name, bool& var, const std::string& = "") {
    opts_.push_back(std::make_unique<Option>(name, [&var](const std::string&) { var = true; }, true));
    return opts_.back().get();
  }
  bool parsed() const { return parsed_; }

  void parse(std::vector<std::string>&& rev) {
    std::vector<std::string> args(rev.rbegin(), rev.rend());
    size_t pos = 0;
    if (pos < args.size() && (args[pos] == "--help" || args[pos] == "-h")) throw CallForHelp();
    App* sub = nullptr;
    if (pos < args.size()) {
      for (auto& s : subs_)
        if (s->name_ == args[pos]) sub = s.get();
    }
    if (!sub) {
      if (require_ > 0 && args.empty()) throw ParseError("RequiredError", "A subcommand is required", 106);
      throw ParseError("ExtrasError", "The following arguments were not expected: " + (args.empty() ? std::string() : args[0]), 109);
    }
    ++pos;
    while (pos < args.size()) {
      std::string a = args[pos++];
      if (a == "--help" || a == "-h") throw CallForHelp();
      std::string value;
      bool has_value = false;
      const size_t eq = a.find('=');
      if (a.rfind("--", 0) == 0 && eq != std::string::npos) {
        value = a.substr(eq + 1);
        a = a.substr(0, eq);
        has_value = true;
      }
      Option* o = nullptr;
      for (auto& x : sub->opts_)
        if (x->name_ == a) o = x.get();
      if (!o) throw ParseError("ExtrasError", "The following arguments were not expected: " + a, 109);
      if (o->flag_) {
        o->set_("");
      } else {
        if (!has_value) {
          if (pos >= args.size()) throw ParseError("ArgumentMismatch", a + ": 1 required", 110);
          value = args[pos++];
        }
        o->set_(value);
      }
      o->seen_ = true;
    }
    for (auto& x : sub->opts_)
      if (x->required_ && !x->seen_) throw ParseError("RequiredError", x->name_ + " is required", 106);
    sub->parsed_ = true;
    parsed_ = true;
  }

  int exit(const Error& e) const {
    if (e.get_exit_code() == 0) {
      std::cout << desc_ << "\n";
      return 0;
    }
    std::cerr << e.what() << "\nRun with --help for more information.\n";
    return e.get_exit_code();
  }

 private:
  std::string desc_, name_;
  int require_ = 0;
  bool parsed_ = false;
  std::vector<std::unique_ptr<App>> subs_;
  std::vector<std::unique_ptr<Option>> opts_;
};

}  // namespace CLI
