// oracle/mini_cli11/CLI11.hpp -- TEST INFRASTRUCTURE ONLY.
//
// The reference CLI (proj/tools/vpip.cpp) parses its arguments with CLI11,
// which the reference tree does not vendor (proj/.gitignore:2 ignores
// vendor/). This is an independent, minimal parser that provides exactly the
// part of that interface vpip.cpp uses -- App, add_subcommand,
// require_subcommand, add_option (string / integer / enum targets) with
// required(), transform(CheckedTransformer(map, ignore_case)) and
// check(IsMember{...}), parse, parsed, exit and ParseError -- so the
// UNMODIFIED CLI can be built against this repository's vpip:: shim and run
// by the reference's own cli_smoke.sh on the B200.
#pragma once

#include <algorithm>
#include <cctype>
#include <charconv>
#include <cstdio>
#include <functional>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

namespace CLI {

class ParseError : public std::runtime_error {
 public:
  explicit ParseError(const std::string& msg, int code = 2) : std::runtime_error(msg), code_(code) {}
  int get_exit_code() const { return code_; }

 private:
  int code_;
};

inline std::string ignore_case(std::string s) {
  for (char& c : s) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
  return s;
}

// transforms (or rejects) an option's text before it is converted
struct Validator {
  std::function<void(std::string&)> fn;
};

template <class Map>
Validator CheckedTransformer(const Map& map, std::string (*filter)(std::string)) {
  std::vector<std::pair<std::string, long long>> table;
  for (const auto& [k, v] : map) table.emplace_back(filter(k), static_cast<long long>(v));
  return {[table, filter](std::string& s) {
    const std::string key = filter(s);
    for (const auto& [k, v] : table)
      if (k == key) {
        s = std::to_string(v);
        return;
      }
    throw ParseError("value '" + s + "' is not one of the allowed names");
  }};
}

inline Validator IsMember(std::vector<std::string> allowed) {
  return {[allowed](std::string& s) {
    if (std::find(allowed.begin(), allowed.end(), s) == allowed.end())
      throw ParseError("value '" + s + "' is not allowed");
  }};
}

class Option {
 public:
  Option(std::string name, std::function<void(const std::string&)> set)
      : name_(std::move(name)), set_(std::move(set)) {}
  Option* required() {
    required_ = true;
    return this;
  }
  Option* transform(Validator v) {
    validators_.push_back(std::move(v));
    return this;
  }
  Option* check(Validator v) { return transform(std::move(v)); }

 private:
  friend class App;
  void apply(std::string text) {
    for (const Validator& v : validators_) v.fn(text);
    set_(text);
    seen_ = true;
  }
  std::string name_;
  std::function<void(const std::string&)> set_;
  std::vector<Validator> validators_;
  bool required_ = false;
  bool seen_ = false;
};

template <class T>
void convert(const std::string& text, T& out, const std::string& name) {
  if constexpr (std::is_same_v<T, std::string>) {
    out = text;
  } else if constexpr (std::is_enum_v<T>) {
    long long v = 0;
    const auto [p, ec] = std::from_chars(text.data(), text.data() + text.size(), v);
    if (ec != std::errc{} || p != text.data() + text.size())
      throw ParseError("option " + name + ": bad value '" + text + "'");
    out = static_cast<T>(v);
  } else {
    T v{};
    const auto [p, ec] = std::from_chars(text.data(), text.data() + text.size(), v);
    if (ec != std::errc{} || p != text.data() + text.size())
      throw ParseError("option " + name + ": could not convert '" + text + "'");
    out = v;
  }
}

class App {
 public:
  explicit App(std::string description = "", std::string name = "")
      : description_(std::move(description)), name_(std::move(name)) {}

  App* add_subcommand(const std::string& name, const std::string& description) {
    subs_.push_back(std::make_unique<App>(description, name));
    return subs_.back().get();
  }
  void require_subcommand(int n) { required_subs_ = n; }

  template <class T>
  Option* add_option(const std::string& name, T& target, const std::string& = "") {
    opts_.push_back(std::make_unique<Option>(
        name, [&target, name](const std::string& text) { convert(text, target, name); }));
    return opts_.back().get();
  }

  bool parsed() const { return parsed_; }

  void parse(int argc, char** argv) {
    std::vector<std::string> args(argv + 1, argv + argc);
    size_t i = 0;
    App* target = this;
    parsed_ = true;
    if (!subs_.empty()) {
      if (args.empty() || args[0].rfind("-", 0) == 0) {
        if (required_subs_ > 0) throw ParseError("a subcommand is required");
      } else {
        target = nullptr;
        for (auto& s : subs_)
          if (s->name_ == args[0]) target = s.get();
        if (!target) throw ParseError("unknown subcommand '" + args[0] + "'");
        target->parsed_ = true;
        i = 1;
      }
    }
    for (; i < args.size(); ++i) {
      std::string key = args[i], value;
      const size_t eq = key.find('=');
      if (eq != std::string::npos) {
        value = key.substr(eq + 1);
        key = key.substr(0, eq);
      } else {
        if (i + 1 >= args.size()) throw ParseError("option " + key + " needs a value");
        value = args[++i];
      }
      Option* opt = nullptr;
      for (auto& o : target->opts_)
        if (o->name_ == key) opt = o.get();
      if (!opt) throw ParseError("unknown argument '" + key + "'");
      opt->apply(value);
    }
    for (auto& o : target->opts_)
      if (o->required_ && !o->seen_) throw ParseError("option " + o->name_ + " is required");
  }

  int exit(const ParseError& e) const {
    std::fprintf(stderr, "%s\n", e.what());
    return e.get_exit_code();
  }

 private:
  std::string description_, name_;
  std::vector<std::unique_ptr<App>> subs_;
  std::vector<std::unique_ptr<Option>> opts_;
  int required_subs_ = 0;
  bool parsed_ = false;
};

}  // namespace CLI
