// Minimal CLI11-compatible argument parser (TEST INFRASTRUCTURE, oracle side).
//
// Supplies only what /root/reference/proj/tools/muxsim.cpp:12-41 uses, because
// CLI11 is not vendored with the reference (.gitignore:2): App{desc},
// require_subcommand(1), add_subcommand(name, desc), add_option("-s,--long",
// std::string&, desc)->required(), parse(argc, argv) throwing ParseError,
// exit(e) (0 for --help, 1 otherwise) and App::parsed(). Independent code.
#pragma once

#include <cstdio>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace CLI {

class ParseError : public std::runtime_error {
 public:
  ParseError(const std::string& what, int code) : std::runtime_error(what), code_(code) {}
  int code() const { return code_; }

 private:
  int code_;
};

class Option {
 public:
  Option(std::string names, std::string* target) : target_(target) {
    size_t start = 0;
    while (start <= names.size()) {
      size_t comma = names.find(',', start);
      std::string n = names.substr(start, comma == std::string::npos ? std::string::npos
                                                                     : comma - start);
      if (!n.empty()) names_.push_back(n);
      if (comma == std::string::npos) break;
      start = comma + 1;
    }
  }
  Option* required() {
    required_ = true;
    return this;
  }
  bool matches(const std::string& arg) const {
    for (const std::string& n : names_)
      if (n == arg) return true;
    return false;
  }
  const std::string& first_name() const { return names_.front(); }

  std::vector<std::string> names_;
  std::string* target_;
  bool required_ = false;
  bool seen_ = false;
};

class App {
 public:
  explicit App(std::string desc = {}, std::string name = {})
      : desc_(std::move(desc)), name_(std::move(name)) {}

  void require_subcommand(int n) { required_subcommands_ = n; }

  App* add_subcommand(const std::string& name, const std::string& desc) {
    subs_.push_back(std::make_unique<App>(desc, name));
    return subs_.back().get();
  }

  Option* add_option(const std::string& names, std::string& target, const std::string&) {
    opts_.push_back(std::make_unique<Option>(names, &target));
    return opts_.back().get();
  }

  bool parsed() const { return parsed_; }

  void parse(int argc, char** argv) {
    std::vector<std::string> args(argv + 1, argv + argc);
    parse_args(args, 0);
  }

  int exit(const ParseError& e) const {
    if (e.code() == 0) {
      std::printf("%s\n", desc_.c_str());
      for (const auto& s : subs_) std::printf("  %s  %s\n", s->name_.c_str(), s->desc_.c_str());
      return 0;
    }
    std::fprintf(stderr, "%s\n", e.what());
    return e.code();
  }

 private:
  void parse_args(const std::vector<std::string>& args, size_t i) {
    parsed_ = true;
    for (; i < args.size(); ++i) {
      const std::string& a = args[i];
      if (a == "-h" || a == "--help") throw ParseError("help", 0);
      bool handled = false;
      for (auto& o : opts_) {
        std::string value;
        bool inline_value = false;
        size_t eq = a.find('=');
        if (eq != std::string::npos && a.rfind("--", 0) == 0 && o->matches(a.substr(0, eq))) {
          value = a.substr(eq + 1);
          inline_value = true;
        } else if (!o->matches(a)) {
          continue;
        }
        if (!inline_value) {
          if (i + 1 >= args.size()) throw ParseError(a + " requires an argument", 1);
          value = args[++i];
        }
        *o->target_ = value;
        o->seen_ = true;
        handled = true;
        break;
      }
      if (handled) continue;
      for (auto& s : subs_) {
        if (s->name_ == a) {
          s->parse_args(args, i + 1);
          check_required();
          return;
        }
      }
      throw ParseError("unexpected argument: " + a, 1);
    }
    check_required();
    if (required_subcommands_ > 0) throw ParseError("a subcommand is required", 1);
  }

  void check_required() const {
    for (const auto& o : opts_)
      if (o->required_ && !o->seen_) throw ParseError(o->first_name() + " is required", 1);
  }

  std::string desc_, name_;
  int required_subcommands_ = 0;
  bool parsed_ = false;
  std::vector<std::unique_ptr<Option>> opts_;
  std::vector<std::unique_ptr<App>> subs_;
};

}  // namespace CLI
