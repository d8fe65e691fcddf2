// CLI11_lite: the handful of CLI11 calls the reference's tools/synth_main.cc
// makes (App, add_option/add_flag, required, delimiter, check(IsMember),
// CLI11_PARSE). Test infrastructure only: it exists so oracle/_ref can build
// the reference CLI unmodified; the product CLI has its own parser.
#ifndef CLI11_LITE_HPP_
#define CLI11_LITE_HPP_

#include <cstdint>
#include <cstdlib>
#include <functional>
#include <iostream>
#include <memory>
#include <set>
#include <sstream>
#include <string>
#include <vector>

namespace CLI {

struct IsMember {
  std::set<std::string> allowed;
  IsMember(std::initializer_list<std::string> items) : allowed(items) {}
};

class Option {
 public:
  Option(std::string name, bool is_flag, std::function<bool(const std::string&)> assign)
      : name_(std::move(name)), is_flag_(is_flag), assign_(std::move(assign)) {}
  Option* required() { required_ = true; return this; }
  Option* delimiter(char d) { delimiter_ = d; return this; }
  Option* check(const IsMember& m) { allowed_ = m.allowed; return this; }

  std::string name_;
  bool is_flag_;
  std::function<bool(const std::string&)> assign_;
  bool required_ = false;
  bool seen_ = false;
  char delimiter_ = '\0';
  std::set<std::string> allowed_;
};

namespace detail {
template <typename T>
bool ParseScalar(const std::string& text, T& out) {
  std::istringstream is(text);
  T value{};
  is >> value;
  if (is.fail() || !is.eof()) return false;
  out = value;
  return true;
}
inline bool ParseScalar(const std::string& text, std::string& out) {
  out = text;
  return true;
}
}  // namespace detail

class App {
 public:
  explicit App(std::string description) : description_(std::move(description)) {}

  template <typename T>
  Option* add_option(const std::string& name, T& target, const std::string& = "") {
    auto opt = std::make_unique<Option>(name, false, nullptr);
    Option* raw = opt.get();
    raw->assign_ = [raw, &target](const std::string& text) {
      if (!raw->allowed_.empty() && !raw->allowed_.count(text)) return false;
      return detail::ParseScalar(text, target);
    };
    options_.push_back(std::move(opt));
    return raw;
  }

  template <typename T>
  Option* add_option(const std::string& name, std::vector<T>& target, const std::string& = "") {
    auto opt = std::make_unique<Option>(name, false, nullptr);
    Option* raw = opt.get();
    raw->assign_ = [raw, &target](const std::string& text) {
      std::vector<std::string> pieces;
      if (raw->delimiter_) {
        std::string cur;
        for (char c : text) {
          if (c == raw->delimiter_) { pieces.push_back(cur); cur.clear(); }
          else cur.push_back(c);
        }
        pieces.push_back(cur);
      } else {
        pieces.push_back(text);
      }
      for (auto& p : pieces) {
        T value{};
        if (!detail::ParseScalar(p, value)) return false;
        target.push_back(value);
      }
      return true;
    };
    options_.push_back(std::move(opt));
    return raw;
  }

  Option* add_flag(const std::string& name, bool& target, const std::string& = "") {
    auto opt = std::make_unique<Option>(name, true, [&target](const std::string&) {
      target = true;
      return true;
    });
    Option* raw = opt.get();
    options_.push_back(std::move(opt));
    return raw;
  }

  // Returns 0 on success, otherwise the exit code to use.
  int parse(int argc, char** argv) {
    for (int i = 1; i < argc; ++i) {
      std::string arg = argv[i];
      if (arg == "--help" || arg == "-h") {
        std::cout << description_ << "\n";
        for (auto& o : options_) std::cout << "  " << o->name_ << "\n";
        return -1;
      }
      std::string value;
      bool has_inline = false;
      size_t eq = arg.find('=');
      if (eq != std::string::npos) {
        value = arg.substr(eq + 1);
        arg = arg.substr(0, eq);
        has_inline = true;
      }
      Option* opt = nullptr;
      for (auto& o : options_) if (o->name_ == arg) opt = o.get();
      if (!opt) {
        std::cerr << "The following argument was not expected: " << argv[i] << "\n";
        return 109;
      }
      if (!opt->is_flag_ && !has_inline) {
        if (i + 1 >= argc) {
          std::cerr << arg << ": 1 required argument missing\n";
          return 107;
        }
        value = argv[++i];
      }
      if (!opt->assign_(value)) {
        std::cerr << arg << ": invalid value '" << value << "'\n";
        return 105;
      }
      opt->seen_ = true;
    }
    for (auto& o : options_) {
      if (o->required_ && !o->seen_) {
        std::cerr << o->name_ << " is required\n";
        return 106;
      }
    }
    return 0;
  }

 private:
  std::string description_;
  std::vector<std::unique_ptr<Option>> options_;
};

}  // namespace CLI

#define CLI11_PARSE(app, argc, argv)              \
  do {                                            \
    int cli11_lite_rc = (app).parse((argc), (argv)); \
    if (cli11_lite_rc == -1) return 0;            \
    if (cli11_lite_rc != 0) return cli11_lite_rc; \
  } while (0)

#endif  // CLI11_LITE_HPP_
