// gtest_lite: a minimal GoogleTest-compatible harness (TEST, TEST_F,
// EXPECT_*/ASSERT_* with streamed messages, ::testing::Test::HasFailure,
// TempDir, PrintToString, --gtest_filter). Test infrastructure only: it lets
// the reference's own suites (/root/reference/proj/tests/*.cc) be compiled
// unmodified, both against the reference sources (oracle/_ref) and against
// this repository's planner library, so the two can be compared test by test.
#ifndef GTEST_LITE_GTEST_H_
#define GTEST_LITE_GTEST_H_

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <iostream>
#include <sstream>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

namespace testing {

class Message {
 public:
  Message() = default;
  Message(const Message& other) { ss_ << other.ss_.str(); }
  template <typename T>
  Message& operator<<(const T& value) {
    if constexpr (std::is_pointer_v<T> && !std::is_same_v<std::decay_t<T>, const char*> &&
                  !std::is_same_v<std::decay_t<T>, char*>) {
      ss_ << static_cast<const void*>(value);
    } else {
      ss_ << value;
    }
    return *this;
  }
  Message& operator<<(std::ostream& (*manip)(std::ostream&)) {
    ss_ << manip;
    return *this;
  }
  std::string str() const { return ss_.str(); }

 private:
  std::stringstream ss_;
};

namespace internal {

template <typename T, typename = void>
struct Streamable : std::false_type {};
template <typename T>
struct Streamable<T, std::void_t<decltype(std::declval<std::ostream&>() << std::declval<const T&>())>>
    : std::true_type {};

template <typename T, typename = void>
struct Iterable : std::false_type {};
template <typename T>
struct Iterable<T, std::void_t<decltype(std::begin(std::declval<const T&>())),
                               decltype(std::end(std::declval<const T&>()))>> : std::true_type {};

template <typename T>
void PrintTo(const T& value, std::ostream& os) {
  if constexpr (std::is_same_v<T, std::string>) {
    os << '"' << value << '"';
  } else if constexpr (Streamable<T>::value) {
    os << value;
  } else if constexpr (Iterable<T>::value) {
    os << "{ ";
    bool first = true;
    for (const auto& item : value) {
      if (!first) os << ", ";
      first = false;
      PrintTo(item, os);
    }
    os << " }";
  } else {
    os << "<" << sizeof(T) << "-byte object>";
  }
}

struct State {
  bool current_failed = false;
  int failures = 0;
};
inline State& state() {
  static State s;
  return s;
}

class Reporter {
 public:
  Reporter(const char* file, int line, std::string text)
      : file_(file), line_(line), text_(std::move(text)) {}
  void operator=(const Message& message) const {
    state().current_failed = true;
    ++state().failures;
    std::cout << file_ << ":" << line_ << ": Failure\n" << text_;
    std::string extra = message.str();
    if (!extra.empty()) std::cout << "\n" << extra;
    std::cout << std::endl;
  }

 private:
  const char* file_;
  int line_;
  std::string text_;
};

template <typename A, typename B, typename Op>
bool Compare(const A& a, const B& b, Op op, const char* ea, const char* eb, const char* opname,
             std::string* detail) {
  if (op(a, b)) return true;
  std::ostringstream os;
  os << "Expected: (" << ea << ") " << opname << " (" << eb << "), actual: ";
  PrintTo(a, os);
  os << " vs ";
  PrintTo(b, os);
  *detail = os.str();
  return false;
}

inline bool Near(double a, double b, double tol, const char* ea, const char* eb, std::string* detail) {
  if (std::fabs(a - b) <= tol) return true;
  std::ostringstream os;
  os.precision(17);
  os << "The difference between " << ea << " and " << eb << " is " << std::fabs(a - b)
     << ", which exceeds " << tol << " (" << a << " vs " << b << ")";
  *detail = os.str();
  return false;
}

struct TestEntry {
  std::string suite;
  std::string name;
  std::function<void()> run;
};
inline std::vector<TestEntry>& registry() {
  static std::vector<TestEntry> r;
  return r;
}
inline int Register(const char* suite, const char* name, std::function<void()> run) {
  registry().push_back({suite, name, std::move(run)});
  return 0;
}

inline bool GlobMatch(const char* pattern, const char* text) {
  if (*pattern == '\0') return *text == '\0';
  if (*pattern == '*') return GlobMatch(pattern + 1, text) || (*text && GlobMatch(pattern, text + 1));
  if (*text == '\0') return false;
  if (*pattern == '?' || *pattern == *text) return GlobMatch(pattern + 1, text + 1);
  return false;
}

inline bool AnyMatch(const std::string& patterns, const std::string& full) {
  size_t start = 0;
  while (start <= patterns.size()) {
    size_t end = patterns.find(':', start);
    std::string p = patterns.substr(start, end == std::string::npos ? std::string::npos : end - start);
    if (!p.empty() && GlobMatch(p.c_str(), full.c_str())) return true;
    if (end == std::string::npos) break;
    start = end + 1;
  }
  return false;
}

inline bool Selected(const std::string& filter, const std::string& full) {
  if (filter.empty()) return true;
  std::string positive = filter, negative;
  size_t dash = filter.find('-');
  if (dash != std::string::npos) {
    positive = filter.substr(0, dash);
    negative = filter.substr(dash + 1);
  }
  if (positive.empty()) positive = "*";
  return AnyMatch(positive, full) && !(negative.size() && AnyMatch(negative, full));
}

}  // namespace internal

class Test {
 public:
  virtual ~Test() = default;
  virtual void SetUp() {}
  virtual void TearDown() {}
  virtual void TestBody() = 0;
  static bool HasFailure() { return internal::state().current_failed; }
};

inline std::string TempDir() {
  const char* env = std::getenv("TEST_TMPDIR");
  std::string dir = env ? env : "/tmp";
  if (dir.empty() || dir.back() != '/') dir += '/';
  return dir;
}

template <typename T>
std::string PrintToString(const T& value) {
  std::ostringstream os;
  internal::PrintTo(value, os);
  return os.str();
}

inline void InitGoogleTest(int*, char**) {}

inline int RunAllTests(int argc, char** argv) {
  std::string filter;
  if (const char* env = std::getenv("GTEST_FILTER")) filter = env;
  for (int i = 1; i < argc; ++i) {
    std::string arg = argv[i];
    if (arg.rfind("--gtest_filter=", 0) == 0) filter = arg.substr(15);
  }
  int ran = 0, failed = 0;
  std::vector<std::string> failed_names;
  for (auto& test : internal::registry()) {
    std::string full = test.suite + "." + test.name;
    if (!internal::Selected(filter, full)) continue;
    internal::state().current_failed = false;
    std::cout << "[ RUN      ] " << full << std::endl;
    test.run();
    ++ran;
    if (internal::state().current_failed) {
      ++failed;
      failed_names.push_back(full);
      std::cout << "[  FAILED  ] " << full << std::endl;
    } else {
      std::cout << "[       OK ] " << full << std::endl;
    }
  }
  std::cout << "[==========] " << ran << " tests ran. [  PASSED  ] " << (ran - failed) << " tests."
            << std::endl;
  for (auto& name : failed_names) std::cout << "[  FAILED  ] " << name << std::endl;
  return failed == 0 ? 0 : 1;
}

}  // namespace testing

#define RUN_ALL_TESTS() ::testing::RunAllTests(0, nullptr)

#define GTEST_LITE_CLASS_(suite, name) suite##_##name##_Test

#define GTEST_LITE_DEFINE_(suite, name, parent)                                          \
  class GTEST_LITE_CLASS_(suite, name) : public parent {                                  \
   public:                                                                                \
    void TestBody() override;                                                             \
  };                                                                                      \
  [[maybe_unused]] static int gtest_lite_reg_##suite##_##name = ::testing::internal::Register( \
      #suite, #name, [] {                                                                 \
        GTEST_LITE_CLASS_(suite, name) t;                                                 \
        t.SetUp();                                                                        \
        t.TestBody();                                                                     \
        t.TearDown();                                                                     \
      });                                                                                 \
  void GTEST_LITE_CLASS_(suite, name)::TestBody()

#define TEST(suite, name) GTEST_LITE_DEFINE_(suite, name, ::testing::Test)
#define TEST_F(fixture, name) GTEST_LITE_DEFINE_(fixture, name, fixture)

#define GTEST_LITE_NONFATAL_(cond, text) \
  if (std::string gtest_lite_detail_; (cond)) \
    ;                                        \
  else                                       \
    ::testing::internal::Reporter(__FILE__, __LINE__, text) = ::testing::Message()

#define GTEST_LITE_FATAL_(cond, text)         \
  if (std::string gtest_lite_detail_; (cond)) \
    ;                                         \
  else                                        \
    return ::testing::internal::Reporter(__FILE__, __LINE__, text) = ::testing::Message()

#define GTEST_LITE_CMP_(a, b, op)                                                       \
  ::testing::internal::Compare(                                                         \
      (a), (b), [](const auto& x, const auto& y) { return static_cast<bool>(x op y); }, \
      #a, #b, #op, &gtest_lite_detail_)

#define EXPECT_TRUE(c) GTEST_LITE_NONFATAL_(static_cast<bool>(c), "Value of: " #c "\n  Actual: false\nExpected: true")
#define EXPECT_FALSE(c) GTEST_LITE_NONFATAL_(!static_cast<bool>(c), "Value of: " #c "\n  Actual: true\nExpected: false")
#define ASSERT_TRUE(c) GTEST_LITE_FATAL_(static_cast<bool>(c), "Value of: " #c "\n  Actual: false\nExpected: true")
#define ASSERT_FALSE(c) GTEST_LITE_FATAL_(!static_cast<bool>(c), "Value of: " #c "\n  Actual: true\nExpected: false")

#define EXPECT_EQ(a, b) GTEST_LITE_NONFATAL_(GTEST_LITE_CMP_(a, b, ==), gtest_lite_detail_)
#define EXPECT_NE(a, b) GTEST_LITE_NONFATAL_(GTEST_LITE_CMP_(a, b, !=), gtest_lite_detail_)
#define EXPECT_LT(a, b) GTEST_LITE_NONFATAL_(GTEST_LITE_CMP_(a, b, <), gtest_lite_detail_)
#define EXPECT_LE(a, b) GTEST_LITE_NONFATAL_(GTEST_LITE_CMP_(a, b, <=), gtest_lite_detail_)
#define EXPECT_GT(a, b) GTEST_LITE_NONFATAL_(GTEST_LITE_CMP_(a, b, >), gtest_lite_detail_)
#define EXPECT_GE(a, b) GTEST_LITE_NONFATAL_(GTEST_LITE_CMP_(a, b, >=), gtest_lite_detail_)
#define ASSERT_EQ(a, b) GTEST_LITE_FATAL_(GTEST_LITE_CMP_(a, b, ==), gtest_lite_detail_)
#define ASSERT_NE(a, b) GTEST_LITE_FATAL_(GTEST_LITE_CMP_(a, b, !=), gtest_lite_detail_)
#define ASSERT_LT(a, b) GTEST_LITE_FATAL_(GTEST_LITE_CMP_(a, b, <), gtest_lite_detail_)
#define ASSERT_LE(a, b) GTEST_LITE_FATAL_(GTEST_LITE_CMP_(a, b, <=), gtest_lite_detail_)
#define ASSERT_GT(a, b) GTEST_LITE_FATAL_(GTEST_LITE_CMP_(a, b, >), gtest_lite_detail_)
#define ASSERT_GE(a, b) GTEST_LITE_FATAL_(GTEST_LITE_CMP_(a, b, >=), gtest_lite_detail_)

#define EXPECT_NEAR(a, b, tol) \
  GTEST_LITE_NONFATAL_(::testing::internal::Near((a), (b), (tol), #a, #b, &gtest_lite_detail_), gtest_lite_detail_)
#define ASSERT_NEAR(a, b, tol) \
  GTEST_LITE_FATAL_(::testing::internal::Near((a), (b), (tol), #a, #b, &gtest_lite_detail_), gtest_lite_detail_)

#endif  // GTEST_LITE_GTEST_H_
