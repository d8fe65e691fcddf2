// gtest_lite entry point (test infrastructure; see gtest/gtest.h).
#include <gtest/gtest.h>

int main(int argc, char** argv) { return ::testing::RunAllTests(argc, argv); }
