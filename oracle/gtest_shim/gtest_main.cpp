// main() for binaries built from several shimmed test files.
#define GTEST_SHIM_NO_MAIN
#include "gtest/gtest.h"
int main() { return ::testing::RunAllTests(); }
