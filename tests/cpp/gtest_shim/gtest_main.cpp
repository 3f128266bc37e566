// main() of the reference-test binaries built against the drop-in headers.
#include "gtest/gtest.h"

int main() { return ::testing::RunAllTests(); }
