// main() of the relinked reference suites (TEST INFRASTRUCTURE): runs every
// registered test through the minimal harness of gtest/gtest.h.
#include <gtest/gtest.h>

int main(int argc, char** argv) { return testing::RunAllTests(argc, argv); }
