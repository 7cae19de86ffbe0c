// main() of the reference unit suites re-run against the B200 drop-in
// (proj/tests/test_main.cpp does the same with the real doctest).
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include <doctest.h>
