// Runner TU for the reference's unmodified Catch2 tests compiled against the
// drop-in headers (tests/cpp/Makefile target ref_tests).
#define ABQ_CATCH_MAIN
#include <catch2/catch_amalgamated.hpp>
