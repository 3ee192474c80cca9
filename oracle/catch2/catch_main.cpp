// TEST INFRASTRUCTURE ONLY: the shim harness main() for the reference suites
#define CATCH_SHIM_MAIN
#include <catch2/catch_amalgamated.hpp>
