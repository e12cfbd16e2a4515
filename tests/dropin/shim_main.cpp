// main() of the Catch2 shim (test infrastructure).
#define SHIM_DEFINE_MAIN
#include "catch_amalgamated.hpp"
