// main() of the shimmed reference unit-test binary
#include "catch2/catch_amalgamated.hpp"
int main() { return catch_shim::run_all(); }
