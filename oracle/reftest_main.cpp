// TEST INFRASTRUCTURE ONLY: main() for the reference's doctest files compiled
// against the B200 library (see oracle/doctest_shim/doctest.h).
#include <doctest.h>

int main() { return doctest::detail::run_all(); }
