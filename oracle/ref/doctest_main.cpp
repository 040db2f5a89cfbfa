// TEST-ONLY: main for the reference's own unit tests compiled against the shims.
#include <doctest.h>
int main() { return doctest::run_all(); }
