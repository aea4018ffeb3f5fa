// Entry point of the reference-test binary (oracle/Makefile `reftests`).
#include "doctest.h"

int main(int argc, char** argv) { return doctest::detail::run(argc, argv); }
