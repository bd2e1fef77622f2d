// main() of the shim-based test binaries (reference doctest_main.cpp equivalent).
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include "doctest.h"
