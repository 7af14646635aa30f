// main() of the reference unit tests built against the Catch2 stand-in.
#include <catch2/catch_amalgamated.hpp>

int main(int argc, char** argv) { return catch_shim::run(argc, argv); }
