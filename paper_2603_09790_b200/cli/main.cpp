// main.cpp -- the `chebstep` binary (reference src/main.cpp role): forwards
// to chebstep::cli::run in libchebstep_gpu.so.
#include "chebstep/cli.hpp"

int main(int argc, char** argv) { return chebstep::cli::run(argc, argv); }
