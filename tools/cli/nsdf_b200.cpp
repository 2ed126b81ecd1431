// `nsdf_b200 train|render|bench ...`: the reference CLI's flows (proj/tools/nsdf_main.cpp) on
// the B200 build — a main() around nsdf_host_cli (paper_2201_09147_b200/host/cli.cpp).
#include "nsdf_host.h"

int main(int argc, char** argv) { return nsdf_host_cli(argc, argv); }
