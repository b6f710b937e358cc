// Translation unit of the clustered forward kernel (several CTAs per batch element, DESIGN.md
// "few large problems").  It is compiled separately from dnls.cu so that its instantiation does not
// change the inlining of the shared device phases in the one-CTA kernel.
#define DNLS_CLUSTER_TU
#include "dnls.cu"
