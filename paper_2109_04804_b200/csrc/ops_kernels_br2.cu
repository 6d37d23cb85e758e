// ops_kernels_br2.cu -- the Navier-Stokes element operators with BR2 face gradients
// (reading R33) on GLL nodes: a compile-time instantiation, so that the BR1
// kernels carry no BR2 branch.
#define HBPDC_OPS_BR2 1
#include "ops_kernels.cu"
