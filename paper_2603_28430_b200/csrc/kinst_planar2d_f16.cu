// Instances for variant=planar2d, dtype=f16 (see kinst.inc).
#define IQ_VAR 2
#define IQ_T __half
#define IQ_FN launch_planar2d_f16
#include "kinst.inc"
