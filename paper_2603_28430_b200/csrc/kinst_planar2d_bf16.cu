// Instances for variant=planar2d, dtype=bf16 (see kinst.inc).
#define IQ_VAR 2
#define IQ_T __nv_bfloat16
#define IQ_FN launch_planar2d_bf16
#include "kinst.inc"
