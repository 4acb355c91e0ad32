// Instances for variant=planar2d, dtype=f32 (see kinst.inc).
#define IQ_VAR 2
#define IQ_T float
#define IQ_FN launch_planar2d_f32
#include "kinst.inc"
