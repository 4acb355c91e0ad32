// Instances for variant=full, dtype=f32 (see kinst.inc).
#define IQ_VAR 0
#define IQ_T float
#define IQ_FN launch_full_f32
#include "kinst.inc"
