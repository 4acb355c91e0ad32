// Instances for variant=fast, dtype=f32 (see kinst.inc).
#define IQ_VAR 1
#define IQ_T float
#define IQ_FN launch_fast_f32
#include "kinst.inc"
