// Instances for variant=fast, dtype=f16 (see kinst.inc).
#define IQ_VAR 1
#define IQ_T __half
#define IQ_FN launch_fast_f16
#include "kinst.inc"
