// Instances for variant=full, dtype=f16 (see kinst.inc).
#define IQ_VAR 0
#define IQ_T __half
#define IQ_FN launch_full_f16
#include "kinst.inc"
