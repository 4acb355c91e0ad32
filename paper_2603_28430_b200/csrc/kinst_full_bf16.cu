// Instances for variant=full, dtype=bf16 (see kinst.inc).
#define IQ_VAR 0
#define IQ_T __nv_bfloat16
#define IQ_FN launch_full_bf16
#include "kinst.inc"
