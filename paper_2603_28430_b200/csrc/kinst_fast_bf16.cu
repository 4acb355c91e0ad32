// Instances for variant=fast, dtype=bf16 (see kinst.inc).
#define IQ_VAR 1
#define IQ_T __nv_bfloat16
#define IQ_FN launch_fast_bf16
#include "kinst.inc"
