// token_stats_fused_small.cu — the fused training-side loss + gradient kernel
// (token_stats.cu) compiled a second time for small
// vocabularies: 8,192-element tiles x 4 policy stages at 3 CTAs per SM.  With
// short rows the two row-end barriers around the fp64 epilogue are a larger
// share of a row; a third resident CTA keeps the SM busy meanwhile, and the
// rows live between the two passes stay far inside L2.  Exported as
// policy_loss_grad_ring_small; policy_loss_grad_launch dispatches by
// vocabulary (V <= 60,000 here).
#define YATT_FUSED_ONLY_TU 1
#define YATT_FUSED_SMALL_TU 1
#undef YATT_A1_TILE
#undef YATT_A1_STAGES
#undef YATT_A1_MINB
#define YATT_A1_TILE 8192
#define YATT_A1_STAGES 2
#define YATT_A1_MINB 3
#undef YATT_FUSED_CW
#define YATT_FUSED_CW 8
#include "token_stats.cu"
