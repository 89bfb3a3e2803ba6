// token_stats_fused_mid.cu — the fused training-side loss + gradient kernel
// (token_stats.cu) in its 2-CTA/SM shape (8 consumer warps,
// 6 policy stages of 16 KB = 3 two-tensor stages), used for the
// full-vocabulary KL at V <= 60,000: the 3-CTA/SM small shape would spill
// there and the 1-CTA/SM large shape hides the row-end barriers poorly on
// short rows.  Exported as policy_loss_grad_ring_mid.
#define YATT_FUSED_ONLY_TU 1
#define YATT_FUSED_MID_TU 1
#undef YATT_A1_TILE
#undef YATT_A1_STAGES
#undef YATT_A1_MINB
#undef YATT_FUSED_CW
#define YATT_A1_TILE 8192
#define YATT_A1_STAGES 3
#define YATT_A1_MINB 2
#define YATT_FUSED_CW 8
#include "token_stats.cu"
