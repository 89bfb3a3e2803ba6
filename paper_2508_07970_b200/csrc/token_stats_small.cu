// token_stats_small.cu — A1 compiled a second time with the
// ring shape that suits small vocabularies: 4,096-element tiles x 4 stages,
// 3 CTAs per SM.  Shorter rows spend a larger share of their time in the
// row-end combine; a third resident CTA keeps HBM busy meanwhile.  Exported
// as token_stats_ring_small; token_stats_launch (token_stats.cu) dispatches
// by vocabulary (V <= 60,000 here; numbers in token_stats.cu).
#ifndef YATT_A1_SMALL_TILE
#define YATT_A1_SMALL_TILE 4096
#endif
#ifndef YATT_A1_SMALL_STAGES
#define YATT_A1_SMALL_STAGES 4
#endif
#ifndef YATT_A1_SMALL_MINB
#define YATT_A1_SMALL_MINB 3
#endif
#define YATT_A1_SMALL_TU 1
#undef YATT_A1_TILE
#undef YATT_A1_STAGES
#undef YATT_A1_MINB
#include "token_stats.cu"
