// select128.cu -- the greedy selection kernel of select64.cu instantiated for
// d = 128: the reference-mode cloud of a 2-head MHA cache (d_model = 2 x 64,
// select_landmarks, synapse.cpp:286-320).  No register rows: every row of a
// CTA is a shared-memory row (fp32, or the fp16 sketch with exact rows from L2).
#define SEL_D 128
#include "select64.cu"
