/* A plain C consumer of the C-ABI (include/cortex_b200.h): no C++, no torch.
 * Known answer (test_synapse.cpp:199-204 "tie"): four points on a line with
 * uniform attention; the reference picks rows {0, 3} for k = 2, lambda = 1
 * (coverage only: the first pick is the farthest from the centroid, ties to the
 * lowest row, the second the farthest from the first). */
#include <stdio.h>
#include <stdint.h>
#include "cortex_b200.h"

int main(void) {
    const float cloud[4 * 2] = {0.f, 0.f, 1.f, 0.f, 2.f, 0.f, 3.f, 0.f};
    const double attn[4] = {0.25, 0.25, 0.25, 0.25};
    int64_t idx[2] = {-1, -1};
    double scores[2] = {0.0, 0.0};
    int64_t n = 0;
    cx_status st = cx_select_landmarks_points(cloud, 4, 2, attn, 4, 2, 1.0, idx, scores, &n);
    if (st != CX_OK) {
        printf("status %d: %s\n", (int)st, cx_last_error());
        return 2;
    }
    printf("n=%lld idx=%lld,%lld scores=%.17g,%.17g\n", (long long)n, (long long)idx[0], (long long)idx[1], scores[0],
           scores[1]);
    /* error categories cross the boundary as status codes: k < 1 is a config_error */
    if (cx_select_landmarks_points(cloud, 4, 2, attn, 4, 0, 1.0, idx, scores, &n) != CX_CONFIG_ERROR) return 3;
    return (n == 2 && idx[0] == 0 && idx[1] == 3) ? 0 : 1;
}
