/* Plain-C consumer of include/relay.h (no torch, no CUDA headers): compiled
 * and run by tests/test_abi.py on the CPU host to prove the boundary is a
 * self-contained C ABI.  Exercises host-side validation and the host-only
 * relay_stats_finalize on a hand-built table (global margins {0.25, 0.75} and
 * one cue window of mean 0.6). */
#include <math.h>
#include <stdio.h>
#include <string.h>

#include "relay.h"

int main(void) {
  if (relay_version() != RELAY_VERSION) return 1;
  /* vocab < 2 is rejected before any device work */
  if (relay_margin_rows((const void*)16, RELAY_DT_BF16, 4, 1, 1, 1.0f, (float*)16, NULL, NULL, NULL,
                        NULL, NULL) != RELAY_ERR_INVALID)
    return 2;
  if (strstr(relay_last_error(), "vocab") == NULL) return 3;
  uint64_t tab[2][RELAY_STAT_FIELDS + 1];
  memset(tab, 0, sizeof tab);
  const uint64_t Q = 1u << 20;
  tab[1][RELAY_F_N] = 2;
  tab[1][RELAY_F_SUM_MQ] = Q / 4 + 3 * Q / 4;
  tab[1][RELAY_F_SUM_MQ2] = (Q / 4) * (Q / 4) + (3 * Q / 4) * (3 * Q / 4);
  tab[1][RELAY_F_SUM_LEN] = 2;
  tab[0][RELAY_F_N] = 1;
  tab[0][RELAY_F_SUM_MQ] = (uint64_t)(0.6 * Q);
  tab[0][RELAY_F_SUM_MQ2] = tab[0][RELAY_F_SUM_MQ] * tab[0][RELAY_F_SUM_MQ];
  tab[0][RELAY_F_SUM_LEN] = 1;
  relay_cue_summary_t out[2];
  if (relay_stats_finalize(&tab[0][0], 1, 1, 1, 2, out) != RELAY_OK) return 4;
  if (fabs(out[1].mean - 0.5) > 1e-12 || fabs(out[1].std - 0.25) > 1e-12) return 5;
  if (out[0].selected != 1) return 6;            /* rule 2: 0.6 > 0.5 */
  if (relay_stats_finalize(&tab[0][0], 1, 1, 1, 0, out) != RELAY_OK) return 7;
  if (out[0].selected != 0) return 8;            /* rule 0: 0.6 < 0.5 + 0.1768 */
  printf("c abi ok\n");
  return 0;
}
