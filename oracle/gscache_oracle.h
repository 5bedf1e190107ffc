/* oracle/gscache_oracle.h -- types shared by the oracle's own C files (test infrastructure
 * only; nothing under paper_2507_19718_b200/ includes it). */
#ifndef GSCACHE_ORACLE_H_
#define GSCACHE_ORACLE_H_

/* Activated Gaussian of one raw parameter row (C1). */
typedef struct {
  double mu[3], qhat[4], qnorm, R[3][3], D[3], A[3][3], w, chat[3], v[3];
  int degenerate;
} orc_gauss;

void orc_activate_row(const double* p, orc_gauss* g);

#endif
