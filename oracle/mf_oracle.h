/* mf_oracle.h -- CPU restatement of the reference path (TEST INFRASTRUCTURE ONLY).
 * See mf_oracle.c for the reference file:line each function follows. */
#ifndef MF_ORACLE_H
#define MF_ORACLE_H
#include <stdint.h>

#define MFO_INFEASIBLE 4

typedef struct mfo_result {
    int64_t n_in, n_out, m_out, c;
    double *positions;
    int64_t *facets;
    double *features;
    int64_t *replace;
    int64_t *mapping;
} mfo_result;

int64_t mfo_round_targets(int64_t n_in, int64_t target, int64_t rounds, int64_t *chain, int64_t cap);
int mfo_decimate_mesh(const double *P, int64_t n, const int64_t *F, int64_t m, const double *X, int64_t c,
                      const int64_t *chain, int64_t nchain, int seeded, const uint64_t pcg[4], int order,
                      int placement, mfo_result **res_out, int64_t *achievable);
void mfo_result_sizes(const mfo_result *r, int64_t *n_in, int64_t *n_out, int64_t *m_out, int64_t *c);
void mfo_result_copy(const mfo_result *r, double *positions, int64_t *facets, double *features, int64_t *replace,
                     int64_t *mapping);
void mfo_result_free(mfo_result *r);
void mfo_vertex_quadrics(const double *P, int64_t n, const int64_t *F, int64_t m, int order, double *Q13);
int mfo_quality_errors(const double *P, int64_t n, const int64_t *F, int64_t m, const int64_t *replace,
                       int64_t n_out, const double *Pout, int order, double *errors);
int64_t mfo_edge_costs(const double *P, int64_t n, const int64_t *F, int64_t m, int order, int64_t *edges_out,
                       double *cost_out);
void mfo_pcg64_random(const uint64_t pcg[4], int64_t n, double *out);
int mfo_pool_f64(const double *X, int64_t n, int64_t c, const int64_t *replace, int64_t n_out, int mode,
                 const double *w, double *out);
int mfo_pool_f32(const float *X, int64_t n, int64_t c, const int64_t *replace, int64_t n_out, int mode,
                 const float *w, float *out);
#endif
