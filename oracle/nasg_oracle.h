/* TEST INFRASTRUCTURE ONLY — CPU restatement of the NASG guiding hot path.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * reference legs may load this.  It is the checker, never the product.
 * Parity status: PINNED — tests/test_oracle.py checks every entry point
 * bit-for-bit (or to 1e-12 where libm calls differ) against the unmodified
 * reference compiled in oracle/_ref/, and against the SPEC.md known-answer
 * examples; tests/golden/ holds fixtures generated from oracle/_ref.
 *
 * Array conventions match oracle/ref_capi.cpp (see there).
 */
#ifndef NASG_ORACLE_H
#define NASG_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_MAX_LOBES 32
#define ORC_IN 64
#define ORC_HIDDEN 128

uint64_t orc_hash_mix(uint64_t x);
uint64_t orc_hash_combine(uint64_t a, uint64_t b);
void orc_pcg32(uint64_t initstate, uint64_t initseq, int n, uint32_t *out);

void orc_init_network(uint64_t seed, int out_dim, float *w_out);
void orc_init_network_hu(uint64_t seed, int hidden, int out_dim, float *w_out);
void orc_one_blob(double x, int k, float *out);
uint64_t orc_encode(int64_t n, const float *q9, const float *bmin, const float *bmax,
                    float *out64);

void orc_forward(const float *w, int out_dim, int64_t n, const float *in64, float *out);
void orc_backward(const float *w, int out_dim, int64_t n, const float *in64,
                  const float *out_grads, float *dw);
int orc_adam_step(int out_dim, float *w, float *m, float *v, const float *g, int64_t *t,
                  float lr);

double orc_norm_const(double lambda, double a, double eps);
int orc_frame_from_euler(double ct, double sp, double cp, double st, double ctau,
                         double *xyz9);
double orc_nasg_log_eval(const double *c12, const double *v);
void orc_nasg_sample(const double *c12, double xi0, double xi1, double xi2, double *out);

void orc_decode(int64_t nq, int n_comp, const float *raw, double *out);
void orc_decode_sample(int64_t nq, int n_comp, const float *raw, const float *xi,
                       double *out4, double *c_out, int nthreads);
void orc_decode_pdf(int64_t nq, int n_comp, const float *raw, const float *dir3, double b,
                    const float *bsdf_pdf, double *mix_out, double *guided_out);
void orc_query_sample(const float *w, int out_dim, int64_t nq, const float *q9,
                      const float *xi, const float *bmin, const float *bmax, float *out4,
                      float *c_out, int nthreads);
void orc_kl_grad(int64_t n, int n_comp, const float *raw, const float *samples, double b,
                 double loss_blend, double *grad_out, int *ok_out, double *loss_out);

void orc_dist_pdf(int kind, int64_t n, int k, const float *comp, const float *w, const float *dir4, double *out);
void orc_dist_sample(int kind, int64_t n, int k, const float *comp, const float *w, const float *xi4, double *out4);
void orc_dist_grad(int kind, int64_t n, int k, const float *comp, const float *w, const float *dir4, double *out);
void orc_vmf_fit_grad(int k, const float *raw, int64_t n, const float *samples4, double *grad_out, int *ok_out);

double orc_stride_update(double l, uint64_t s, uint64_t cap);
double orc_blend_coefficient(int64_t i, int m, int bsteps);

void *orc_trainer_create(int n_comp, int capacity, int batch, int step_factor, float lr,
                         double loss_blend, uint64_t seed, const float *bmin,
                         const float *bmax);
void orc_trainer_destroy(void *t);
void orc_trainer_train(void *t, int64_t n, const float *samples, double b, double *stats4);
void orc_trainer_get_weights(void *t, float *w);
void orc_trainer_set_weights(void *t, const float *w);

void orc_set_reverse_sum(int on);
int orc_save_checkpoint(const char *path, const float *w, int out_dim, int n_comp);
int orc_load_checkpoint(const char *path, float *w, int max_floats, int *n_comp);

/* synthetic workloads: byte-identical to nasg_synth_queries / nasg_synth_samples */
void orc_synth_queries(uint64_t seed, int64_t first, int64_t n, const float *bmin, const float *bmax, float *x,
                       float *wo, float *nrm, float *xi);
void orc_synth_samples(uint64_t seed, int64_t first, int64_t n, const float *bmin, const float *bmax, float *out16);

#ifdef __cplusplus
}
#endif
#endif
