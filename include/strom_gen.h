/*
 * strom_gen.h -- C-ABI of the fast relaxation generator (libstrom_gen.so; NEXT-3 of
 * SURVEY.md §8(f), the paper's STROM converter).
 *
 * Compiles a chain-sparse POP (Definition 1) into the kappa-th order
 * sparse moment relaxation as the standard multi-block SDP min <C,X> s.t. A(X) = b,
 * X in Omega_+ (PAPER.md:244-416): blocks clique-major (moment matrix M_k, then the
 * localizing matrices L_{k,i}), rows clique-major and family-minor (normalisation, A_mom,
 * A_ineq, A_eq, A_sen), A in CSR over svec columns (SDPT3 svec). The output
 * equals strom_inputs.relax.compile_relaxation byte for byte (tests/test_generator.py).
 * This is the input side: it holds none of the sGS-ADMM arithmetic.
 *
 * Ownership: inputs are read during the call only; the result is owned by the library
 * until strom_gen_free. Errors: strom_gen_compile returns 0 on success, -1 bad arguments,
 * -2 a clique with more than 21 variables, -3 a constraint degree above 2 kappa, -4 a
 * monomial outside the clique's moment matrix.
 */
#ifndef STROM_GEN_H
#define STROM_GEN_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* One clique: nvars ordered local variables with global ids vars[nvars] (consensus rows
 * pair equal ids of consecutive cliques). Polynomials as term lists: exponent rows
 * [nterms][nvars] (uint8) and coefficients [nterms], in the caller's term order (the order
 * of the floating-point sums). g (inequalities g >= 0) and h (equalities h = 0) are
 * concatenated: g_nterms[ng] terms each. Constraint polynomials are taken as given (the
 * max-|coef| normalisation of reading Q12 is the caller's). */
typedef struct {
  int32_t nvars;
  const int32_t *vars;
  int32_t f_nterms; const uint8_t *f_exp; const double *f_coef;
  int32_t ng; const int32_t *g_nterms; const uint8_t *g_exp; const double *g_coef;
  int32_t nh; const int32_t *h_nterms; const uint8_t *h_exp; const double *h_coef;
} strom_gen_clique;

typedef struct strom_gen_result strom_gen_result;

int32_t strom_gen_compile(int32_t ncliques, const strom_gen_clique *cliques, int32_t kappa,
                          strom_gen_result **out);
void strom_gen_sizes(const strom_gen_result *r, int32_t *nblocks, int64_t *n, int64_t *m, int64_t *nnz);
/* Copies into caller arrays: block_n, block_stage, block_kind [nblocks], block_offset
 * [nblocks + 1], indptr [m + 1], indices, data [nnz], b [m], C [n], row_family, row_stage [m]. */
void strom_gen_copy(const strom_gen_result *r, int32_t *block_n, int32_t *block_stage, int8_t *block_kind,
                    int64_t *block_offset, int64_t *indptr, int32_t *indices, double *data, double *b,
                    double *C, int8_t *row_family, int32_t *row_stage);
void strom_gen_free(strom_gen_result *r);

#ifdef __cplusplus
}
#endif
#endif /* STROM_GEN_H */
