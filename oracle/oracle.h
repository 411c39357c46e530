/*
 * oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's scheduling hot path
 * (/root/reference/proj/src/{taskgraph,attributes,platform,policies,engine,
 * generators}.cpp).  It is the CHECKER the B200 product is compared against:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load it.  Parity of this restatement is pinned against the reference
 * itself (oracle/_ref, tests/test_oracle_pins.py) and against the golden
 * fixtures the reference produced (tests/golden/, tests/golden/make_golden.py).
 *
 * Same batch layout and output structs as the product C-ABI
 * (include/tbsim_b200.h) so every implementation sees identical bytes.
 */
#ifndef TBSIM_ORACLE_H
#define TBSIM_ORACLE_H

#include "tbsim_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

const char* orc_last_error(void);

int orc_attributes(const tbsim_batch_desc* b, const tbsim_costs* costs, int request,
                   int priority_kind, tbsim_attr_out* out);

int orc_simulate(const tbsim_batch_desc* b, const tbsim_platform_desc* platforms,
                 const int32_t* platform_of, int policy, const tbsim_regulator_cfg* reg,
                 const tbsim_attr_in* attrs, tbsim_sim_out* out);

/* default_regulator_config for graph g of the batch on a platform. */
int orc_default_regulator_config(const tbsim_batch_desc* b, int64_t g,
                                 const tbsim_platform_desc* p, tbsim_regulator_cfg* out);

/* Host rules (policies.cpp:153-203). */
double orc_calculate_k(const double* t, const int64_t* v, int n);
void orc_regulator_step(tbsim_regulator_state* st, const tbsim_regulator_cfg* cfg,
                        int64_t cur_nready, double now_ms);

/* Generators (generators.cpp).  Output arrays are malloc'ed; free with
 * orc_free.  Layout: single graph CSR (dep_off[n+1], dep, in_off[n+1], in,
 * out_off[n+1], out, type[n], handle_bytes[nh]); type ids follow the
 * canonical table of paper_2404_03226_b200/platform.py TYPE_NAMES. */
typedef struct orc_graph {
    int32_t n, n_dep, n_in, n_out, n_handles;
    int32_t *dep_off, *dep, *in_off, *in, *out_off, *out, *type;
    int64_t* handle_bytes;
} orc_graph;

int orc_gen_layered(int32_t n_tasks, int32_t n_layers, double edge_prob, uint64_t seed,
                    orc_graph* out);
int orc_gen_cholesky(int32_t nblocks, int64_t block_bytes, orc_graph* out);
int orc_gen_lu(int32_t nblocks, int64_t block_bytes, orc_graph* out);
void orc_graph_free(orc_graph* g);

#ifdef __cplusplus
}
#endif
#endif
