// tbsim/csr_cache.hpp -- extension of the drop-in API (no reference
// counterpart): NDJSON DAG files (src/dagio.cpp:86-138) compiled once into
// the binary CSR cache of include/tbsim_b200.h (tbsim_batch_desc_save /
// tbsim_hostbatch_load), so a sweep over file DAGs uploads packed CSR
// sections instead of re-parsing JSON on every run.
#pragma once

#include <string>
#include <vector>

namespace tbsim {

// Loads each file with load_dag_file (the reference's parsing, validation
// and exceptions) and writes all graphs, in order, as one cache file.
void compile_dag_cache(const std::vector<std::string>& dag_files, const std::string& cache_path);

}  // namespace tbsim
