// csr_cache.cpp -- tbsim::compile_dag_cache (tbsim/csr_cache.hpp).
#include "tbsim/csr_cache.hpp"

#include "device.hpp"
#include "tbsim/taskgraph.hpp"

namespace tbsim {

void compile_dag_cache(const std::vector<std::string>& dag_files, const std::string& cache_path) {
    device::Csr csr;
    for (const auto& f : dag_files) csr.add(load_dag_file(f));
    device::check(tbsim_batch_desc_save(&csr.finish(), cache_path.c_str()));
}

}  // namespace tbsim
