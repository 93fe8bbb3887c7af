#pragma once
// Flat parameter map (reference: proj/include/synq/params.hpp).  The built-in
// defaults equal configs/model_defaults.cfg so the shipped configs run
// unchanged.
#include <map>
#include <string>

namespace synq {

using param_set = std::map<std::string, double>;

param_set builtin_defaults();
void merge_params_file(param_set& base, const std::string& path);  // later wins
void merge_param_kv(param_set& base, const std::string& kv);       // "key=value"
double param(const param_set& ps, const std::string& key);         // throws if missing

}  // namespace synq
