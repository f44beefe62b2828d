// rxg_set_option: process-wide tuning / test switches (see options.hpp).
#include "options.hpp"

#include <deque>
#include <map>
#include <mutex>
#include <string>

#include "rxg.h"

namespace {

std::mutex g_mu;
std::map<std::string, const char*> g_values;
std::deque<std::string> g_store;   // append-only: returned pointers stay valid

}  // namespace

namespace rxg {

const char* option(const char* name) {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_values.find(name);
    return it == g_values.end() ? nullptr : it->second;
}

}  // namespace rxg

extern "C" int rxg_set_option(const char* name, const char* value) {
    if (!name || !*name) return RXG_EINVAL;
    std::lock_guard<std::mutex> lk(g_mu);
    if (!value || !*value) {
        g_values.erase(name);
    } else {
        g_store.emplace_back(value);
        g_values[name] = g_store.back().c_str();
    }
    return RXG_OK;
}
