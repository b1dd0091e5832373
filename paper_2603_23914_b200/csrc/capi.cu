// C-ABI plumbing: version, thread-local error message, launch accounting.
#include <atomic>
#include <string>

#include "common.cuh"

namespace kvp {
namespace {
thread_local std::string g_last_error;
std::atomic<uint64_t> g_launches{0};
}  // namespace
void set_last_error(const std::string& m) { g_last_error = m; }
void note_launch(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
}  // namespace kvp

extern "C" int kvp_abi_version(void) { return KVP_ABI_VERSION; }
extern "C" const char* kvp_last_error_message(void) { return kvp::g_last_error.c_str(); }
extern "C" uint64_t kvp_launch_count(void) { return kvp::g_launches.load(); }
