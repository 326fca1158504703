// abi.cu -- error reporting and version entry points of libsaix_b200.so
// (status codes + thread-local message; the Python layer maps them to the
// reference's exception types, e.g. SequenceError, sequence.py:152-156).
#include <cstdarg>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"

namespace saix {

static thread_local char g_last_error[512] = "";

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
    va_end(ap);
}

struct ProfRec {
    const char *name;
    double bytes;
    cudaEvent_t a, b;
};
static std::mutex g_prof_mu;
static bool g_prof = false;
static std::vector<ProfRec> g_recs;
static std::vector<size_t> g_open;
static std::vector<cudaEvent_t> g_pool;

static cudaEvent_t prof_event() {
    if (!g_pool.empty()) {
        cudaEvent_t e = g_pool.back();
        g_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

bool prof_on() { return g_prof; }

void prof_mark(const char *name, double bytes, cudaStream_t st, bool begin) {
    std::lock_guard<std::mutex> g(g_prof_mu);
    if (begin) {
        ProfRec r{name, bytes, prof_event(), prof_event()};
        cudaEventRecord(r.a, st);
        g_recs.push_back(r);
        g_open.push_back(g_recs.size() - 1);
    } else if (!g_open.empty()) {
        cudaEventRecord(g_recs[g_open.back()].b, st);
        g_open.pop_back();
    }
}

static void prof_clear() {
    for (auto &r : g_recs) {
        g_pool.push_back(r.a);
        g_pool.push_back(r.b);
    }
    g_recs.clear();
    g_open.clear();
}

}  // namespace saix

extern "C" void saix_prof_enable(int on) {
    std::lock_guard<std::mutex> g(saix::g_prof_mu);
    saix::prof_clear();
    saix::g_prof = on != 0;
}

extern "C" int saix_prof_collect(saix_prof_entry *out, int max_entries) {
    using namespace saix;
    std::lock_guard<std::mutex> g(g_prof_mu);
    std::map<std::string, saix_prof_entry> agg;
    std::vector<std::string> order;
    for (auto &r : g_recs) {
        cudaEventSynchronize(r.b);
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, r.a, r.b) != cudaSuccess) continue;
        auto it = agg.find(r.name);
        if (it == agg.end()) {
            saix_prof_entry e;
            memset(&e, 0, sizeof(e));
            strncpy(e.name, r.name, sizeof(e.name) - 1);
            it = agg.emplace(r.name, e).first;
            order.push_back(r.name);
        }
        it->second.launches += 1;
        it->second.total_ms += ms;
        it->second.bytes += r.bytes;
    }
    prof_clear();
    int n = 0;
    for (auto &k : order) {
        if (n < max_entries && out) out[n] = agg[k];
        n++;
    }
    return n;
}

extern "C" const char *saix_last_error(void) { return saix::g_last_error; }

extern "C" int saix_abi_version(void) { return 1; }
