// knobs.cuh -- the one place the library reads its FFG_* environment switches.
//
// The environment is snapshotted ONCE (first use) into a table; every tuning value, test hook and
// diagnostic switch is then a table lookup, so no call path runs getenv.  ffg_knobs_reload() takes
// a fresh snapshot (tests change switches between calls; a long-lived process does not need it).
// The switches and their defaults are listed in DESIGN.md ("Tuning knobs").
#pragma once
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>

extern "C" char** environ;

namespace ffg {

struct KnobTable {
    std::unordered_map<std::string, std::string> kv;
};

inline std::atomic<const KnobTable*>& knob_table_slot() {
    static std::atomic<const KnobTable*> slot{nullptr};
    return slot;
}

inline const KnobTable* knobs_snapshot() {
    auto* t = new KnobTable;
    for (char** e = environ; e && *e; ++e) {
        if (strncmp(*e, "FFG_", 4) != 0) continue;
        const char* eq = strchr(*e, '=');
        if (!eq) continue;
        t->kv.emplace(std::string(*e, (size_t)(eq - *e)), std::string(eq + 1));
    }
    return t;
}

// A superseded table stays allocated: callers may still hold pointers into it.
inline void knobs_reload() { knob_table_slot().store(knobs_snapshot(), std::memory_order_release); }

inline const char* knob_str(const char* name) {  // the switch's value, nullptr when unset
    const KnobTable* t = knob_table_slot().load(std::memory_order_acquire);
    if (!t) {
        static std::mutex mu;
        std::lock_guard<std::mutex> lk(mu);
        t = knob_table_slot().load(std::memory_order_acquire);
        if (!t) {
            t = knobs_snapshot();
            knob_table_slot().store(t, std::memory_order_release);
        }
    }
    if (t->kv.empty()) return nullptr;
    const auto it = t->kv.find(name);
    return it == t->kv.end() ? nullptr : it->second.c_str();
}
inline bool knob_set(const char* name) { return knob_str(name) != nullptr; }
inline bool knob_on(const char* name) {  // set and nonzero
    const char* s = knob_str(name);
    return s && atoi(s) != 0;
}
inline long long knob_int(const char* name, long long dflt) {
    const char* s = knob_str(name);
    return s ? atoll(s) : dflt;
}
inline double knob_num(const char* name, double dflt) {
    const char* s = knob_str(name);
    return s ? atof(s) : dflt;
}

}  // namespace ffg
