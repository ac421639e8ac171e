// Launch plan, step a-2 of SURVEY §8a: "choose variant and tile ... from a
// compiled-in per-pattern table (the paper's 'presets')" -- PAPER.md:735
// (presets for its patterns) and PAPER.md:1206-1208 (parameters auto-tuned per
// pattern and per GPU architecture).
//
// Each kernel family exposes its measured design alternatives as KsKnob bits
// (ks_internal.h).  ks_presets.inc is GENERATED (scripts/gen_presets.py) from an
// offline autotune on a B200 (scripts/autotune.py, profiles/r02/autotune.json):
// for every configs[2] sweep pattern and every configs[3]/[4] factor, per
// layout, math and batch bucket floor(log2 B), the knob set that measured
// fastest (kept only when it beat the rules by more than the noise margin).
// Lookup order: the handle's ks_set_knobs override, the table, the rules.
// Setting any experiment environment switch (KS_TF32_V2, KS_V2_NKB,
// KS_TF32_DENSIFY, KS_BSFJ_J8, KS_BSFJ_BN256, KS_FFMA_KB32, KS_FFMA_WS,
// KS_FFMA_WSG) bypasses the table so A/B runs see the rules they change.
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>

#include "ks_internal.h"

namespace {

struct KsPreset {
    int32_t a, b, c, d;
    int8_t layout, math, lg_batch;
    uint32_t knobs;
};

const KsPreset kPresets[] = {
#include "ks_presets.inc"
    {0, 0, 0, 0, 0, 0, 0, 0},   // sentinel (never matches: a >= 1)
};

using Key = std::tuple<int64_t, int64_t, int64_t, int64_t, int, int, int>;

const std::map<Key, uint32_t>& table() {
    static const std::map<Key, uint32_t> t = [] {
        std::map<Key, uint32_t> m;
        for (const KsPreset& p : kPresets)
            if (p.a >= 1) m[Key{p.a, p.b, p.c, p.d, p.layout, p.math, p.lg_batch}] = p.knobs;
        return m;
    }();
    return t;
}

int lg_batch(int64_t B) {
    int l = 0;
    while (B > 1) {
        B >>= 1;
        ++l;
    }
    return l;
}

// Process-wide experiment switches: -1 unset, else the value.
int env_switch(const char* name) {
    const char* e = getenv(name);
    return e ? atoi(e) : -1;
}

struct EnvKnobs {
    uint32_t set = 0, clear = 0;
    bool any = false;
};

const EnvKnobs& env_knobs() {
    static const EnvKnobs k = [] {
        EnvKnobs r;
        auto put = [&](bool on, uint32_t bit) {
            (on ? r.set : r.clear) |= bit;
            r.any = true;
        };
        int v;
        if ((v = env_switch("KS_TF32_V2")) >= 0) put(v == 1, KS_KNOB_TF32_V2);
        if ((v = env_switch("KS_V2_NKB")) >= 0) put(v == 2, KS_KNOB_V2_NKB2);
        if ((v = env_switch("KS_TF32_DENSIFY")) >= 0 && v != 1) put(v == 2, KS_KNOB_DENSIFY);
        if ((v = env_switch("KS_BSFJ_J8")) >= 0) put(v == 1, KS_KNOB_J8);
        if ((v = env_switch("KS_BSFJ_BN256")) >= 0) put(v != 0, KS_KNOB_BN256);
        if ((v = env_switch("KS_FFMA_KB32")) >= 0) put(v != 0, KS_KNOB_KB32);
        if ((v = env_switch("KS_FFMA_WS")) >= 0) put(v != 0, KS_KNOB_FFMA_WS);
        if ((v = env_switch("KS_FFMA_WSG")) >= 0) put(v != 0, KS_KNOB_FFMA_WSG);
        if ((v = env_switch("KS_TF32_MN")) >= 0) put(v != 0, KS_KNOB_TF32_MN);
        if ((v = env_switch("KS_FFMA_WSL")) >= 0) put(v != 0, KS_KNOB_FFMA_WSL);
        return r;
    }();
    return k;
}

}  // namespace

namespace ks {

// The hand-written rules (round 1 measurements), used where the
// table has no entry.
uint32_t rule_knobs(const ks_handle_s& h, const KsCall& call) {
    (void)call;
    uint32_t k = KS_KNOB_BN256 | KS_KNOB_KB32 | KS_KNOB_FFMA_WS | KS_KNOB_FFMA_WSG;
    // densified super-blocks: a single super-block with d in {2, 3, 6}, or d = 8 with
    // small blocks, measured 1.1-1.4x faster (profiles/r02/exp_tf32_densify.txt)
    if (h.a == 1 && (h.d == 2 || h.d == 3 || h.d == 6 || (h.d == 8 && h.b * h.c <= 48 * 48)))
        k |= KS_KNOB_DENSIFY;
    // MN-major A for TF32 BSL inputs: 1.04-1.21x on every b = 48 sweep pattern, 0.89-1.0x
    // on b >= 64 (profiles/r02/mn_time.jsonl); the preset table refines it per pattern
    if (h.b <= 48) k |= KS_KNOB_TF32_MN;
    const EnvKnobs& e = env_knobs();
    return (k | e.set) & ~e.clear;
}

uint32_t plan_knobs(const ks_handle_s& h, const KsCall& call, int* source) {
    if (h.knobs_override >= 0) {
        if (source) *source = 2;
        return (uint32_t)h.knobs_override;
    }
    if (!env_knobs().any) {
        const auto& t = table();
        auto it = t.find(Key{h.a, h.b, h.c, h.d, call.layout, (int)h.math, lg_batch(call.B)});
        if (it != t.end()) {
            if (source) *source = 1;
            return it->second;
        }
    }
    if (source) *source = 0;
    return rule_knobs(h, call);
}

int preset_count() { return (int)table().size(); }

}  // namespace ks
