// Experiment switches: compiled into libfasted_exp.so only.
//
// The product library (libfasted.so) is built WITHOUT FASTED_EXPERIMENTS.
// There, the kernel form is a fixed rule of (d_pad, rows, cols) and the
// caller's LOW_OUTPUT / SPARSE hints (all forms give bit-identical records,
// tests/test_gpu.py), nothing reads the environment, and the diagnostic
// flags below do not exist -- results never depend on configuration
// (the reference's own rule, tiling.py:296-297).
//
// libfasted_exp.so (same sources, -DFASTED_EXPERIMENTS) is used by scripts/
// (A/B timing, power and trace experiments) and by the bit-identity tests,
// which force every kernel form through the environment overrides and
// compare the records with the product library's.
#pragma once

#include <stdlib.h>

namespace fasted {

#ifdef FASTED_EXPERIMENTS

// Diagnostic fasted_join flags (results are NOT valid unless stated).
enum {
    FASTED_JOIN_DIAG_NOEPI = 256,      // tcgen05 kernel: skip the epilogue entirely
    FASTED_JOIN_DIAG_NOMMA = 512,      // tcgen05 kernel: skip the MMAs (TMA + epilogue)
    FASTED_JOIN_DIAG_LOADONLY = 1024,  // epilogue: TMEM loads only, no math
    FASTED_JOIN_DIAG_NOSLOW = 2048,    // epilogue: sign test only, never write
    FASTED_JOIN_DIAG_SPIN = 8192,      // accumulator waits spin (no suspend hint)
    FASTED_JOIN_DIAG_LDX64 = 16384,    // epilogue: 32x32b.x64 TMEM loads
    FASTED_JOIN_DIAG_AEVL = 32768,     // CTA pair: A panel loads with L2 evict_last
    FASTED_JOIN_DIAG_TRACE = 65536,    // resident kernel: clock64 timeline of CTA 0 in the
                                       // last 266240 bytes of out_records
    // epilogue hit-search A/B (results stay valid): always per-lane masks /
    // always transposed rows
    FASTED_JOIN_DIAG_RARE_LM = 131072,
    FASTED_JOIN_DIAG_RARE_ROWS = 262144,
    // attribution of the augment step (results NOT valid): skip the
    // kind::tf32 augment MMA / issue it as a kind::f16 MMA instead
    FASTED_JOIN_DIAG_NOAUG = 524288,
    FASTED_JOIN_DIAG_AUGF16 = 1048576,
    // hit-warp attribution (results NOT valid): producers push the entry's
    // metadata only / hit warps consume entries without testing or writing
    FASTED_JOIN_DIAG_HITMETA = 2097152,
    FASTED_JOIN_DIAG_HITSKIP = 4194304,
    // resident kernel: the producer arrives on the B stages' full barriers
    // without loading them (MMA + handshakes alone; results NOT valid)
    FASTED_JOIN_DIAG_NOTMA = 8388608,
    // resident CTA pair: the peer CTA's epilogue warps do not release the
    // accumulator (tempty counts the leader's warps only; results NOT valid)
    FASTED_JOIN_DIAG_NOREMOTE = 16777216,
    // hit warps: candidate rows with <= 3 hits travel as (mask, values)
    // instead of all 32 words (results stay valid; A/B of the packing)
    FASTED_JOIN_DIAG_HITPACK = 33554432,
    // hit warps: queue entries written with generic shared stores and a
    // release arrive on the slot's full barrier instead of st.async +
    // complete_tx (results stay valid; A/B of the hand-off)
    FASTED_JOIN_DIAG_GENERICQ = 67108864,
    // epilogue warps wait for the accumulator by test_wait spin (results valid)
    FASTED_JOIN_DIAG_EPISPIN = 134217728,
    // resident kernel with hit warps: one epilogue warp waits for the
    // accumulator, the other 15 block on a named barrier (results valid)
    FASTED_JOIN_DIAG_EPIBAR = 268435456
};
constexpr int FASTED_JOIN_DIAG_ALL =
    FASTED_JOIN_DIAG_NOEPI | FASTED_JOIN_DIAG_NOMMA | FASTED_JOIN_DIAG_LOADONLY |
    FASTED_JOIN_DIAG_NOSLOW | FASTED_JOIN_DIAG_SPIN | FASTED_JOIN_DIAG_LDX64 |
    FASTED_JOIN_DIAG_AEVL | FASTED_JOIN_DIAG_TRACE | FASTED_JOIN_DIAG_RARE_LM |
    FASTED_JOIN_DIAG_RARE_ROWS | FASTED_JOIN_DIAG_NOAUG | FASTED_JOIN_DIAG_AUGF16 |
    FASTED_JOIN_DIAG_HITMETA | FASTED_JOIN_DIAG_HITSKIP | FASTED_JOIN_DIAG_NOTMA |
    FASTED_JOIN_DIAG_NOREMOTE | FASTED_JOIN_DIAG_HITPACK | FASTED_JOIN_DIAG_GENERICQ |
    FASTED_JOIN_DIAG_EPISPIN | FASTED_JOIN_DIAG_EPIBAR;

inline int env_int(const char* name, int dflt) {
    const char* v = getenv(name);
    return v && *v ? atoi(v) : dflt;
}
// An environment override of a kernel-form or schedule default.
#define FASTED_KNOB(name, dflt) ::fasted::env_int(name, dflt)
// The diagnostic flags of a launch.
#define FASTED_DFLAGS(a) ((a).diag_flags)

#else

constexpr int FASTED_JOIN_DIAG_ALL = 0;
// Product build: every knob is its default, no diagnostic flag is set (the
// compiler removes the diagnostic branches).
#define FASTED_KNOB(name, dflt) (dflt)
#define FASTED_DFLAGS(a) 0
enum {
    FASTED_JOIN_DIAG_NOEPI = 0,
    FASTED_JOIN_DIAG_NOMMA = 0,
    FASTED_JOIN_DIAG_LOADONLY = 0,
    FASTED_JOIN_DIAG_NOSLOW = 0,
    FASTED_JOIN_DIAG_SPIN = 0,
    FASTED_JOIN_DIAG_LDX64 = 0,
    FASTED_JOIN_DIAG_AEVL = 0,
    FASTED_JOIN_DIAG_TRACE = 0,
    FASTED_JOIN_DIAG_RARE_LM = 0,
    FASTED_JOIN_DIAG_RARE_ROWS = 0,
    FASTED_JOIN_DIAG_NOAUG = 0,
    FASTED_JOIN_DIAG_AUGF16 = 0,
    FASTED_JOIN_DIAG_HITMETA = 0,
    FASTED_JOIN_DIAG_HITSKIP = 0,
    FASTED_JOIN_DIAG_NOTMA = 0,
    FASTED_JOIN_DIAG_NOREMOTE = 0,
    FASTED_JOIN_DIAG_HITPACK = 0,
    FASTED_JOIN_DIAG_GENERICQ = 0,
    FASTED_JOIN_DIAG_EPISPIN = 0,
    FASTED_JOIN_DIAG_EPIBAR = 0
};

#endif

}  // namespace fasted
