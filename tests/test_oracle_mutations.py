"""The oracle's pins must catch plausible mistakes (task ③): each mutant below is a copy of
oracle/rgc_oracle.c with one reading or step changed the way a slip would change it, built
with the same flags, and at least one pin of tests/test_oracle_pins.py has to fail on it.

The three readings the round-1 review found unpinned come first (R2's tile exponent, R3's
double-precision thresholds, R18's EPS_BEST choice); the others guard the pins that already
caught their mutations.  CPU only (gcc), a few seconds per mutant.
"""
import os

import pytest

import oracle as O
import test_oracle_pins as P

SRC = os.path.join(os.path.dirname(O.__file__), "rgc_oracle.c")

FLOAT_THRESH = """static float thresh_at(double mean, double maxd, double ratio)
{
    float d = (float)maxd - (float)mean;
    float p = (float)ratio * d;
    return (float)mean + p;
}
"""

# name -> (exact text in rgc_oracle.c, replacement, pins expected to catch it)
MUTANTS = {
    # R2: E_t = floor(log2 tile max) = e - 1 for frexp's e
    "R2_tile_exponent_e": (
        "int E = e - 1;", "int E = e;",
        [P.test_mean_fx_hand_worked_bins]),
    "R2_term_rounds_instead_of_truncating": (
        "S += (uint64_t)floor(ldexp(", "S += (uint64_t)nearbyint(ldexp(",
        [P.test_mean_fx_hand_worked_bins]),
    # R3: thresholds in double with one rounding to f32
    "R3_float_thresholds": (
        None, FLOAT_THRESH,
        [P.test_bs_hand_worked_paths]),
    # R18: EPS_BEST = the evaluated threshold with the smallest nnz >= k (first on a tie)
    "R18_first_best": (
        "if (nnz >= k && (!have_best || nnz < best_c)) {",
        "if (nnz >= k && !have_best) {",
        [P.test_bs_hand_worked_paths]),
    "R18_last_best": (
        "if (nnz >= k && (!have_best || nnz < best_c)) {",
        "if (nnz >= k) {",
        [P.test_bs_hand_worked_paths]),
    "R18_largest_best": (
        "if (nnz >= k && (!have_best || nnz < best_c)) {",
        "if (nnz >= k && (!have_best || nnz > best_c)) {",
        [P.test_bs_hand_worked_paths]),
    # R9: strict break k < nnz < 2k
    "R9_break_not_strict": (
        "if (nnz > k && 2 * k > nnz) { broke = 1; break; }",
        "if (nnz >= k && 2 * k > nnz) { broke = 1; break; }",
        [P.test_bs_hand_worked_paths]),
    # R7: MONOTONE branch nnz <= k -> r
    "R7_monotone_strict": (
        "if (nnz <= k) r = ratio; else l = ratio;",
        "if (nnz < k) r = ratio; else l = ratio;",
        [P.test_bs_hand_worked_paths]),
    # R6: ties broken by the lower index
    "R6_tie_higher_index": (
        "return (x->i < y->i) ? -1 : (x->i > y->i);",
        "return (x->i > y->i) ? -1 : (x->i < y->i);",
        [P.test_exact_topk_exhaustive_small_alphabet]),
    # O2: V <- V + u (the momentum-corrected gradient), not V + g
    "O2_residual_adds_g": (
        "V[i] = V[i] + u[i];", "V[i] = V[i] + g[i];",
        [P.test_accumulate_exact_fma_and_add]),
    # O11 / R13: the rank-ordered sum is scaled by fl32(1/p)
    "O11_no_scale": (
        "for (uint64_t i = 0; i < n; i++) out[i] = out[i] * s;",
        "for (uint64_t i = 0; i < n; i++) out[i] = out[i] + 0.0f * s;",
        [P.test_decompress_dense_equivalence_and_scale]),
}


def _mutant_source(old, new):
    src = open(SRC).read()
    if old is None:   # replace the whole thresh_at function
        a = src.index("static float thresh_at(")
        b = src.index("}\n", a) + 2
        return src[:a] + new + src[b:]
    assert src.count(old) == 1, f"mutation anchor not unique / missing: {old!r}"
    return src.replace(old, new)


def _fails(fn):
    try:
        fn()
    except AssertionError:
        return True
    return False


@pytest.mark.parametrize("name", list(MUTANTS))
def test_pins_catch_mutant(name, tmp_path):
    old, new, pins = MUTANTS[name]
    so = O.build_variant(_mutant_source(old, new), str(tmp_path / f"mut_{name}.so"))
    # the real oracle passes these pins
    for fn in pins:
        fn()
    with O.use_library(so):
        caught = [fn.__name__ for fn in pins if _fails(fn)]
    assert caught, f"mutant {name} survives {[f.__name__ for f in pins]}"
