"""Mutation probe of the CPU oracle's pins (round-1 VERDICT, "What's weak" 1).

Builds oracle/dabs_oracle.c with one deliberate mistake at a time (the eight
mutants the round-1 review found surviving, plus a few more), loads each build
through DABS_ORACLE_LIB and runs the oracle pin suites.  A mutant is "killed"
when at least one pin fails.  Exit status 1 if any mutant survives.

    python tools/mutation_probe.py            # all mutants
    python tools/mutation_probe.py -k tabu    # those whose name contains "tabu"
"""
import argparse
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "dabs_oracle.c")
PINS = ["tests/test_oracle_rules.py", "tests/test_oracle_pins.py", "tests/test_async_oracle.py",
        "tests/test_jump_oracle.py"]

# (name, function the edit is confined to, old text, new text)
MUTANTS = [
    ("cyclicmin_window_all_n", "sel_cyclicmin", "if (w > (uint64_t)n) w = n;", "w = n;"),
    ("cyclicmin_cursor_fixed", "sel_cyclicmin", "*cursor = (int)((*cursor + w) % n);", "*cursor = *cursor;"),
    ("cyclicmin_c16", "sel_cyclicmin", "n < 32 ? (uint64_t)n : 32u", "n < 16 ? (uint64_t)n : 16u"),
    ("cyclicmin_floor_not_ceil", "sel_cyclicmin", "((num + T3 - 1) / T3)", "(num / T3)"),
    ("randommin_p_linear", "sel_randommin", "uint64_t t3 = (uint64_t)t * t * t;",
     "uint64_t t3 = (uint64_t)t * s->T * s->T;"),
    ("randommin_floor_16_over_n", "sel_randommin", "2097152u / (uint32_t)n", "1048576u / (uint32_t)n"),
    ("randommin_highest_index_ties", "sel_randommin", "(j < 0 || s->delta[k] < s->delta[j])) j = k;",
     "(j < 0 || s->delta[k] <= s->delta[j])) j = k;"),
    ("maxmin_square_law", "sel_maxmin", "(u * u * u)", "(u * u * T)"),
    ("maxmin_u_eq_t", "sel_maxmin", "u = (uint64_t)(s->T - t);", "u = (uint64_t)t;"),
    ("maxmin_span_ignores_tabu", "sel_maxmin",
     "if (elig[k]) { if (s->delta[k] < lo)", "if (1) { if (s->delta[k] < lo)"),
    ("posmin_nonstrict_positive", "sel_positivemin", "s->delta[k] > 0 &&", "s->delta[k] >= 0 &&"),
    ("tabu_period_plus_one", "is_tabu", "j < s->tabu;", "j <= s->tabu;"),
    ("tabu_period_minus_one", "is_tabu", "j < s->tabu;", "j < s->tabu - 1;"),
    ("tabu_disabled", "is_tabu", "if (s->ring[j] == k) return 1;", "if (0) return 1;"),
    ("eps_threshold_32bit", "orc_world_new", "w->eps_thr = ((uint64_t)eps_ppm << 32) / 1000000u;",
     "w->eps_thr = (uint32_t)(((uint64_t)eps_ppm << 32) / 1000000u);"),
]


def mutate(src: str, func: str, old: str, new: str) -> str:
    start = src.index(func + "(")
    at = src.index(old, start)
    return src[:at] + new + src[at + len(old):]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("-k", default="")
    args = ap.parse_args()
    src = open(SRC).read()
    survived = []
    with tempfile.TemporaryDirectory() as tmp:
        for name, func, old, new in MUTANTS:
            if args.k not in name:
                continue
            m = mutate(src, func, old, new)
            assert m != src, name
            c = os.path.join(tmp, name + ".c")
            so = os.path.join(tmp, name + ".so")
            open(c, "w").write(m)
            subprocess.check_call(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", c, "-o", so])
            env = dict(os.environ, DABS_ORACLE_LIB=so)
            r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-m", "not gpu", *PINS],
                               cwd=ROOT, env=env, capture_output=True, text=True)
            failed = [ln for ln in r.stdout.splitlines() if ln.startswith("FAILED")]
            status = "killed" if r.returncode != 0 else "SURVIVED"
            print(f"{name:32s} {status:9s} {failed[0][7:] if failed else ''}", flush=True)
            if r.returncode == 0:
                survived.append(name)
    print(f"{len(survived)} survived" + (": " + ", ".join(survived) if survived else ""))
    sys.exit(1 if survived else 0)


if __name__ == "__main__":
    main()
