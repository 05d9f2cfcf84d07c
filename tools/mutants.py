"""Mutation check of the oracle's pins: each mutant is a one-line change to
oracle/ekya_oracle.c (a plausible mistake); the -m "not gpu" oracle pins must fail on it.
Runs in a scratch copy under /tmp; prints the first failing test per mutant.
usage: python tools/mutants.py [name ...]"""
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

MUTANTS = {
    # NEXT-1 window timeline (readings W3, W6)
    "W3-idle-no-rescale": ("if (stt[v] == 0) cs = isinf(c) ? c : c * sc;", "if (stt[v] == 0) cs = c;"),
    "W3-retraining-no-rescale": ("else if (stt[v] == 1 && k + 1 == g[v]) cs = R[v] * sc;",
                                 "else if (stt[v] == 1 && k + 1 == g[v]) cs = R[v];"),
    "W6-keep-done-fraction": ("const float keep = 1.0f - q;", "const float keep = q;"),
    # A1 RADIUS threshold (C17)
    "C17-strict": ("sim[h] = dist <= p->tau;", "sim[h] = dist < p->tau;"),
    "rule5-d2-as-d": ("float dist = sqrtf(d2);", "float dist = d2;"),
    "C18-nan-counted": ("if (!sim[h] || isnan(a)) continue;", "if (!sim[h]) continue;"),
    "C19-init-ceil": ("hq + ((i * H) / K) * C", "hq + ((i * H + K - 1) / K) * C"),
    "C19-nearest-ties": ("if (di < bd) {                     /* lowest index on ties (C19) */",
                         "if (di <= bd) {                     /* lowest index on ties (C19) */"),
    "C19-empty-cluster": ("if (cnt[i] == 0) continue;   /* empty", "if (0) continue;   /* empty"),
    # rules 1-4 (Alg. 2)
    "C5-strict-feasible": ("return f <= 1.0f;", "return f < 1.0f;"),
    "rule2-sign": ("float g = post - prod;", "float g = post + prod;"),
    "rule4-truncating-q32": ("return (uint64_t)llrintf(y);", "return (uint64_t)y;"),
    "C7-last-index-wins": ("if (a > best) {                    /* strict", "if (a >= best) {                    /* strict"),
    "C7-lambda-last-index": ("if (best < 0 || acc > best_acc) {", "if (best < 0 || acc >= best_acc) {"),
    "C2-keepup-strict": ("if (ri < (int32_t)lmu[l]) continue;", "if (ri <= (int32_t)lmu[l]) continue;"),
    "C3-amin-strict": ("if (!(acc >= a_min)) continue;", "if (!(acc > a_min)) continue;"),
    # Alg. 1 (A4-A5)
    "C9-fair-half-up": ("int32_t rt = share / 2;", "int32_t rt = (share + 1) / 2;"),
    "C14-floor": ("if (temp[victim] < 0) break;", "if (temp[victim] <= 0) break;"),
    # rules 1-2 (Alg. 2)
    "rule1-denominator-rt+1": ("float denom = (float)rt * uT;          /* fl(float(rt) * uT) */",
                               "float denom = (float)(rt + 1) * uT;          /* fl(float(rt) * uT) */"),
    # (rule 1's explicit rt < 1 test is redundant in IEEE arithmetic -- cost / (0 uT) is +INF or
    # NaN, never <= 1 -- so dropping it is an equivalent mutant, not listed)
    "rule2-post-as-base": ("float g = post - prod;", "float g = stale + prod;"),
    # Alg. 1: LITERAL order and acceptance, STEEPEST ties and victim floor
    "C10-literal-victim-first": ("for (int32_t thief = 0; thief < J; ++thief) {          /* line 5 */",
                                 "for (int32_t thief = J - 1; thief >= 0; --thief) {          /* line 5 */"),
    "C12-steepest-ties-last": ("                if (s > best) {\n                    best = s;\n                    bt = t;",
                               "                if (s >= best && s > cur) {\n                    best = s;\n                    bt = t;"),
    # A1 CLUSTER (C19): Lloyd iteration count and the query's cluster
    "C19-max-iter-off-by-one": ("for (int32_t it = 0; it < p->max_iter; ++it) {",
                                "for (int32_t it = 0; it + 1 < p->max_iter; ++it) {"),
    "C19-no-convergence-stop": ("if (!changed) break;", "if (0 && !changed) break;"),
    "C20-fallback-zero": ("out_est[q * G + g] = n > 0 ? orc_mean_from_q32(s, n) : fallback[q * G + g];",
                          "out_est[q * G + g] = n > 0 ? orc_mean_from_q32(s, n) : 0.0f;"),
    # Eq. 1 constraint 2 (LIST)
    "EQ1-strict-total": ("if (tot > d->units) row_ok = 0;   /* Eq. 1 constraint 2 */",
                         "if (tot >= d->units) row_ok = 0;   /* Eq. 1 constraint 2 */"),
    "rule4-mean-over-V+1": ("double m = (double)s / ((double)n * 4294967296.0);",
                            "double m = (double)s / ((double)(n + 1) * 4294967296.0);"),
    # NEXT-4 placement (PL1, PL2) and checkpoint (CK1)
    "PL1-quantize-up": ("while ((r << k) < (int64_t)U) ++k;", "while ((r << k) <= (int64_t)U) ++k;"),
    "PL2-strict-fit": ("if (load[g] + pc[i].q <= ORC_Q_ONE)", "if (load[g] + pc[i].q < ORC_Q_ONE)"),
    "PL2-ties-job-desc": ("if (a->job != b->job) return a->job < b->job ? -1 : 1;",
                          "if (a->job != b->job) return a->job > b->job ? -1 : 1;"),
    "CK1-ge": ("out[i] = lhs > rhs;", "out[i] = lhs >= rhs;"),
    "CK1-gain-sign": ("const float gain = a_star[i] - a[i];", "const float gain = a[i] - a_star[i];"),
    # NEXT-3 uniform (U1, U2), Pareto (PR1), pruning (PN1, PN2)
    "U1-ceil": ("const int32_t rt = (int32_t)floorf(x);", "const int32_t rt = (int32_t)ceilf(x);"),
    "U2-best-last-index": ("if (g == 0 || pv[k] > bp) { g = k + 1; bp = pv[k]; }",
                           "if (g == 0 || pv[k] >= bp) { g = k + 1; bp = pv[k]; }"),
    "U2-infeasible-zero": ("                float acc = st;\n", "                float acc = 0.0f;\n"),
    "PR1-weak-dominance": ("if (c[j] <= c[k] && p[j] >= p[k] && (c[j] < c[k] || p[j] > p[k])) dominated = 1;",
                           "if (c[j] <= c[k] && p[j] >= p[k]) dominated = 1;"),
    "PN1-strict-cost": ("if (c[k2] <= c[k] && a[k2] > boundary) boundary = a[k2];",
                        "if (c[k2] < c[k] && a[k2] > boundary) boundary = a[k2];"),
    "PN2-half-inclusive": ("if (!(2 * far > measured)) keep |= 1u << k;",
                           "if (!(2 * far >= measured)) keep |= 1u << k;"),
    "PN1-gap-ge": ("if (gap > margin) ++far;", "if (gap >= margin) ++far;"),
    # NEXT-2 curve fit (CF1-CF3)
    "CF2-grid-ties-last": ("if (i == 0 || e < best) {", "if (i == 0 || e <= best) {"),
    # (CF1's tie between the two boundary fits, `e1 < e0` -> `<=`, is left out: it changes the
    # output only on an exact SSE tie of two distinct fits, none in 800 K random 64ths sets)
    "CF3-no-clamp": ("p = p < 0.0f ? 0.0f : (p > 1.0f ? 1.0f : p);", "p = p;"),
    "CF1-x-offset": ("const float den = (float)(k + 1) + c;", "const float den = (float)k + c;"),

    "C13-accept-ties": ("if (acc > best_acc) {", "if (acc >= best_acc) {"),
    "C12-steepest-victim-floor": ("if (t == w || alloc[w] < D) continue;", "if (t == w || alloc[w] <= D) continue;"),
}


def run(name, old, new):
    tmp = f"/tmp/ekya_mut_{os.getpid()}"
    shutil.rmtree(tmp, ignore_errors=True)
    os.makedirs(tmp)
    for d in ("oracle", "synth", "tests"):
        shutil.copytree(os.path.join(ROOT, d), os.path.join(tmp, d),
                        ignore=shutil.ignore_patterns("_build", "__pycache__"))
    shutil.copy(os.path.join(ROOT, "pytest.ini"), tmp)
    src_path = os.path.join(tmp, "oracle", "ekya_oracle.c")
    src = open(src_path).read()
    assert src.count(old) == 1, f"{name}: pattern not unique"
    open(src_path, "w").write(src.replace(old, new))
    r = subprocess.run([sys.executable, "-m", "pytest", "tests/test_oracle_pins.py", "-x", "-q", "-m", "not gpu",
                        "-p", "no:cacheprovider"], cwd=tmp, capture_output=True, text=True)
    shutil.rmtree(tmp, ignore_errors=True)
    failed = [ln.split(" ")[1] for ln in r.stdout.splitlines() if ln.startswith("FAILED")]
    return r.returncode != 0, failed


if __name__ == "__main__":
    names = sys.argv[1:] or list(MUTANTS)
    ok = True
    for n in names:
        killed, failed = run(n, *MUTANTS[n])
        ok &= killed
        print(f"{n:28s} {'killed by ' + (failed[0] if failed else '?') if killed else 'SURVIVED'}")
    sys.exit(0 if ok else 1)
