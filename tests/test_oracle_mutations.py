"""The oracle pins are not self-consistent only: each plausible misreading of the paper
below, built into a copy of oracle/oracle.c, makes at least one pin of
tests/test_oracle_pins.py fail (the pins constrain the oracle from outside).

The mutations are the ones a reader could make of PAPER.md or of DESIGN.md's readings:
R-2 (stop rule, threshold), R-3 (update order), R-4 (alpha cap), R-14 (Jacobian clamp,
dilation), Eq. (3) (sign of the cross term), R-12 (tie-break), the 3-sigma radius and the
1/255 skip threshold.
"""
import os
import subprocess
import sys
import tempfile

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "oracle.c")

MUTATIONS = {
    # R-4: no alpha cap (PAPER.md P:169 / P:376 read literally)
    "no_alpha_cap": [("const double alpha = a_raw < 0.99 ? a_raw : 0.99;", "const double alpha = a_raw;"),
                     ("if (alpha > 0.99) alpha = 0.99;", "")],
    # R-2: the stopping Gaussian composited before the stop
    "stopper_composited": [
        ("if (tT < t_min) break;                                      /* R-2 */\n"
         "                for (int ch = 0; ch < 3; ch++) C[ch] += (double)J->rgb[3 * i + ch] * alpha * T; /* R-3 */\n"
         "                T = tT;",
         "for (int ch = 0; ch < 3; ch++) C[ch] += (double)J->rgb[3 * i + ch] * alpha * T;\n"
         "                T = tT;\n"
         "                if (tT < t_min) break;"),
        ("if (tT < 1e-4) break;\n        for (int ch = 0; ch < 3; ch++) C[ch] += (double)rgb[3 * i + ch] * alpha * T;\n"
         "        T = tT;",
         "for (int ch = 0; ch < 3; ch++) C[ch] += (double)rgb[3 * i + ch] * alpha * T;\n        T = tT;\n"
         "        if (tT < 1e-4) break;")],
    # R-2: termination threshold 1e-6 instead of 1e-4
    "threshold_1e-6": [("const double t_min = 1e-4, ln_tmin = log(1e-4);",
                        "const double t_min = 1e-6, ln_tmin = log(1e-6);"),
                       ("if (tT < 1e-4) break;", "if (tT < 1e-6) break;")],
    # R-2: the paper's literal "T <= 0 -> stop"
    "stop_at_T_le_0": [("if (tT < t_min) break;", "if (tT <= 0.0) break;"),
                       ("if (tT < 1e-4) break;", "if (tT <= 0.0) break;")],
    # R-3: Alg. 1's order (T updated before the colour) instead of Eq. (1)
    "accumulate_with_new_T": [("C[ch] += (double)J->rgb[3 * i + ch] * alpha * T; /* R-3 */",
                               "C[ch] += (double)J->rgb[3 * i + ch] * alpha * tT;"),
                              ("C[ch] += (double)rgb[3 * i + ch] * alpha * T;",
                               "C[ch] += (double)rgb[3 * i + ch] * alpha * tT;")],
    # R-14: Jacobian clamp at 1.0 tan(fov/2) instead of 1.3
    "clamp_1.0": [("float lx = 1.3f * cam->tan_fovx, ly = 1.3f * cam->tan_fovy;",
                   "float lx = 1.0f * cam->tan_fovx, ly = 1.0f * cam->tan_fovy;")],
    # R-14: no clamp at all
    "no_clamp": [("float cxz = fminf(lx, fmaxf(-lx, ux));", "float cxz = ux;"),
                 ("float cyz = fminf(ly, fmaxf(-ly, uy));", "float cyz = uy;")],
    # R-14: no +0.3 low-pass dilation
    "no_dilation": [("float a = c00 + 0.3f, b = c01, c = c11 + 0.3f;", "float a = c00, b = c01, c = c11;")],
    # Eq. (3): sign of the cross term
    "cross_term_sign": [("const double power = -0.5 * (A * dx * dx + Cc * dy * dy) - B * dx * dy;\n"
                         "                const double o = J->opacity[i];",
                         "const double power = -0.5 * (A * dx * dx + Cc * dy * dy) + B * dx * dy;\n"
                         "                const double o = J->opacity[i];"),
                        ("const double power = -0.5 * (A * dx * dx + Cc * dy * dy) - B * dx * dy;\n"
                         "        double alpha",
                         "const double power = -0.5 * (A * dx * dx + Cc * dy * dy) + B * dx * dy;\n"
                         "        double alpha")],
    # R-12: equal depths ordered by descending index
    "tie_break_desc": [("if (a->idx != b->idx) return a->idx < b->idx ? -1 : 1;",
                        "if (a->idx != b->idx) return a->idx > b->idx ? -1 : 1;")],
    # radius 2 sigma instead of 3 sigma
    "radius_2sigma": [("float rr = ceilf(3.0f * sqrtf(lam));", "float rr = ceilf(2.0f * sqrtf(lam));")],
    # skip threshold 1/256 instead of 1/255
    "skip_1_over_256": [("const double a_min = (double)(1.0f / 255.0f);", "const double a_min = (double)(1.0f / 256.0f);"),
                        ("if (alpha < (double)(1.0f / 255.0f)) continue;", "if (alpha < (double)(1.0f / 256.0f)) continue;")],
}


@pytest.mark.parametrize("name", ["control"] + list(MUTATIONS))
def test_pins_catch_the_mutation(name, tmp_path):
    """control: the unmodified source built the same way passes every pin (so a failure
    below is the mutation's, not the rebuild's)."""
    src = open(SRC).read()
    for old, new in MUTATIONS.get(name, []):
        assert src.count(old) == 1, (name, old)
        src = src.replace(old, new)
    c = tmp_path / "oracle_mut.c"
    c.write_text(src)
    so = tmp_path / "liboracle_mut.so"
    import oracle
    subprocess.check_call(["gcc", *oracle.CFLAGS, str(c), "-o", str(so), "-lm"])
    env = dict(os.environ, ORACLE_LIB=str(so))
    r = subprocess.run([sys.executable, "-m", "pytest", os.path.join(ROOT, "tests", "test_oracle_pins.py"), "-x", "-q",
                        "-p", "no:cacheprovider"], env=env, capture_output=True, text=True, cwd=ROOT, timeout=600)
    if name == "control":
        assert r.returncode == 0, r.stdout[-2000:]
        return
    assert r.returncode == 1, f"mutation {name} passed every pin:\n{r.stdout[-2000:]}"
    assert "failed" in r.stdout
