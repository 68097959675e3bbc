"""Pivot bounded walks + spill rounds (csrc/kc_count.cu kc_do_count, kct::Spill).

The spill machinery only changes WHO walks which subtree, so counts and
visits must equal the unbounded walk's -- the reference's (engine_pivot.py:
117-233).  Budgets are read once per process (KC_SPILL, KC_SPILL_BUDGET), so
each configuration runs in its own subprocess: the default budget, a tiny
budget (64 branches: thousands of rounds of kind-0 / kind-2 items, big items
on the CTA tier), and spilling off.  Dense G(n, p) graphs put vertex tasks
above 128 locals (CTA tier, big items); rmat14 k=10 is checked against the
reference's own golden record.
"""

import json
import os
import subprocess
import sys

import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)

CASES = [  # (graph, k, scheme)
    ("gnp400", 8, "vertex"),
    ("gnp400", 10, "edge"),
    ("gnp300", 10, "edge"),
    ("gnp300", 6, "vertex"),
    ("rmat14", 10, "edge"),
]

SNIPPET = r"""
import json, sys
sys.path.insert(0, %(repo)r)
import paper_2104_13209_b200 as kc
from paper_2104_13209_b200 import synth
graphs = {"gnp400": synth.erdos_renyi(400, 0.5, seed=5), "gnp300": synth.erdos_renyi(300, 0.6, seed=5),
          "rmat14": synth.workload("rmat14")}
out = []
for name, k, scheme in %(cases)r:
    g = kc.from_edges(graphs[name])
    r = kc.run_count(g, kc.RunConfig(k=k, algorithm="pivot", scheme=scheme, criterion="degeneracy"))
    out.append([name, k, scheme, str(r.count), int(r.load.total), r.counters.get("launches")])
    g.free()
print("RESULT " + json.dumps(out))
"""


def _run(env_extra):
    env = dict(os.environ)
    env.update(env_extra)
    env.setdefault("KC_DEVICE", "0")
    src = SNIPPET % {"repo": REPO, "cases": CASES}
    r = subprocess.run([sys.executable, "-c", src], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    line = [x for x in r.stdout.splitlines() if x.startswith("RESULT ")][-1]
    return json.loads(line[len("RESULT "):])


@pytest.fixture(scope="module")
def expected():
    import oracle
    from paper_2104_13209_b200 import synth

    graphs = {"gnp400": synth.erdos_renyi(400, 0.5, seed=5),
              "gnp300": synth.erdos_renyi(300, 0.6, seed=5)}
    exp = {}
    for name, k, scheme in CASES:
        if name == "rmat14":
            rec = [r for r in load_golden("scale.json")
                   if (r["workload"], r["k"], r["algorithm"], r["scheme"], r["criterion"])
                   == ("rmat14", k, "pivot", scheme, "degeneracy")][0]
            exp[(name, k, scheme)] = (rec["count"], rec["visits"])
            continue
        og = oracle.from_edges(graphs[name])
        o = oracle.run_count(og, k, "pivot", scheme, "degeneracy", workers=8)
        exp[(name, k, scheme)] = (str(o.count), int(o.visits))
    return exp


@pytest.mark.parametrize("env", [{}, {"KC_SPILL_BUDGET": "64"}, {"KC_SPILL": "0"}],
                         ids=["default", "budget64", "nospill"])
def test_spill_rounds_keep_counts_and_visits(expected, env):
    for name, k, scheme, count, visits, _ in _run(env):
        assert (count, visits) == expected[(name, k, scheme)], (name, k, scheme, env)
