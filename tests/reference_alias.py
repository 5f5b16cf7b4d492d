"""pytest plugin (TEST INFRASTRUCTURE): makes ``import prodmatch...`` resolve to
this package, so the reference's own test files run against it unchanged
(tests/test_reference_api.py)."""
import sys

import paper_2310_08230_b200 as pkg
from paper_2310_08230_b200 import bdd, errors, ilp, splitting

for name, mod in (("prodmatch", pkg), ("prodmatch.bdd", bdd), ("prodmatch.errors", errors), ("prodmatch.ilp", ilp),
                  ("prodmatch.splitting", splitting)):
    sys.modules[name] = mod
