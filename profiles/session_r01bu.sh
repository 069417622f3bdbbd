#!/bin/bash
# Round-1 session bu: final full GPU suite + smoke on the final code.
O=gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > $O/bu_pytest.log 2>&1; echo "pytest rc $?" >> $O/bu_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/bu_smoke.log 2>&1; echo "smoke rc $?" >> $O/bu_smoke.log
tail -3 $O/bu_pytest.log; tail -3 $O/bu_smoke.log
