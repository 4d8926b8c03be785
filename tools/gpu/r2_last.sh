#!/usr/bin/env bash
# End-of-round check: full GPU suite, smoke, the default bench (c2 + secondary rows),
# the reference arm.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2l; mkdir -p $O
timeout 2400 python -m pytest tests -q -m gpu --timeout 900 -p no:cacheprovider > $O/pytest.log 2>&1
echo "pytest rc=$?"; tail -1 $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?"
