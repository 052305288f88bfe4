timeout 900 python -m pytest tests -m gpu -q 2>&1 | grep -E "FAILED|passed|failed" | head -5
./paper_2401_09792_b200/_build/test_dropin 2>&1 | tail -1
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
