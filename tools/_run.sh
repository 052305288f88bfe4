./paper_2401_09792_b200/_build/test_dropin 2>&1 | tail -5
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
