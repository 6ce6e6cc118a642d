timeout 1500 python -m pytest tests -q -m gpu -x -k "not test_reference_acceptance" 2>&1 | tail -4
timeout 300 python -m pytest tests -q -m gpu -k "test_reference_acceptance" 2>&1 | tail -3
