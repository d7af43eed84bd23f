python __graft_entry__.py >/dev/null 2>&1
timeout 600 python -m pytest tests -m gpu -q -k "wide_schedule" 2>&1 | tail -15
