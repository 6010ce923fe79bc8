timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -2
timeout 600 python tools/probe.py big 2>&1 | grep "^ch"
timeout 600 python tools/probe.py big 2>&1 | grep "^ch"
MSY_NO_STREAM_PRIORITY=1 timeout 600 python tools/probe.py big 2>&1 | grep "^ch"
MSY_NO_STREAM_PRIORITY=1 timeout 600 python tools/probe.py big 2>&1 | grep "^ch"
