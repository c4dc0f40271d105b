timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --tb=short 2>&1 | tail -6
QT_GRAPH=20 timeout 300 python tools/quick_time.py c4 c5
