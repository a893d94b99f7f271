python -c "import __graft_entry__ as g; g.build()"
timeout 300 python tools/net_trace.py
