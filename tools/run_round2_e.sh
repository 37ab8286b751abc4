python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
python tools/relabel_probe.py --dtype f32,f64 --L 20 2>&1 | grep "config 3"
