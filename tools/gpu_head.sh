# full GPU test suite, one bench line, one ncu capture of the event-loop kernel
TAG=${1:-head}
python -m pytest tests/ -x -q -m gpu 2>&1 | tail -4
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
NCU=${NCU:-1} bash tools/gpu_iter.sh $TAG
