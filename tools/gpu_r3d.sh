python -c "import __graft_entry__ as g; g.build()" || exit 1
python tools/quant_time.py --config c3; python tools/quant_time.py --config c2
python -c "
import sys; sys.path.insert(0, '.')
from paper_2406_02528_b200 import build as b
b.FLAGS.append('-DTERN_QUANT_NOSUM'); b.build(force=True)" || exit 1
python tools/quant_time.py --config c3 | sed 's/^/nosum /'; python tools/quant_time.py --config c2 | sed 's/^/nosum /'
