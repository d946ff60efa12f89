"""``fastsearch.bench.persist`` module path (bench/persist.py:1-112): the
FBSIDX1 index-file API lives in ``paper_1506_08620_b200.persist``."""

from ..persist import (  # noqa: F401
    MAGIC,
    VERSION,
    device_crc32,
    load_index,
    pack_header,
    parse_header,
    prepare_loaded,
    save_index,
)
