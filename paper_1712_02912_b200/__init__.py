"""paper_1712_02912_b200 -- B200-native (sm_100a) PQ ADC scan engine.

Drop-in for the hot path of `pqscan` (arxiv/paper_1712_02912): lookup tables,
the float ADC scan over 8-bit codes, the Quick ADC 4-bit quantized scan,
IVFADC probing and top-r selection, plus batched device APIs and a sharded
multi-GPU search.  All compute runs in libpqs.so (hand-written CUDA for
sm_100a); there is no CPU fallback.
"""

from .types import (  # noqa: F401
    BINS,
    BLOCK,
    DEFAULT_INIT_COUNT,
    DEFAULT_INIT_COUNT_BILLION,
    CodeList,
    IvfIndex,
    LookupTables,
    NeighborSet,
    ProductQuantizer,
    QuantizedTables4,
    QuantParams,
    TrainError,
    TransposedCodeList,
)
from .scan import (  # noqa: F401
    adc_distance,
    compute_tables,
    compute_tables_batch,
    detranspose_blocks,
    scan,
    scan_distances,
    transpose_blocks,
)
from .quantizer import encode  # noqa: F401
from .formats import (  # noqa: F401
    FormatError,
    load_codes,
    load_codes_device,
    load_ivf,
    load_ivf_device,
    load_quantizer,
    save_codes,
    save_ivf,
    save_quantizer,
)
from .quickadc import qadc_block, qadc_scan, quantize, quantize_tables_4bit, quantized_distances  # noqa: F401
from .fastscan import (  # noqa: F401
    GroupedDatabase,
    ScanStats,
    SmallTables,
    build_small_tables,
    compute_quant_params,
    fast_scan,
    group_codes,
    group_key,
    load_grouped,
    lower_bound,
    pack_code,
    relabel_codes,
    save_grouped,
)
from .derived import (  # noqa: F401
    CBINS,
    DerivedPQ,
    compute_compact_tables,
    load_derived,
    load_quantizer_any,
    save_derived,
    search_two_pass,
)
from .ivf import KERNELS, default_r2, device_index, query_ivf, query_ivf_batch  # noqa: F401
from .engine import DeviceCodes, DeviceIvf, DeviceQuantizer, merge_topr, nearest  # noqa: F401
from ._lib import Context, default_context, load_library  # noqa: F401

__version__ = "0.1.0"
