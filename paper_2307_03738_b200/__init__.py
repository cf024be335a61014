"""qigen-b200: QIGen's quantized-GEMV hot path (arXiv 2307.03738), rebuilt for
NVIDIA B200 (sm_100a).

Public API mirrors the reference package ``qigen`` (config / quant / packing /
perfmodel entry points and the runtime it specified): quantize and pack are
bit-exact with the reference, ``qgemv`` runs the hand-written CUDA kernel in
``libqigen_b200.so``.  See DESIGN.md.
"""

from .config import (FULL_COLUMN, SUPPORTED_BITS, ConfigError, QuantConfig, ZeroMode,
                     check_row_count, codes_per_word, pack_unit, row_alignment)
from .perfmodel import (DEFAULT_HARDWARE, HardwareSpec, PlanError, TilePlan, load_hardware_spec,
                        plan, save_hardware_spec, select_cache_block, select_register_tile)
from .quant import (CodeMatrix, GroupParams, dequantize, dequantize_matrix, quantize_group,
                    quantize_matrix)
from .packing import (Layout, PackedMatrix, PackError, block_order, extract_codes,
                      lay_out_blocks, morton_index, pack_words, unpack_words)
from .runtime import (GemvGroup, InputSums, PanelWeights, input_sums, memory_report, qgemv,
                      qgemv_batch, qgemv_batch_inputs, qgemv_reference)

from .weightfile import (BadMagicError, ChecksumError, TruncatedError, VersionError,
                         WeightFileError, load_panels, read_weight_file, write_weight_file)

__version__ = "0.1.0"
