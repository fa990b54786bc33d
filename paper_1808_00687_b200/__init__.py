"""B200-native WFST Viterbi decoder (arXiv 1808.00687), drop-in for ``lsd_wfst``'s decode path.

Public names mirror ``lsd_wfst`` (reference ``pkg/src/lsd_wfst/__init__.py``) for the decode
path: graph + per-frame acoustic scores in; best path, cost and lattices out.  The search
itself runs in hand-written sm_100a CUDA kernels (``csrc/``) behind the C ABI declared in
``include/wfst_b200.h``.
"""
__version__ = "0.1.0"

from .decoder import (BatchDecoder, BatchOutput, DecodeConfig, DecodeResult, DeviceGraph,
                      SearchDied, as_wfst, decode, decode_batch, decode_fsd, decode_lsd,
                      parallel_decode)
from .lattice import LatticeError, LatticeRecorder, PipelinedLatticeBuilder
from .posteriors import (BlankMask, PosteriorBatch, PosteriorFormatError, PosteriorMatrix, acoustic_cost,
                         classify_blank_frames, cost_table, frame_costs, load_posteriors,
                         save_posteriors)
from .lattice import (EMPTY_LATTICE, Lattice, build_lattice, lattice_best_path, prune_lattice)
from .pipeline import LatticePipeline
from .shard import decode_multi_device, decode_sharded, shard_utterances
from .wfst import (Arc, EpsilonCycle, ParseError, SymbolError, SymbolTable, Wfst, WfstError,
                   format_wfst_text, load_wfst_binary, parse_wfst_text, save_wfst_binary,
                   validate_epsilon_acyclic)

__all__ = [
    "Arc", "BatchDecoder", "BatchOutput", "BlankMask", "DecodeConfig", "DecodeResult",
    "DeviceGraph", "EpsilonCycle", "LatticeError", "LatticeRecorder", "ParseError",
    "PosteriorBatch", "PosteriorFormatError", "PosteriorMatrix", "SearchDied", "Wfst", "WfstError",
    "acoustic_cost", "as_wfst", "classify_blank_frames", "cost_table", "decode",
    "decode_batch", "decode_fsd", "decode_lsd", "frame_costs", "parallel_decode",
    "parse_wfst_text", "validate_epsilon_acyclic", "load_posteriors", "save_posteriors",
    "EMPTY_LATTICE", "Lattice", "build_lattice", "lattice_best_path", "prune_lattice",
    "LatticePipeline", "decode_multi_device", "decode_sharded", "shard_utterances",
    "PipelinedLatticeBuilder", "SymbolError", "SymbolTable", "format_wfst_text", "load_wfst_binary", "save_wfst_binary",
]
