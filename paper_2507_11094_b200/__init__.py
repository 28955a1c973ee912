"""B200-native dynamic-graph hot path of StarPlat Dynamic (arXiv 2507.11094).

Drop-in for the reference `graphdyn` package's store + engine front door on
the three shipped programs: load a graph into a GPU-resident diff-CSR store,
apply ΔG batches, incrementally recompute SSSP / PageRank / triangle count.
All compute runs in sm_100a kernels behind the C ABI of include/gd_capi.h.
"""

from .engine import (CheckResult, ExecContext, NodePropertyTable, PRHandle, SSSPHandle, TCHandle, compile_source,
                     needs_reverse, run_batches, run_program, shipped_program, source_digest)
from .errors import (CompileError, ConfigurationError, ContractViolation, DeviceError, DivergenceError, ExecError,
                     GraphDynError, MalformedInputError)
from .graph import SENTINEL, Csr, DeleteReport, DiffCsr, DynamicGraph, EdgeRef
from .io import dump_graph, load_graph, parse_edge_lines
from .updates import (ADD, DELETE, RecordArrays, UpdateBatch, UpdateRecord, UpdateStream, dump_update_stream,
                      load_update_stream, parse_update_line)

__version__ = "0.1.0"

__all__ = [
    "ADD", "DELETE", "SENTINEL", "CheckResult", "CompileError", "ConfigurationError", "ContractViolation", "Csr",
    "DeleteReport", "DeviceError", "DiffCsr", "DivergenceError", "DynamicGraph", "EdgeRef", "ExecContext",
    "ExecError", "GraphDynError", "MalformedInputError", "NodePropertyTable", "PRHandle", "RecordArrays",
    "SSSPHandle", "TCHandle", "UpdateBatch", "UpdateRecord", "UpdateStream", "compile_source", "dump_graph",
    "dump_update_stream", "load_graph", "load_update_stream", "needs_reverse", "parse_edge_lines",
    "parse_update_line", "run_batches", "run_program", "shipped_program", "source_digest",
]
