"""B200-native layout conversion and transfer of record collections.

Drop-in for the hot path of soakit (Marionette, arXiv 2511.04853): the same
collection / layout / transfer / behavior API, with the transfer engine, the
jagged packer and the case-study kernel running as hand-written sm_100a
kernels in libsoakit_b200.so (C-ABI in include/soakit_b200.h).
"""

from . import behaviors, convert, jagged, layouts, memctx, schema, sensor, transfer, workloads
from .collection import Collection
from .convert import Aosoa, AosoaField, from_aosoa, to_aosoa
from .devarray import DeviceArray
from .errors import (
    AccessError,
    AllocationError,
    BenchConfigError,
    BoundsError,
    BufferStateError,
    CapacityError,
    CollectionError,
    CopyError,
    KindError,
    LayoutError,
    MemoryContextError,
    NotResizableError,
    PlanError,
    RegistryError,
    SchemaError,
    SchemaMismatchError,
    SoakitError,
    StaleViewError,
    TransferError,
    UnboundLeafError,
    UnknownBehaviorError,
    UnsupportedTransferError,
)
from .layouts import AOS, ARENA, PER_FIELD, ArenaSpec
from .memctx import CUDA, HOST, PINNED, ContextInfo, execution_scope
from .schema import (
    BOOL,
    F32,
    F64,
    I32,
    I64,
    MAIN_TAG,
    U8,
    U16,
    U32,
    U64,
    Schema,
    declare_array,
    declare_behavior,
    declare_global,
    declare_jagged,
    declare_per_item,
    declare_subgroup,
    enum_type,
)
from .transfer import (
    ExternalBinding,
    PreparedTransfer,
    TransferPriority,
    copy_collection,
    export_external,
    import_external,
    move_collection,
    prepare,
    register_transfer,
)

__version__ = "0.1.0"
