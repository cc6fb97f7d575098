"""END-TO-END TEST HARNESS (not product code): the reference's toy decoder and
request loop (ToyModel, run_request, run_dense) with the B200 hot path inside,
built from harness/engine.cpp into harness/libsfi_toy.so and the _sfi_toy
module by paper_2603_12038_b200/build.py. Used by tests/test_engine.py."""
import paper_2603_12038_b200  # noqa: F401  (loads _sfi_b200 and libsfi_b200.so first)

from ._sfi_toy import (  # noqa: F401
    DenseResult,
    RequestResult,
    RunOptions,
    ToyModel,
    argmax_token,
    run_dense,
    run_request,
)
