"""paper_1704_00605_b200 -- base64 encode / validating decode on B200.

Thin Python binding (ctypes argument marshalling only) over the C ABI of
``libb64gpu.so`` (``include/b64gpu.h``).  Every step of the codec runs in the
library's sm_100a kernels; PyTorch supplies device memory and streams.  There
is no CPU fallback: if the shared library is missing, importing the binding
functions raises.

Paper: W. Mula, D. Lemire, "Faster Base64 Encoding and Decoding using AVX2
Instructions", arXiv 1704.00605 (Alg 1, Alg 2).
"""
from ._lib import (  # noqa: F401
    B64_ERR_ARG,
    B64_ERR_CUDA,
    B64_ERR_INVALID_CHAR,
    B64_ERR_LENGTH,
    B64_ERR_NONCANONICAL,
    B64_FLAG_NOPAD,
    B64_FLAG_STRICT,
    B64_FLAG_URL,
    b64_decode_ex,
    b64_despace,
    b64_decode_ws,
    b64_batch_shard,
    b64_encode_wrapped,
    b64_encoded_len_wrapped,
    b64_decode_ws_async,
    b64_decode_ws_workspace_bytes,
    b64_decode_ex_async,
    b64_decoded_max_len_ex,
    b64_encode_ex,
    b64_encoded_len_ex,
    B64_ERR_WORKSPACE,
    B64_OK,
    B64Error,
    b64_batch_workspace_bytes,
    b64_build_info,
    b64_decode,
    b64_decode_async,
    b64_decode_batch,
    b64_decode_host,
    b64_decode_shard_async,
    b64_decoded_max_len,
    b64_encode,
    b64_encode_batch,
    b64_encode_host,
    b64_encoded_len,
    b64_shard,
    b64_shard_key,
    b64_combine_shards,
    b64_combine_shards_async,
    b64_decode_shard_ex_async,
    INT64_MAX,
    b64_decode_scratch_async,
    scratch_tensor,
    b64_status_str,
    lib_path,
    load_library,
    result_tensor,
    unpack_result,
)
from ._lib import EXPORTS  # noqa: F401
