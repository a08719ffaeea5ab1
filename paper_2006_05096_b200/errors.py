"""Error hierarchy for the B200 hot path.

Mirrors the stable ``code`` / ``http_status`` contract of the reference's
``modelci.errors`` (pkg/src/modelci/errors.py:8-173) so callers that switch on
``exc.code`` keep working when they swap in this package.  Only the classes the
hot path can raise are defined; each one keeps the reference's code string.

C-ABI status codes from ``libb2`` (include/b2.h) map onto these classes in
``runtime.py``:  B2_ERR_FORMAT -> PlanFormatError (a ToyFormatError sibling),
B2_ERR_LAUNCH/B2_ERR_CUDA at plan creation -> LaunchFailure, at forward/bench
time -> CellFailure.
"""

from __future__ import annotations


class ModelCIError(Exception):
    """Root of every error this package raises (reference errors.py:8-20)."""

    code = "INTERNAL"
    http_status = 500

    def __init__(self, message: str = "", **details):
        text = message or type(self).__name__
        super().__init__(text)
        self.message = text
        self.details = details

    def to_dict(self) -> dict:
        return {"code": self.code, "message": self.message, "details": self.details}


def _kind(name: str, code: str, status: int, doc: str = "", base=ModelCIError):
    cls = type(name, (base,), {"code": code, "http_status": status,
                               "__doc__": doc or f"{code} ({status})"})
    return cls


# registry-side codes the profiler can surface (errors.py:25-70)
NotFound = _kind("NotFound", "NOT_FOUND", 404)
InvalidManifest = _kind("InvalidManifest", "INVALID_MANIFEST", 422)
IllegalTransition = _kind("IllegalTransition", "ILLEGAL_TRANSITION", 409)
# converter (errors.py:75-106)
DuplicatePlugin = _kind("DuplicatePlugin", "DUPLICATE_PLUGIN", 409)
InvalidPlugin = _kind("InvalidPlugin", "INVALID_PLUGIN", 422)
UnsupportedConversion = _kind("UnsupportedConversion", "UNSUPPORTED_CONVERSION", 422)
PluginFailure = _kind("PluginFailure", "PLUGIN_FAILURE", 500)
ConversionTimeout = _kind("ConversionTimeout", "CONVERSION_TIMEOUT", 500)
ToyFormatError = _kind("ToyFormatError", "TOY_FORMAT_ERROR", 422,
                       "Malformed toy-format payload (reference errors.py:101-106).")
PlanFormatError = _kind("PlanFormatError", "PLAN_FORMAT_ERROR", 422,
                        "Malformed b200-plan blob (bad magic, CRC, op table).")
# dispatcher (errors.py:111-127)
IncompatibleFormat = _kind("IncompatibleFormat", "INCOMPATIBLE_FORMAT", 422)
UnknownDevice = _kind("UnknownDevice", "UNKNOWN_DEVICE", 422)
LaunchFailure = _kind("LaunchFailure", "LAUNCH_FAILURE", 500)
ReadyTimeout = _kind("ReadyTimeout", "READY_TIMEOUT", 503)
# profiler (errors.py:132-157)
EmptySamples = _kind("EmptySamples", "EMPTY_SAMPLES", 400)
EmptyTrace = _kind("EmptyTrace", "EMPTY_TRACE", 400)
CellFailure = _kind("CellFailure", "CELL_FAILURE", 500)
RequestFailure = _kind("RequestFailure", "REQUEST_FAILURE", 500)
JobAborted = _kind("JobAborted", "JOB_ABORTED", 409)
# telemetry / gateway (errors.py:162-173)
ProviderFailure = _kind("ProviderFailure", "PROVIDER_FAILURE", 503)
InvalidRequest = _kind("InvalidRequest", "INVALID_REQUEST", 400)
