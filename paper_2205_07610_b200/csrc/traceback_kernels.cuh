// placeholder: replaced by the direction-code traceback kernels
#pragma once
namespace wsb { struct TracebackState { void release() {} }; }
