// sb_error.h -- thread-local last-error message shared by every C-ABI entry point.
#pragma once
namespace sb {
// Records a printf-style message for sb_last_error() and returns `code`.
int fail(int code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
const char* last_error();
}  // namespace sb
