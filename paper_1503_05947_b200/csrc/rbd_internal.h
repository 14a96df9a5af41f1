// rbd_internal.h — shared between the library's translation units (not part of
// the C ABI; hidden from the shared object's dynamic symbol table).
#pragma once

#include <string>

// Records msg as the thread's rbd_last_error() and returns code.
extern "C" __attribute__((visibility("hidden"))) int rbd_internal_set_error(int code,
                                                                            const char* msg);

inline int rbd_internal_set_error(int code, const std::string& msg) {
  return rbd_internal_set_error(code, msg.c_str());
}
