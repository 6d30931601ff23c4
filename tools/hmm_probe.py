from cuda.bindings import runtime as rt
for name in ("cudaDevAttrPageableMemoryAccess", "cudaDevAttrPageableMemoryAccessUsesHostPageTables",
             "cudaDevAttrConcurrentManagedAccess", "cudaDevAttrHostRegisterSupported",
             "cudaDevAttrHostRegisterReadOnlySupported", "cudaDevAttrCanUseHostPointerForRegisteredMem"):
    print(name, rt.cudaDeviceGetAttribute(getattr(rt.cudaDeviceAttr, name), 0))
